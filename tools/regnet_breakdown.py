#!/usr/bin/env python
"""Per-kernel breakdown of the LAS-RegNetY-800MF forward (eager, CUDA events around
every library launch), dynamic and dense comparator.  python tools/regnet_breakdown.py [--n 512]"""
import argparse
import ctypes
import os
import statistics
import sys
from collections import defaultdict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    args = ap.parse_args()
    lib = L._lib.load()
    net = L.LASRegNet(args.n, synth.make_regnet_weights(seed=21), hw=224)
    x = synth.make_image_batch(args.n, 224, seed=1).cuda()
    net.forward(synth.make_image_batch(args.n, 224, seed=2).cuda(), calibrate_r=0.5)
    st = torch.cuda.current_stream()
    nmax = 256
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nmax)]
    for e in evs:
        e.record(st)
    arr = (ctypes.c_void_p * len(evs))(*[e.cuda_event for e in evs])
    for dense in (False, True):
        agg = defaultdict(list)
        for rep in range(4):
            trace = []
            lib.lasnet_set_kernel_events(arr, nmax)
            net.forward(x, dense=dense, trace=trace)
            cnt = lib.lasnet_kernel_event_count()
            names = [lib.lasnet_kernel_event_name(i).decode() for i in range(cnt)]
            lib.lasnet_set_kernel_events(None, 0)
            torch.cuda.synchronize()
            if rep:
                tot = defaultdict(float)
                for t in trace:
                    for i in range(t["ev0"], t["ev1"]):
                        tot[(t.get("stage"), t["kind"], names[i])] += evs[2 * i].elapsed_time(evs[2 * i + 1])
                for k, v in tot.items():
                    agg[k].append(v)
        print("dense" if dense else "dynamic", "total %.3f ms" % sum(statistics.median(v) for v in agg.values()))
        for k, v in sorted(agg.items(), key=lambda kv: -statistics.median(kv[1])):
            print("  ", k, "%.4f" % statistics.median(v))


if __name__ == "__main__":
    main()
