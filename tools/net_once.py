#!/usr/bin/env python
"""One eager LAS-ResNet-101 forward (BASELINE configs[2] shape, N=256 224x224, r=0.5,
biases calibrated on a separate batch) between cudaProfilerStart/Stop, for
`ncu --profile-from-start off`; prints the library's kernel-event names in launch
order (one name may cover two launches: decide+ids / decide+gather) as JSON to
--names.  --regnet: the LAS-RegNetY-800MF forward (N=512) instead."""
import argparse
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--regnet", action="store_true")
    ap.add_argument("--names", default=os.path.join(ROOT, "gpurun_out", "net_once_names.json"))
    args = ap.parse_args()
    lib = L._lib.load()
    if args.regnet:
        net = L.LASRegNet(args.n, synth.make_regnet_weights(seed=21), hw=224)
    else:
        net = L.LASResNet(args.n, synth.make_lasnet_weights(seed=11), hw=224)
    x = synth.make_image_batch(args.n, 224, seed=1).cuda()
    net.forward(synth.make_image_batch(args.n, 224, seed=2).cuda(), calibrate_r=0.5)
    net.forward(x)
    torch.cuda.synchronize()
    nmax = 512
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nmax)]
    for e in evs:
        e.record()
    arr = (ctypes.c_void_p * len(evs))(*[e.cuda_event for e in evs])
    trace = []
    torch.cuda.profiler.start()
    lib.lasnet_set_kernel_events(arr, nmax)
    net.forward(x, trace=trace)
    cnt = lib.lasnet_kernel_event_count()
    names = [lib.lasnet_kernel_event_name(i).decode() for i in range(cnt)]
    lib.lasnet_set_kernel_events(None, 0)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    layers = []
    for t in trace:
        layers.append({"kind": t["kind"], "stage": t.get("stage"), "block": t.get("block"),
                       "names": names[t["ev0"]:t["ev1"]]})
    json.dump({"names": names, "layers": layers}, open(args.names, "w"), indent=1)
    print(len(names), "event names")


if __name__ == "__main__":
    main()
