#!/usr/bin/env python
"""A/B timing of the configs[1] block (N=128, 28x28x512, c_mid 128) for library
build variants: S in {2, 4, 7}, r = 0.5, both schedules, mean of 30 CUDA-graph
replays with the L2 flushed (256 MiB read) before each, plus the dense comparator,
and per-kernel event times of the fused schedule at S = 4.  Prints one JSON line."""
import ctypes
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "default"
    n, h, w, c, cm = 128, 28, 28, 512, 128
    x = synth.make_x(n, h, w, c, seed=0).cuda()
    xc = synth.make_x(n, h, w, c, seed=1000).cuda()
    wts = synth.make_block_weights(c, cm, c, seed=1)
    wm = synth.make_masker_weights(c, seed=2)
    flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    y = torch.empty_like(x)
    out = {"tag": tag}
    for s in (2, 4, 7):
        for sched in (L.SCHED_FUSED, None):
            blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, s), wts, wm, 0.0, schedule=sched)
            blk.calibrate_bias(xc, 0.5)
            y.copy_(x)
            g = blk.capture(y)
            ts = []
            for k in range(35):
                y.copy_(x)
                flush.sum()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                g.replay()
                b.record(st)
                if k >= 5:
                    ts.append((a, b))
            torch.cuda.synchronize()
            out[f"S{s}_{'fused' if sched else 'sep'}_us"] = round(statistics.fmean(a.elapsed_time(b) for a, b in ts) * 1e3, 1)
            if s == 4 and sched:
                lib = L._lib.load()
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(16)]
                for e in evs:
                    e.record(st)
                arr = (ctypes.c_void_p * 16)(*[e.cuda_event for e in evs])
                per = []
                for k in range(10):
                    y.copy_(x)
                    flush.sum()
                    lib.lasnet_set_kernel_events(arr, 8)
                    blk.forward(y)
                    cnt = lib.lasnet_kernel_event_count()
                    names = [lib.lasnet_kernel_event_name(i).decode() for i in range(cnt)]
                    lib.lasnet_set_kernel_events(None, 0)
                    torch.cuda.synchronize()
                    per.append([evs[2 * i].elapsed_time(evs[2 * i + 1]) * 1e3 for i in range(cnt)])
                out["S4_fused_kernels_us"] = {nm: round(statistics.fmean(v), 1) for nm, v in zip(names, zip(*per))}
            del g, blk
    blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, 4), wts, wm, 0.0)
    y2 = torch.empty_like(x)
    ts = []
    for k in range(35):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        blk.dense(x, y2)
        b.record(st)
        if k >= 5:
            ts.append((a, b))
    torch.cuda.synchronize()
    out["dense_us"] = round(statistics.fmean(a.elapsed_time(b) for a, b in ts) * 1e3, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
