#!/usr/bin/env python
"""BASELINE configs[0] / SURVEY C1: one LASNet bottleneck, N=1, 14x14x256 (c_mid 64),
S=2, 25 of 49 cells active, fp32 -- the fp32 CUDA-core path (masker + compaction +
three convolutions).  SURVEY 8(d): its roofline (21.7 MFLOP at the fp32 SIMT
peak, ~0.3 us) is far below launch latency, so the number is latency-bound by
construction; reported eager (one launch per kernel, PDL) and as a CUDA-graph replay,
with the dense comparator, median of --steps.

  python tools/config1.py [--steps 200] [--out gpurun_out/config1]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402


def med(fn, steps):
    st = torch.cuda.current_stream()
    ev = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "config1"))
    args = ap.parse_args()
    from paper_2210_06223_b200 import build

    build.build()
    n, h, w, c, cm, s = 1, 14, 14, 256, 64, 2
    res = {}
    for dt, tdt in (("f32", torch.float32), ("bf16", torch.bfloat16)):
        x = synth.make_x(n, h, w, c, seed=0, dtype=dt).cuda()
        wts = synth.make_block_weights(c, cm, c, seed=1, dtype=dt)
        wm = synth.make_masker_weights(c, seed=2)
        blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, s, tdt), wts, wm, 0.0)
        blk.calibrate_bias(synth.make_x(n, h, w, c, seed=1000, dtype=dt).cuda(), 25 / 49)
        y, y2 = x.clone(), torch.empty_like(x)
        for _ in range(5):
            blk.forward(y)
        torch.cuda.synchronize()
        eager = med(lambda: blk.forward(y), args.steps)
        g = blk.capture(y)
        graph = med(g.replay, args.steps)
        dense = med(lambda: blk.dense(x, y2), args.steps)
        active = int(blk.count.item())
        res[dt] = dict(eager_us=eager, graph_us=graph, dense_us=dense, active_cells=active, cells=49)
        print(f"{dt}: dyn block eager {eager:.2f} us, graph replay {graph:.2f} us, dense {dense:.2f} us, "
              f"active {active}/49", flush=True)
    out = dict(config="N=1 14x14x256 c_mid 64 S=2 (BASELINE configs[0])", device=torch.cuda.get_device_name(0),
               steps=args.steps, results=res, roofline_us_f32_simt=0.29,
               note="latency-bound by construction (SURVEY 8(d)); not L2-flushed (inputs stay L2-resident)")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out + ".json", "w"), indent=1)


if __name__ == "__main__":
    main()
