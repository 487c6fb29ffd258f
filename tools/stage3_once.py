#!/usr/bin/env python
"""One LAS-R101 stage-3 identity block (N=256, 14x14x1024, c_mid 256, S=2, r=0.5),
masker-fused schedule, and the dense comparator under cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures.  Shape overrides: --n --hw --c --cm --s."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--hw", type=int, default=14)
ap.add_argument("--c", type=int, default=1024)
ap.add_argument("--cm", type=int, default=256)
ap.add_argument("--s", type=int, default=2)
ap.add_argument("--no-dense", action="store_true")
a = ap.parse_args()
n, h, w, c, cm, s = a.n, a.hw, a.hw, a.c, a.cm, a.s
x = synth.make_x(n, h, w, c, seed=0).cuda()
wts = synth.make_block_weights(c, cm, c, seed=1)
wm = synth.make_masker_weights(c, seed=2)
b = L.DynBlock(L.BlockShape(n, h, w, c, cm, s), wts, wm, 0.0, schedule=L.SCHED_FUSED)
b.calibrate_bias(synth.make_x(n, h, w, c, seed=1000).cuda(), 0.5)
y = x.clone()
y2 = torch.empty_like(x)
b.forward(y)
b.dense(x, y2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
y.copy_(x)
b.forward(y)
if not a.no_dense:
    b.dense(x, y2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("stage3_once ok")
