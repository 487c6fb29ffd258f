#!/usr/bin/env python
"""The configs[1] block (N=128, 28x28x512, c_mid 128, S=4, r=0.5) under
cudaProfilerStart/Stop, both schedules and the dense comparator, for
`ncu --profile-from-start off` captures of the block's kernels."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

n, h, w, c, cm, s = 128, 28, 28, 512, 128, 4
x = synth.make_x(n, h, w, c, seed=0).cuda()
wts = synth.make_block_weights(c, cm, c, seed=1)
wm = synth.make_masker_weights(c, seed=2)
blks = [L.DynBlock(L.BlockShape(n, h, w, c, cm, s), wts, wm, 0.0, schedule=sc) for sc in (L.SCHED_FUSED, None)]
for b in blks:
    b.calibrate_bias(synth.make_x(n, h, w, c, seed=1000).cuda(), 0.5)
y = x.clone()
y2 = torch.empty_like(x)
for b in blks:
    b.forward(y)
blks[0].dense(x, y2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for b in blks:
    y.copy_(x)
    b.forward(y)
blks[0].dense(x, y2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("block_once ok")
