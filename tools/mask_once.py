"""The first blocks' standalone masker at LAS-R101 shapes (stage 0: 256 x 56 x 56 x 64, window 4;
stage 1: 256 x 56 x 56 x 256, window 8 = stride 2 x S 4; stage 2: 256 x 28 x 28 x 512, window 4)
under cudaProfilerStart/Stop, for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

cases = [(256, 56, 56, 64, 4), (256, 56, 56, 256, 8), (256, 28, 28, 512, 4)]
xs = [synth.make_x(n, h, w, c, seed=1).cuda() for n, h, w, c, s in cases]
wms = [synth.make_masker_weights(c, seed=2).cuda() for n, h, w, c, s in cases]
for _ in range(2):
    for (n, h, w, c, s), x, wm in zip(cases, xs, wms):
        L.mask(x, wm, 0.0, s)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for (n, h, w, c, s), x, wm in zip(cases, xs, wms):
    L.mask(x, wm, 0.0, s)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("mask_once ok")
