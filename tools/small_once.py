"""config 1 (N=1, 14x14x256, c_mid 64, S=2, fp32) through lasnet_block_forward (the
single-launch small-batch block) and lasnet_dense_block, under cudaProfilerStart/Stop."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

n, h, w, c, cm, s = 1, 14, 14, 256, 64, 2
x = synth.make_x(n, h, w, c, seed=0, dtype="f32").cuda()
wts = synth.make_block_weights(c, cm, c, seed=1, dtype="f32")
blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, s, torch.float32), wts, synth.make_masker_weights(c, seed=2), 0.0,
                 schedule=L.SCHED_SEPARATE)
blk.calibrate_bias(x, 25 / 49)
y, y2 = x.clone(), torch.empty_like(x)
for _ in range(3):
    blk.forward(y)
    blk.dense(x, y2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
blk.forward(y)
blk.dense(x, y2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("small_once ok", int(blk.count.item()))
