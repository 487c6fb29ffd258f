"""Graph-replay times of the LAS-R101 forward (N=256, r=0.5) and the configs[1]
block (N=128, 28x28x512, c_mid 128, S=4, fused), for env-knob A/B probes
(e.g. LASNET_DECIDE_PROBE=2: no decide launch in captures).  No correctness checks."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402


def timed(g, k=20, pre=None):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


N = 256
weights = synth.make_lasnet_weights(seed=1)
net = L.LASResNet(N, weights, hw=224)
net.forward(synth.make_image_batch(N, 224, seed=5000).cuda(), calibrate_r=0.5)
x = synth.make_image_batch(N, 224, seed=1).cuda()
net.forward(x)
gf = net.capture(x)
print(f"net {timed(gf):.4f} ms")
n, h, w, c, cm = 128, 28, 28, 512, 128
xb = synth.make_x(n, h, w, c, seed=0).cuda()
blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, 4), synth.make_block_weights(c, cm, c, seed=1),
                 synth.make_masker_weights(c, seed=2), 0.0, schedule=L.SCHED_FUSED)
blk.calibrate_bias(synth.make_x(n, h, w, c, seed=1000).cuda(), 0.5)
y = xb.clone()
blk.forward(y)
g = blk.capture(y)
print(f"block {1e3 * timed(g, 200):.1f} us (in place, L2-warm)")
