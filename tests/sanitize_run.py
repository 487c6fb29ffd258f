"""Tiny invocation of every kernel of the library, for compute-sanitizer
(tests/test_sanitizer.py): masker (alone and fused with compaction), compaction,
both block schedules at S = 2 / 4 (gather, direct and fused conv23 paths, the
cooperative decide with its grid barrier), the unfused conv2/conv3 (c_mid 256),
the dense comparator, the projection block, stem / max pool / head and a small
LAS-ResNet forward.  Exits 0 after a synchronize; the sanitizer reports errors."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402


def dev(w):
    return {k: v.cuda() for k, v in w.items()}


def main():
    torch.cuda.init()
    for (n, h, w, c, cm, s) in [(2, 12, 12, 256, 64, 2), (2, 16, 16, 256, 128, 4), (1, 14, 14, 512, 256, 2)]:
        x = synth.make_x(n, h, w, c, seed=1).cuda()
        wts = dev(synth.make_block_weights(c, cm, c, seed=2))
        wm = synth.make_masker_weights(c, seed=3).cuda()
        L.mask(x, wm, 0.0, s, logits=True)
        m = L.mask(x, wm, 0.01, s)
        idx, cnt = L.compact(m)
        L.dyn_block(x.clone(), wts, idx, cnt, s)
        for sched in (L.SCHED_SEPARATE, L.SCHED_FUSED):
            L.block_forward(x.clone(), wts, wm, 0.0, s, sched)
        L.dense_block(x, wts)
    # fp32 CUDA-core path (config 1)
    x = synth.make_x(1, 14, 14, 256, seed=8, dtype="f32").cuda()
    wts = dev(synth.make_block_weights(256, 64, 256, seed=9, dtype="f32"))
    wm = synth.make_masker_weights(256, seed=10).cuda()
    m = L.mask(x, wm, 0.0, 2)
    idx, cnt = L.compact(m)
    L.dyn_block(x.clone(), wts, idx, cnt, 2)
    L.dense_block(x, wts)  # the single-launch small-batch block (fp32)
    L.block_forward(x.clone(), wts, wm, 0.0, 2, L.SCHED_SEPARATE)
    xp = synth.make_x(2, 16, 16, 128, seed=4).cuda()
    L.proj_block(xp, dev(synth.make_proj_weights(128, 64, 256, seed=5)), 2)
    # LAS-RegNetY: both dynamic schedules (grouped conv, SE) and a static stride-2 first block
    for sched in (L.SCHED_SEPARATE, L.SCHED_FUSED):
        rw = synth.make_regnet_block_weights(144, 144, 36, False, seed=11)
        xr = torch.zeros((2, 14, 14, 192), dtype=torch.bfloat16)
        xr[..., :144] = synth.make_x(2, 14, 14, 144, seed=12)
        blk = L.RegNetBlock(2, 14, 14, 192, 192, 1, rw, s=2, dynamic=True, schedule=sched)
        blk.forward(xr.cuda())
    rp = synth.make_regnet_block_weights(64, 144, 16, True, seed=13)
    L.RegNetBlock(2, 16, 16, 64, 192, 2, rp).forward(synth.make_x(2, 16, 16, 64, seed=14).cuda())
    net = L.LASResNet(1, synth.make_lasnet_weights(seed=6), hw=64)
    net.forward(synth.make_image_batch(1, 64, seed=7).cuda())
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
