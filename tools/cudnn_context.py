#!/usr/bin/env python
"""Context only (SURVEY 8(d) "dense comparators"): the same static bottleneck
block run by PyTorch / cuDNN (channels_last bf16 conv2d x 3 + bias + ReLU +
residual), next to this library's lasnet_dense_block (the same kernels as the
dynamic path, on every pixel) and the dynamic block at r = 0.5.  NOT the product
path -- a yardstick for the dense kernels.

  python tools/cudnn_context.py [--steps 50] [--out gpurun_out/cudnn_context]
"""
import argparse
import json
import os
import statistics
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

SHAPES = [  # n, hw, c_in, c_mid, S
    (128, 28, 512, 128, 4),    # bench workload (BASELINE configs[1])
    (256, 14, 1024, 256, 2),   # LAS-R101 stage 3 block (configs[2])
]


def timed(fn, steps, flush):
    st = torch.cuda.current_stream()
    for _ in range(5):
        flush.sum()
        fn()
    ev = []
    for _ in range(steps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cudnn_context"))
    args = ap.parse_args()
    from paper_2210_06223_b200 import build

    build.build()
    torch.backends.cudnn.benchmark = True
    flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
    rows = []
    for n, hw, c_in, c_mid, s in SHAPES:
        x = synth.make_x(n, hw, hw, c_in, seed=0).cuda()
        wts = synth.make_block_weights(c_in, c_mid, c_in, seed=1)
        wm = synth.make_masker_weights(c_in, seed=2)
        # torch layouts: NCHW-logical tensors in channels_last memory, OIHW weights
        xt = x.permute(0, 3, 1, 2)  # NHWC storage == channels_last
        w1 = wts["w1"].cuda()[:, :, None, None].contiguous(memory_format=torch.channels_last)
        w2 = wts["w2"].cuda().permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
        w3 = wts["w3"].cuda()[:, :, None, None].contiguous(memory_format=torch.channels_last)
        b1, b2, b3 = (wts[k].cuda().to(torch.bfloat16) for k in ("b1", "b2", "b3"))

        def torch_block():
            h1 = F.relu(F.conv2d(xt, w1, b1))
            h2 = F.relu(F.conv2d(h1, w2, b2, padding=1))
            return F.relu(F.conv2d(h2, w3, b3) + xt)

        blk = L.DynBlock(L.BlockShape(n, hw, hw, c_in, c_mid, s), wts, wm, 0.0,
                         schedule=L.choose_schedule(n, hw, hw, c_in, c_mid, c_in, s, 0.5))
        blk.calibrate_bias(synth.make_x(n, hw, hw, c_in, seed=1000).cuda(), 0.5)
        y, y2 = torch.empty_like(x), torch.empty_like(x)
        t_torch = timed(torch_block, args.steps, flush)
        t_dense = timed(lambda: blk.dense(x, y2), args.steps, flush)
        t_dyn = timed(lambda: blk.forward(y.copy_(x)), args.steps, flush)
        t_copy = timed(lambda: y.copy_(x), args.steps, flush)
        rows.append(dict(n=n, hw=hw, c_in=c_in, c_mid=c_mid, S=s, torch_cudnn_us=t_torch, lasnet_dense_us=t_dense,
                         lasnet_dyn_r05_us=t_dyn - t_copy))
        print(rows[-1], flush=True)
    json.dump(dict(rows=rows, device=torch.cuda.get_device_name(0), note="context only, not the product path"),
              open(args.out + ".json", "w"), indent=1)


if __name__ == "__main__":
    main()
