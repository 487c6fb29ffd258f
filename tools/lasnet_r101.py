#!/usr/bin/env python
"""LAS-ResNet-101 network throughput (BASELINE configs[2]): ImageNet
224x224, batch N on one GPU (default 256), S_net 4-4-2-1, masker biases
calibrated so that ~r of the cells of every dynamic block are active on the
activations it sees.  The whole forward (stem, pool, 4 projection blocks, 29
dynamic identity blocks, head) is one CUDA graph; the comparator is the same
network with the identity blocks run dense (lasnet_dense_block).  Random-init
weights, synthetic N(0,1) images.  Median of --steps replays.

  python tools/lasnet_r101.py [--n 256] [--r 0.5] [--steps 10] [--out gpurun_out/lasnet_r101]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402


def timed(fn, steps, warmup=3):
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    ev = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        ev.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return statistics.median(ms), ms[0], ms[-1]


def breakdown(net, x, steps):
    """Eager per-section times (ms, medians): stem + pool, each projection block, each
    stage's dynamic blocks, head."""
    lib = L._lib.load()
    st = torch.cuda.current_stream()
    secs = {}

    def rec(name, fn):
        ts = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        secs[name] = statistics.median(a.elapsed_time(b) for a, b in ts)

    n, h = net.n, net.hw // 2
    rec("stem+pool", lambda: (L.stem(x, net.stem_w, net.stem_b, ws=net.stem_ws), None))
    y = L.stem(x, net.stem_w, net.stem_b, ws=net.stem_ws)
    rec("stem+pool", lambda: (lib.lasnet_stem(n, h, h, L.block._p(x), L.block._p(net.stem_w), L.block._p(net.stem_b),
                                              L.block._p(net.stem_y), L.block._p(net.stem_ws), net.stem_ws.numel(),
                                              L.block._stream()),
                              lib.lasnet_maxpool(n, h // 2, h // 2, 64, L.block._p(net.stem_y), L.block._p(net.pool_y),
                                                 L.block._stream())))
    del y
    cur = net.pool_y
    for si, (proj, dyn) in enumerate(net.stages):
        rec(f"proj{si}", lambda: proj.forward(cur))
        out = proj.forward(cur)
        keep = out.clone()

        def run_dyn():
            out.copy_(keep)
            for blk in dyn:
                blk.forward(out)

        rec(f"dyn{si} (+copy)", run_dyn)
        cur = out
    return secs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--r", type=float, nargs="+", default=[0.5])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "lasnet_r101"))
    args = ap.parse_args()
    from paper_2210_06223_b200 import build

    build.build()
    wts = synth.make_lasnet_weights(seed=11)
    x = synth.make_image_batch(args.n, 224, seed=0).cuda()
    rows = []
    dense = None
    for r in args.r:
        net = L.LASResNet(args.n, wts, hw=224, r=r)
        net.forward(x, calibrate_r=r)
        torch.cuda.synchronize()
        rates = [float(b.mask_buf.float().mean().item()) for b in net.blocks()]
        g = net.capture(x)
        t, lo, hi = timed(g.replay, args.steps)
        if dense is None:
            gd = net.capture(x, dense=True)
            dense = timed(gd.replay, args.steps)
            del gd
        parts = breakdown(net, x, args.steps) if r == args.r[0] else None
        rows.append(dict(r_target=r, r_patch_mean=sum(rates) / len(rates), ms=t, ms_min=lo, ms_max=hi,
                         images_per_s=args.n / (t * 1e-3), speedup_vs_dense=dense[0] / t, breakdown_ms=parts))
        if parts:
            print("  eager breakdown (ms):", {k: round(v, 3) for k, v in parts.items()}, flush=True)
        print(f"r={r}: {t:.3f} ms/forward ({args.n / (t * 1e-3):.0f} images/s), dense identity blocks "
              f"{dense[0]:.3f} ms ({args.n / (dense[0] * 1e-3):.0f} images/s), x{dense[0] / t:.2f}; "
              f"mean r_patch {rows[-1]['r_patch_mean']:.3f}", flush=True)
        del net, g
        torch.cuda.empty_cache()
    out = dict(model="LAS-ResNet-101 (S_net 4-4-2-1; projection blocks static)", n=args.n, hw=224, rows=rows,
               dense_ms=dense[0], dense_images_per_s=args.n / (dense[0] * 1e-3),
               device=torch.cuda.get_device_name(0), data="synthetic N(0,1) images, random-init weights",
               launch="one CUDA graph per forward")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out + ".json", "w"), indent=1)


if __name__ == "__main__":
    main()
