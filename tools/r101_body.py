#!/usr/bin/env python
"""LAS-ResNet-101 identity-block body at ImageNet shapes (BASELINE configs[2]).

ResNet-101 has 33 bottlenecks; 29 are stride-1 identity blocks -- the ones
this library runs dynamically (the 4 stride-2 / projection first blocks, the
stem and the classifier are SURVEY 8(f) NEXT-f1 and are NOT timed here).  Per
stage (56x56/256/64 S=4 x2, 28x28/512/128 S=4 x3, 14x14/1024/256 S=2 x22,
7x7/2048/512 S=1 x2; S_net 4-4-2-1), one identity block is timed
at batch N (default 256 = the whole global batch on one GPU): the whole
dynamic block (masker-driven, bias calibrated to r on a separate batch,
schedule = lasnet_choose_schedule unless --schedule) and the dense comparator
(the same kernels on every pixel).  Each is a median of --steps runs with L2
flushed before each; the body time is the per-stage block time times the
number of identity blocks.  Random-init weights, synthetic inputs.

  python tools/r101_body.py [--n 256] [--r 0.5] [--steps 10] [--out gpurun_out/r101_body]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

STAGES = [  # h, c_in, c_mid, S, identity blocks
    (56, 256, 64, 4, 2),
    (28, 512, 128, 4, 3),
    (14, 1024, 256, 2, 22),
    (7, 2048, 512, 1, 2),
]


def timed(fn, prep, steps, warmup):
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        prep()
        fn()
    ev = []
    for _ in range(steps):
        prep()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def chained(args, flush):
    """Each stage's identity blocks as a real forward: block k's in-place output is
    block k+1's input, every block with its own weights and masker (bias calibrated
    in sequence on the activations it actually sees), the whole stage captured in
    one CUDA graph; median replay time, L2 flushed before each."""
    res, tot = [], 0.0
    for si, (h, c_in, c_mid, s, nblk) in enumerate(STAGES):
        n = args.n
        x0 = synth.make_x(n, h, h, c_in, seed=10 + si).cuda()
        y = x0.clone()
        blks = []
        for b in range(nblk):
            wts = synth.make_block_weights(c_in, c_mid, c_in, seed=100 * si + 2 * b + 1)
            wm = synth.make_masker_weights(c_in, seed=100 * si + 2 * b + 2)
            sched = L.choose_schedule(n, h, h, c_in, c_mid, c_in, s, args.r)
            blk = L.DynBlock(L.BlockShape(n, h, h, c_in, c_mid, s), wts, wm, 0.0, schedule=sched)
            blk.calibrate_bias(y, args.r)  # on this block's actual input
            blk.forward(y)
            blks.append(blk)
        torch.cuda.synchronize()
        rates = [float(b.mask_buf.float().mean().item()) for b in blks]

        def fwd():
            for b in blks:
                b.forward(y)

        y.copy_(x0)
        for _ in range(2):
            fwd()
        y.copy_(x0)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fwd()

        def prep():
            y.copy_(x0)
            flush.sum()

        t = timed(g.replay, prep, args.steps, args.warmup)
        tot += t
        res.append(dict(h=h, c_in=c_in, c_mid=c_mid, S=s, blocks=nblk, ms=t, r_patch_mean=sum(rates) / len(rates)))
        print(f"chained stage {h}x{h}x{c_in} x{nblk}: {t * 1e3:.1f} us ({t / nblk * 1e3:.1f} us/block), "
              f"mean r_patch {res[-1]['r_patch_mean']:.3f}", flush=True)
        del blks, x0, y, g
        torch.cuda.empty_cache()
    print(f"chained identity body: {tot:.3f} ms -> {args.n / (tot * 1e-3):.0f} images/s", flush=True)
    return dict(stages=res, body_ms=tot, images_per_s=args.n / (tot * 1e-3))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--r", type=float, default=0.5)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--schedule", default="auto", choices=["auto", "separate", "fused"])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "r101_body"))
    ap.add_argument("--per-block", type=int, default=1, help="time one block per stage (eager) and the dense comparator")
    ap.add_argument("--chain", type=int, default=1, help="also time each stage's identity blocks chained (block k "
                                                         "feeds block k+1, own weights and masker per block) as one "
                                                         "CUDA graph")
    args = ap.parse_args()
    from paper_2210_06223_b200 import build

    build.build()
    hbm, tfl, _, psrc = bench.peaks()
    flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
    rows, dyn_tot, dense_tot, roof_tot = [], 0.0, 0.0, 0.0
    for h, c_in, c_mid, s, nblk in (STAGES if args.per_block else []):
        n = args.n
        x = synth.make_x(n, h, h, c_in, seed=0).cuda()
        wts = synth.make_block_weights(c_in, c_mid, c_in, seed=1)
        wm = synth.make_masker_weights(c_in, seed=2)
        if args.schedule == "auto":
            sched = L.choose_schedule(n, h, h, c_in, c_mid, c_in, s, args.r)
        else:
            sched = L.SCHED_FUSED if args.schedule == "fused" else L.SCHED_SEPARATE
        blk = L.DynBlock(L.BlockShape(n, h, h, c_in, c_mid, s), wts, wm, 0.0, schedule=sched)
        blk.calibrate_bias(synth.make_x(n, h, h, c_in, seed=1000).cuda(), args.r)
        y, y2 = torch.empty_like(x), torch.empty_like(x)

        def prep():
            y.copy_(x)
            flush.sum()

        t_dyn = timed(lambda: blk.forward(y), prep, args.steps, args.warmup)
        t_dense = timed(lambda: blk.dense(x, y2), lambda: flush.sum(), args.steps, args.warmup)
        blk.forward(y.copy_(x))
        torch.cuda.synchronize()
        m = blk.mask_buf.cpu().numpy()
        _, bw, dw, st = bench.algorithmic_work(m, n, h, h, c_in, c_mid, c_in, s)
        t_roof = max(bw["bytes"] / (hbm * 1e9), bw["flops"] / (tfl * 1e12)) * 1e3
        t_dense_ideal = max(dw["bytes"] / (hbm * 1e9), dw["flops"] / (tfl * 1e12)) * 1e3
        row = dict(h=h, c_in=c_in, c_mid=c_mid, S=s, blocks=nblk, n=n, schedule="fused" if sched == L.SCHED_FUSED
                   else "separate", r_pixel=st["r_pixel"], dyn_ms=t_dyn, dense_ms=t_dense, t_roof_ms=t_roof,
                   dense_ideal_ms=t_dense_ideal, roof_frac=t_roof / t_dyn, speedup=t_dense / t_dyn)
        rows.append(row)
        dyn_tot += nblk * t_dyn
        dense_tot += nblk * t_dense
        roof_tot += nblk * t_roof
        print(f"stage {h}x{h}x{c_in} c_mid {c_mid} S={s} x{nblk} [{row['schedule']}] r_pix {st['r_pixel']:.3f}: "
              f"dyn {t_dyn * 1e3:.1f} us  dense {t_dense * 1e3:.1f} us  x{row['speedup']:.2f}  "
              f"T_roof {t_roof * 1e3:.1f} us ({row['roof_frac']:.2f})", flush=True)
        del x, y, y2, blk
        torch.cuda.empty_cache()
    chain = chained(args, flush) if args.chain else None
    out = dict(n=args.n, r=args.r, rows=rows, chained=chain, body_dyn_ms=dyn_tot, body_dense_ms=dense_tot, body_roof_ms=roof_tot,
               body_images_per_s_dyn=args.n / (dyn_tot * 1e-3), body_images_per_s_dense=args.n / (dense_tot * 1e-3),
               device=torch.cuda.get_device_name(0), peaks=dict(hbm_gbs=hbm, bf16_tflops=tfl, src=psrc))
    print(f"identity body (29 of 33 blocks): dyn {dyn_tot:.3f} ms, dense {dense_tot:.3f} ms, x{dense_tot / dyn_tot:.2f}; "
          f"roofline {roof_tot:.3f} ms ({roof_tot / dyn_tot:.2f}); {out['body_images_per_s_dyn']:.0f} images/s")
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(out, open(args.out + ".json", "w"), indent=1)
    with open(args.out + ".md", "w") as f:
        f.write(f"# LAS-ResNet-101 identity-block body ({out['device']}), N={args.n}, r={args.r}\n\n"
                "29 of the 33 bottlenecks (stride-1 identity blocks); stem, the 4 stride-2/projection blocks and the "
                "classifier are not included (SURVEY 8(f) NEXT-f1). Median of "
                f"{args.steps} runs per block, L2 flushed before each; body = per-stage block time x blocks.\n\n"
                "| stage | S | blocks | schedule | r pixel | dyn (us) | dense (us) | dense/dyn | T_roof (us) | roofline frac |\n"
                "|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['h']}x{r['h']}x{r['c_in']} (c_mid {r['c_mid']}) | {r['S']} | {r['blocks']} | {r['schedule']} | "
                    f"{r['r_pixel']:.3f} | {r['dyn_ms'] * 1e3:.1f} | {r['dense_ms'] * 1e3:.1f} | {r['speedup']:.2f} | "
                    f"{r['t_roof_ms'] * 1e3:.1f} | {r['roof_frac']:.2f} |\n")
        f.write(f"| **body** | | 29 | | | **{dyn_tot * 1e3:.0f}** | **{dense_tot * 1e3:.0f}** | "
                f"**{dense_tot / dyn_tot:.2f}** | {roof_tot * 1e3:.0f} | {roof_tot / dyn_tot:.2f} |\n\n"
                f"Body throughput: {out['body_images_per_s_dyn']:.0f} images/s dynamic vs "
                f"{out['body_images_per_s_dense']:.0f} images/s dense (identity blocks only).\n")
        if chain:
            f.write("\n## Chained forward (block k feeds block k+1, own weights/masker per block, one CUDA graph per "
                    "stage)\n\n| stage | blocks | time (us) | us/block | mean r_patch |\n|---|---|---|---|---|\n")
            for c in chain["stages"]:
                f.write(f"| {c['h']}x{c['h']}x{c['c_in']} | {c['blocks']} | {c['ms'] * 1e3:.1f} | "
                        f"{c['ms'] / c['blocks'] * 1e3:.1f} | {c['r_patch_mean']:.3f} |\n")
            f.write(f"| **body** | 29 | **{chain['body_ms'] * 1e3:.0f}** | | |\n\n"
                    f"Chained identity body: {chain['images_per_s']:.0f} images/s.\n")


if __name__ == "__main__":
    main()
