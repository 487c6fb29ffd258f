#!/usr/bin/env python
"""Calibrate and validate the B200 latency predictor (csrc/predictor.cu, NEXT-f4).

  measure (GPU):  python tools/calibrate_predictor.py measure --out profiles/predictor_r2.json
  fit (CPU):      python tools/calibrate_predictor.py fit profiles/predictor_r2.json

measure: every block call of the calibration set (ResNet-50 stage-3 identity
blocks, N = 128, S in {1,2,4,7} x r in {0.25,0.5,0.75,1.0}, both schedules, the
dense block, and the projection (first) blocks of LAS-R101 at N = 64 with r in
{0.25, 0.5, 0.75}) and the validation set (the LAS-R101 identity stages at
N = 256, S_net 4-4-2-1, r in {0.25, 0.5, 0.75}, both schedules and dense),
each with synthetic uniform cell masks drawn by the masker (bias calibrated to
r), timed eagerly with a CUDA-event pair around every kernel (median of 5 after
2 warm-ups); the predictor's per-launch times with every efficiency 1 are stored
beside the measured ones.

fit: per kernel type, eff = median over the calibration launches of
(predicted_at_eff_1 - launch) / (measured - launch); writes
csrc/predictor_b200.inc and reports the block-level error of the calibrated
predictor on the calibration and the (held-out) validation set -- the paper's
Fig. 4 check on B200.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

K_NAMES = ["mask_compact", "conv1_dyn", "conv1_mask", "decide", "decide+gather", "conv23", "conv23_direct", "conv2_dyn",
           "conv3_dyn", "conv1_dense", "conv2_dense", "conv3_dense", "conv23_dense", "subsample", "shortcut", "mask",
           "compact", "conv2_gather"]
ALIASES = {"decide+ids": "decide"}  # the two-launch decide of the same kernel type


def configs():
    cal, val = [], []
    for s in (1, 2, 4, 7):
        for r in (0.25, 0.5, 0.75, 1.0):
            for sched in (0, 1):
                cal.append(dict(n=128, h=28, w=28, c_in=512, c_mid=128, c_out=512, s=s, stride=1, r=r, sched=sched))
    cal.append(dict(n=128, h=28, w=28, c_in=512, c_mid=128, c_out=512, s=4, stride=1, r=1.0, sched=2))
    for (h, c_in, c_mid, stride, s) in [(56, 64, 64, 1, 4), (28, 256, 128, 2, 4), (14, 512, 256, 2, 2),
                                        (7, 1024, 512, 2, 1)]:
        for r in (0.25, 0.5, 0.75):
            cal.append(dict(n=64, h=h, w=h, c_in=c_in, c_mid=c_mid, c_out=4 * c_mid, s=s, stride=stride, r=r, sched=0))
        cal.append(dict(n=64, h=h, w=h, c_in=c_in, c_mid=c_mid, c_out=4 * c_mid, s=s, stride=stride, r=1.0, sched=2))
    for (h, c_mid, s) in [(56, 64, 4), (28, 128, 4), (14, 256, 2), (7, 512, 1)]:
        for r in (0.25, 0.5, 0.75):
            for sched in (0, 1):
                val.append(dict(n=256, h=h, w=h, c_in=4 * c_mid, c_mid=c_mid, c_out=4 * c_mid, s=s, stride=1, r=r,
                                sched=sched))
        val.append(dict(n=256, h=h, w=h, c_in=4 * c_mid, c_mid=c_mid, c_out=4 * c_mid, s=s, stride=1, r=1.0, sched=2))
    return cal, val


def predict(cfg, hw=None):
    import paper_2210_06223_b200 as L

    t, ks = L.predict_latency(cfg["n"], cfg["h"], cfg["w"], cfg["c_in"], cfg["c_mid"], cfg["c_out"], cfg["s"],
                              cfg["r"], cfg["sched"], stride=cfg["stride"], hw=hw)
    return t, ks


def measure_one(cfg, lib):
    import torch

    import synth
    import paper_2210_06223_b200 as L
    from paper_2210_06223_b200 import _lib

    n, h, w, c_in, c_mid, c_out, s, st = (cfg[k] for k in ("n", "h", "w", "c_in", "c_mid", "c_out", "s", "stride"))
    hi, wi = h * st, w * st
    x = synth.make_x(n, hi, wi, c_in, seed=1).cuda()
    proj = st != 1 or c_in != c_out
    if proj:
        wts = {k: v.cuda() for k, v in synth.make_proj_weights(c_in, c_mid, c_out, seed=2).items()}
    else:
        wts = {k: v.cuda() for k, v in synth.make_block_weights(c_in, c_mid, c_out, seed=2).items()}
    wm = synth.make_masker_weights(c_in, seed=3)
    if cfg["sched"] == 2:
        if proj:
            call = lambda: L.proj_block(x, wts, st)  # noqa: E731
        else:
            y = torch.empty_like(x)
            ws = None
            call = lambda: L.dense_block(x, wts, y=y)  # noqa: E731
    elif proj:
        blk = L.ProjDynBlock(n, hi, wi, c_in, c_mid, c_out, st, s, wts, wm)
        blk.calibrate_bias(x, cfg["r"])
        call = lambda: blk.forward(x)  # noqa: E731
    else:
        blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), {k: v.cpu() for k, v in wts.items()}, wm, 0.0,
                         schedule=cfg["sched"])
        blk.calibrate_bias(x, cfg["r"])
        y = x.clone()
        call = lambda: (y.copy_(x), blk.forward(y))  # noqa: E731
    nmax = 16
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nmax)]
    st_ = torch.cuda.current_stream()
    for e in evs:
        e.record(st_)
    arr = (ctypes.c_void_p * len(evs))(*[e.cuda_event for e in evs])
    runs = []
    names = None
    for rep in range(7):
        lib.lasnet_set_kernel_events(arr, nmax)
        call()
        cnt = int(lib.lasnet_kernel_event_count())
        names = [ALIASES.get(lib.lasnet_kernel_event_name(i).decode(), lib.lasnet_kernel_event_name(i).decode())
                 for i in range(cnt)]
        lib.lasnet_set_kernel_events(None, 0)
        torch.cuda.synchronize()
        if rep >= 2:
            runs.append([evs[2 * i].elapsed_time(evs[2 * i + 1]) * 1e3 for i in range(cnt)])
    us = [statistics.median(v) for v in zip(*runs)]
    keep = [i for i, nm in enumerate(names) if nm in K_NAMES]  # add_bias (a 1 K-element add) is not modelled
    names, us = [names[i] for i in keep], [us[i] for i in keep]
    r_meas = float(blk.count.item()) / blk.ncells if cfg["sched"] != 2 else 1.0
    return names, us, r_meas


def cmd_measure(args):
    import torch

    from paper_2210_06223_b200 import _lib, build

    build.build()
    lib = _lib.load()
    cal, val = configs()
    out = []
    for split, cs in (("cal", cal), ("val", val)):
        for cfg in cs:
            names, us, r_meas = measure_one(cfg, lib)
            cfg2 = dict(cfg, r=r_meas)
            hw1 = unit_hw()
            _, ks = predict(cfg2, hw1)
            out.append(dict(split=split, cfg=cfg, r_meas=r_meas, names=names, measured_us=us,
                            pred_eff1=[[k, t] for k, t in ks]))
            print(split, cfg, [f"{a}:{b:.1f}" for a, b in zip(names, us)], flush=True)
            torch.cuda.empty_cache()
    json.dump(out, open(args.out, "w"), indent=1)


def unit_hw():
    import paper_2210_06223_b200 as L

    hw = L.hw_b200()
    for k in range(len(K_NAMES)):  # the bare bound: efficiency 1, no fixed cost (the fit's model)
        hw.eff[k] = 1.0
        hw.t0_us[k] = 0.0
    return hw


def cmd_repredict(args):
    """Recompute the stored predictions at efficiency 1 (pred_eff1) for the recorded
    configurations (host-only: the predictor runs on the CPU)."""
    data = json.load(open(args.data))
    for rec in data:
        _, ks = predict(dict(rec["cfg"], r=rec["r_meas"]), unit_hw())
        rec["pred_eff1"] = [[k, t] for k, t in ks]
    json.dump(data, open(args.data, "w"), indent=1)


def cmd_fit(args):
    """Per kernel type: (measured - launch) = t0 + (predicted at eff 1 - launch) / eff, a
    relative-error weighted least-squares fit (t0 >= 0, 0 < eff <= 1) on the calibration
    records -- every activation rate except the held-out r = 0.5 -- then the block-level
    error on both splits (validation: r = 0.5 at every shape, the shapes' r never seen)."""
    import numpy as np

    import paper_2210_06223_b200 as L

    data = json.load(open(args.data))
    launch = L.hw_b200().launch_us

    def split(rec):
        return "val" if abs(rec["cfg"]["r"] - 0.5) < 1e-9 else "cal"

    pts = {k: [] for k in K_NAMES}
    for rec in data:
        pk = [k for k, _ in rec["pred_eff1"]]
        if pk != rec["names"]:
            print("plan mismatch", rec["cfg"], pk, rec["names"])
            continue
        if split(rec) != "cal":
            continue
        for (k, tp), tm in zip(rec["pred_eff1"], rec["measured_us"]):
            pts[k].append((max(tp - launch, 0.0), max(tm - launch, 0.0)))
    eff, t0 = {}, {}
    for k, v in pts.items():
        if not v:
            eff[k], t0[k] = 1.0, 0.0
            continue
        a = np.array(v)
        wgt = 1.0 / np.maximum(a[:, 1], 1.0)
        if np.ptp(a[:, 0]) > 1e-6 * max(a[:, 0].max(), 1e-9):
            A = np.c_[np.ones(len(a)), a[:, 0]]
            (c0, c1), *_ = np.linalg.lstsq(A * wgt[:, None], a[:, 1] * wgt, rcond=None)
        else:
            c0, c1 = 0.0, 0.0
        if c0 < 0 or c1 <= 1.0:  # t0 >= 0, eff <= 1: refit the one-parameter forms
            c0 = max(0.0, float(np.median(a[:, 1] - a[:, 0])))
            c1 = 1.0
            if np.median(a[:, 1]) > 0 and np.median(a[:, 0]) > 0:
                s1 = float(np.median(a[:, 1] / np.maximum(a[:, 0], 1e-9)))
                e1 = np.mean(np.abs(a[:, 0] * s1 - a[:, 1]) / np.maximum(a[:, 1], 1))
                e0 = np.mean(np.abs(a[:, 0] + c0 - a[:, 1]) / np.maximum(a[:, 1], 1))
                if s1 >= 1.0 and e1 < e0:
                    c0, c1 = 0.0, s1
        eff[k], t0[k] = 1.0 / c1, float(c0)
    lines = ["// Calibrated per-kernel-type efficiencies and fixed costs of the B200 latency predictor",
             "// (predictor.cu): relative-error weighted least squares of (measured - launch) = t0 +",
             "// (predicted at eff 1 - launch) / eff over the calibration launches (r != 0.5),",
             f"// written by tools/calibrate_predictor.py fit {os.path.relpath(args.data, ROOT)}"]
    for i, k in enumerate(K_NAMES):
        lines.append(f"hw->eff[{i}] = {eff[k]:.4f};  hw->t0_us[{i}] = {t0[k]:.3f};  // {k} ({len(pts[k])} launches)")
    open(os.path.join(ROOT, "paper_2210_06223_b200", "csrc", "predictor_b200.inc"), "w").write("\n".join(lines) + "\n")
    hw = L.hw_b200()
    for i, k in enumerate(K_NAMES):
        hw.eff[i] = eff[k]
        hw.t0_us[i] = t0[k]
    report = {"eff": eff, "t0_us": t0, "blocks": []}
    errs = {"cal": [], "val": []}
    for rec in data:
        cfg = dict(rec["cfg"], r=rec["r_meas"])
        t, _ = predict(cfg, hw)
        m = sum(rec["measured_us"])
        sp = split(rec)
        errs[sp].append(abs(t - m) / m)
        report["blocks"].append(dict(split=sp, cfg=rec["cfg"], r_meas=rec["r_meas"], measured_us=round(m, 2),
                                     predicted_us=round(t, 2), rel_err=round((t - m) / m, 4)))
    for sp in ("cal", "val"):
        e = errs[sp]
        report[f"{sp}_mean_abs_rel_err"] = round(statistics.fmean(e), 4) if e else None
        report[f"{sp}_max_abs_rel_err"] = round(max(e), 4) if e else None
        print(sp, "blocks", len(e), "mean |err|", report[f"{sp}_mean_abs_rel_err"], "max", report[f"{sp}_max_abs_rel_err"])
    out = args.report or args.data.replace(".json", "_fit.json")
    json.dump(report, open(out, "w"), indent=1)
    print("eff", {k: round(v, 3) for k, v in eff.items()})
    print("t0", {k: round(v, 1) for k, v in t0.items()})


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    m = sub.add_parser("measure")
    m.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "predictor_r2.json"))
    f = sub.add_parser("fit")
    f.add_argument("data")
    f.add_argument("--report", default=None)
    rp = sub.add_parser("repredict")
    rp.add_argument("data")
    args = ap.parse_args()
    {"measure": cmd_measure, "fit": cmd_fit, "repredict": cmd_repredict}[args.cmd](args)


if __name__ == "__main__":
    main()
