"""The B200 latency predictor G(H, P, S, r) (csrc/predictor.cu; App. A
P:483-523).  Host-side, pure: runs on CPU (-m "not gpu").

The committed calibration (csrc/predictor_b200.inc, fitted by
tools/calibrate_predictor.py on profiles/predictor_r2.json, B200 per-kernel event
timings) is checked against the same measurements: the block latencies at the
held-out activation rate r = 0.5 (never used by the fit) within 15 % on average,
the paper's Fig. 4 check (predicted vs measured latency across r) on B200."""
import json
import os
import statistics

import pytest

import paper_2210_06223_b200 as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pred(n, h, c, cm, s, r, sched, stride=1, c_out=None):
    return L.predict_latency(n, h, h, c, cm, c_out or c, s, r, sched, stride=stride)


def test_dynamic_latency_grows_with_r_and_dense_does_not():
    for sched in (L.SCHED_SEPARATE, L.SCHED_FUSED):
        ts = [pred(128, 28, 512, 128, 4, r, sched)[0] for r in (0.0, 0.25, 0.5, 0.75, 1.0)]
        assert all(b >= a for a, b in zip(ts, ts[1:])), ts
    td = [pred(128, 28, 512, 128, 4, r, L.SCHED_DENSE)[0] for r in (0.1, 0.9)]
    assert td[0] == td[1]


def test_plan_lists_the_library_launches():
    names = lambda r: [k for k, _ in r[1]]  # noqa: E731
    assert names(pred(128, 28, 512, 128, 4, 0.5, L.SCHED_FUSED)) == ["conv1_mask", "decide", "conv23_direct"]
    assert names(pred(128, 28, 512, 128, 2, 0.5, L.SCHED_FUSED)) == ["conv1_mask", "decide+gather", "conv23"]
    assert names(pred(128, 28, 512, 128, 4, 0.5, L.SCHED_SEPARATE)) == ["mask_compact", "conv1_dyn", "conv23"]
    assert names(pred(256, 14, 1024, 256, 2, 0.5, L.SCHED_FUSED)) == ["conv1_mask", "decide", "conv2_gather",
                                                                      "conv3_dyn"]
    assert names(pred(64, 28, 256, 128, 4, 0.5, L.SCHED_SEPARATE, stride=2, c_out=512)) == [
        "mask", "compact", "shortcut", "conv1_dyn", "conv23"]
    assert names(pred(128, 28, 512, 128, 4, 1.0, L.SCHED_DENSE)) == ["conv1_dense", "conv23_dense"]


def test_invalid_arguments():
    with pytest.raises(ValueError):
        pred(128, 28, 512, 128, 4, 1.5, L.SCHED_FUSED)
    with pytest.raises(ValueError):  # first blocks: masker-separate schedule only
        pred(64, 28, 256, 128, 4, 0.5, L.SCHED_FUSED, stride=2, c_out=512)


def test_hardware_model_scales():
    """Halving the HBM bandwidth slows an HBM-bound dynamic block; the tensor peak
    matters little to it (the paper's hardware-model inputs)."""
    base = pred(128, 28, 512, 128, 4, 0.5, L.SCHED_FUSED)[0]
    hw = L.hw_b200()
    hw.hbm_gbs /= 2
    slow = L.predict_latency(128, 28, 28, 512, 128, 512, 4, 0.5, L.SCHED_FUSED, hw=hw)[0]
    assert slow > 1.3 * base


def test_calibration_reproduces_held_out_measurements():
    data = json.load(open(os.path.join(ROOT, "profiles", "predictor_r2.json")))
    errs = {"cal": [], "val": []}
    for rec in data:
        c = rec["cfg"]
        t, ks = L.predict_latency(c["n"], c["h"], c["w"], c["c_in"], c["c_mid"], c["c_out"], c["s"], rec["r_meas"],
                                  c["sched"], stride=c["stride"])
        assert [k for k, _ in ks] == rec["names"], (c, ks, rec["names"])
        m = sum(rec["measured_us"])
        errs["val" if abs(c["r"] - 0.5) < 1e-9 else "cal"].append(abs(t - m) / m)
    assert len(errs["val"]) >= 20
    assert statistics.fmean(errs["val"]) < 0.15, statistics.fmean(errs["val"])
    assert statistics.fmean(errs["cal"]) < 0.15


def test_schedule_choice_follows_the_predictor():
    d = (128, 28, 28, 512, 128, 512, 4)
    for r in (0.1, 0.5, 0.9):
        ts = L.predict_latency(*d, r, L.SCHED_SEPARATE)[0]
        tf = L.predict_latency(*d, r, L.SCHED_FUSED)[0]
        assert L.choose_schedule(*d, r) == (L.SCHED_FUSED if tf < ts else L.SCHED_SEPARATE)
