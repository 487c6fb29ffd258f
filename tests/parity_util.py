"""Shared helpers for the GPU parity tests (oracle vs CUDA path)."""
import numpy as np
import torch

import oracle
import synth

BF16_TOL = 2e-2   # north_star: max-abs-rel 2e-2 for bf16 with fp32 accumulation
F32_TOL = 1e-5    # north_star: 1e-5 for the fp32 path


def max_abs_rel(got: np.ndarray, want: np.ndarray) -> float:
    """err = max|g - o| / max(max|o|, 1e-30) per tensor (reading R14)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    if want.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want)) / max(float(np.max(np.abs(want))), 1e-30))


def margin_bias(logits0: np.ndarray, r: float) -> float:
    """Masker bias (fp32) placing ~r of the cells above threshold, midway between
    two neighbouring oracle logits so every cell keeps a margin."""
    lg = np.sort(logits0.reshape(-1))
    G = lg.size
    k = int(round(r * G))
    if k <= 0:
        b = -(lg[-1] + 1.0)
    elif k >= G:
        b = -(lg[0] - 1.0)
    else:
        b = -0.5 * (lg[G - k - 1] + lg[G - k])
    return float(np.float32(b))


def make_case(n, h, w, c_in, c_mid, s, seed=0, dtype="bf16", relu=True):
    x = synth.make_x(n, h, w, c_in, seed=seed, dtype=dtype, relu=relu)
    wts = synth.make_block_weights(c_in, c_mid, c_in, seed=seed + 1, dtype=dtype)
    wm = synth.make_masker_weights(c_in, seed=seed + 2)
    return x, wts, wm


def to_dev(wts):
    return {k: v.cuda().contiguous() for k, v in wts.items()}


def rmode(dtype):
    return oracle.ROUND_BF16 if dtype == "bf16" else oracle.ROUND_F32


def tol(dtype):
    return BF16_TOL if dtype == "bf16" else F32_TOL
