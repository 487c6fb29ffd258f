"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws random
tensors and random cell masks.  Both the tests
(oracle vs CUDA parity) and bench.py draw their inputs from here, so the two
sides see the same bytes.

Recipe (SURVEY.md 8(d) / DESIGN.md):
  x      = ReLU(N(0,1)) stored NHWC, bf16 (or fp32 for config 1)   -- post-ReLU block input
  W1, W2 = He-normal (std sqrt(2/fan_in)); W3 = He-normal * 0.1 (gamma = 0.1)
  b1..b3 = N(0, 0.05^2), fp32 (BN folded)
  wm     = N(0, 1/c_in) fp32  -- reduced masker weight W_0 - W_1
  cell masks: exactly k = floor(r*G + 0.5) active cells per image from a seeded
  permutation (uniform family) or the top-k of 3x3-box-smoothed noise
  (clustered family; real masks follow objects).
"""
from __future__ import annotations

import numpy as np
import torch


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def _dt(dtype: str):
    return {"bf16": torch.bfloat16, "f32": torch.float32}[dtype]


def make_x(n: int, h: int, w: int, c: int, seed: int = 0, dtype: str = "bf16",
           relu: bool = True) -> torch.Tensor:
    """Block input, NHWC, on the CPU. relu=False gives signed inputs (R5 pin)."""
    t = torch.randn((n, h, w, c), generator=_gen(seed), dtype=torch.float32)
    if relu:
        t = torch.clamp_min(t, 0.0)
    return t.to(_dt(dtype)).contiguous()


def make_block_weights(c_in: int, c_mid: int, c_out: int, seed: int = 1,
                       dtype: str = "bf16", w3_gamma: float = 0.1,
                       bias_std: float = 0.05) -> dict:
    """BN-folded bottleneck weights: w1 [c_mid][c_in], w2 [c_mid][3][3][c_mid] (OHWI),
    w3 [c_out][c_mid]; biases fp32."""
    g = _gen(seed)
    w1 = torch.randn((c_mid, c_in), generator=g) * (2.0 / c_in) ** 0.5
    w2 = torch.randn((c_mid, 3, 3, c_mid), generator=g) * (2.0 / (9 * c_mid)) ** 0.5
    w3 = torch.randn((c_out, c_mid), generator=g) * (2.0 / c_mid) ** 0.5 * w3_gamma
    b1 = torch.randn((c_mid,), generator=g) * bias_std
    b2 = torch.randn((c_mid,), generator=g) * bias_std
    b3 = torch.randn((c_out,), generator=g) * bias_std
    dt = _dt(dtype)
    return {
        "w1": w1.to(dt).contiguous(), "b1": b1.float().contiguous(),
        "w2": w2.to(dt).contiguous(), "b2": b2.float().contiguous(),
        "w3": w3.to(dt).contiguous(), "b3": b3.float().contiguous(),
    }


def make_proj_weights(c_in: int, c_mid: int, c_out: int, seed: int = 1, dtype: str = "bf16") -> dict:
    """Bottleneck weights plus the projection shortcut wd [c_out][c_in] (He-normal)
    and bd [c_out] fp32, for a stage's first block."""
    wts = make_block_weights(c_in, c_mid, c_out, seed=seed, dtype=dtype, w3_gamma=1.0)
    g = _gen(seed + 7919)
    wts["wd"] = (torch.randn((c_out, c_in), generator=g) * (2.0 / c_in) ** 0.5).to(_dt(dtype)).contiguous()
    wts["bd"] = (torch.randn((c_out,), generator=g) * 0.05).float().contiguous()
    return wts


def make_lasnet_weights(depths=(3, 4, 23, 3), widths=(64, 128, 256, 512), classes: int = 1000, seed: int = 11,
                        dtype: str = "bf16") -> dict:
    """Random-init weights of a LAS-ResNet (BN folded): stem [64][7][7][8] (channels
    3..7 zero), per stage a projection block and depth-1 identity blocks (with a
    masker weight each), classifier [classes][4*widths[-1]]."""
    g = _gen(seed)
    dt = _dt(dtype)
    stem = torch.randn((64, 7, 7, 8), generator=g) * (2.0 / (7 * 7 * 3)) ** 0.5
    stem[..., 3:] = 0.0
    w = {"stem_w": stem.to(dt).contiguous(), "stem_b": (torch.randn((64,), generator=g) * 0.05).float().contiguous()}
    c_in = 64
    for si, (depth, width) in enumerate(zip(depths, widths)):
        c_out = 4 * width
        w[f"s{si}_proj"] = make_proj_weights(c_in, width, c_out, seed=seed * 1000 + 100 * si, dtype=dtype)
        # masker of the (dynamic) first block: it pools the block INPUT (c_in channels)
        w[f"s{si}_proj"]["wm"] = make_masker_weights(c_in, seed=seed * 1000 + 100 * si + 99)
        for b in range(1, depth):
            wb = make_block_weights(c_out, width, c_out, seed=seed * 1000 + 100 * si + 2 * b, dtype=dtype)
            wb["wm"] = make_masker_weights(c_out, seed=seed * 1000 + 100 * si + 2 * b + 1)
            w[f"s{si}_b{b}"] = wb
        c_in = c_out
    w["fc_w"] = (torch.randn((classes, c_in), generator=g) * (1.0 / c_in) ** 0.5).to(dt).contiguous()
    w["fc_b"] = torch.zeros((classes,)).float().contiguous()
    return w


def make_image_batch(n: int, hw=224, seed: int = 0, dtype: str = "bf16") -> torch.Tensor:
    """ImageNet/COCO-normalised-like input N(0,1) with 3 channels, in the stem's
    padded layout [n][H][W + 8][8] (channels 3..7 and 4 pixels left/right zero);
    hw is H = W or (H, W)."""
    H, W = (hw, hw) if isinstance(hw, int) else tuple(hw)
    x = torch.zeros((n, H, W + 8, 8), dtype=torch.float32)
    x[:, :, 4:4 + W, :3] = torch.randn((n, H, W, 3), generator=_gen(seed))
    return x.to(_dt(dtype)).contiguous()


def make_masker_weights(c_in: int, seed: int = 3) -> torch.Tensor:
    """Reduced masker weight w = W_0 - W_1, fp32 [c_in]."""
    return (torch.randn((c_in,), generator=_gen(seed)) * (1.0 / c_in) ** 0.5).float().contiguous()


def make_masker_weights_2ch(c_in: int, seed: int = 3):
    """Two-channel masker weights W [2][c_in] and bias [2] (paper form)."""
    g = _gen(seed)
    W = (torch.randn((2, c_in), generator=g) * (1.0 / c_in) ** 0.5).float()
    b = (torch.randn((2,), generator=g) * 0.05).float()
    return W.contiguous(), b.contiguous()


def active_cells(r: float, cells: int) -> int:
    """k = floor(r*G + 0.5) (R16)."""
    return int(np.floor(r * cells + 0.5))


def make_cell_mask(n: int, gh: int, gw: int, r: float, seed: int = 2,
                   family: str = "uniform") -> np.ndarray:
    """uint8 [n][gh][gw] with exactly active_cells(r, gh*gw) ones per image."""
    rng = np.random.default_rng(int(seed))
    G = gh * gw
    k = active_cells(r, G)
    m = np.zeros((n, G), np.uint8)
    for i in range(n):
        if family == "uniform":
            sel = rng.permutation(G)[:k]
        elif family == "clustered":
            noise = rng.standard_normal((gh + 2, gw + 2))
            sm = np.zeros((gh, gw))
            for dy in range(3):
                for dx in range(3):
                    sm += noise[dy:dy + gh, dx:dx + gw]
            sel = np.argsort(-sm.reshape(-1), kind="stable")[:k]
        else:
            raise ValueError(family)
        m[i, sel] = 1
    return m.reshape(n, gh, gw)


def to_f64(t: torch.Tensor) -> np.ndarray:
    """Exact float64 copy of a bf16/fp32 tensor (for the oracle)."""
    return t.detach().to("cpu").to(torch.float64).numpy()


def weights_f64(wts: dict) -> dict:
    return {k: to_f64(v) for k, v in wts.items()}


def weights_f64_nested(wts: dict) -> dict:
    """weights_f64 over a nested weight dict (make_lasnet_weights)."""
    return {k: weights_f64_nested(v) if isinstance(v, dict) else to_f64(v) for k, v in wts.items()}


def lasnet_oracle_biases(weights: dict, seed: int = 5000, depths=(3, 4, 23, 3), s_net=(4, 4, 2, 1)) -> dict:
    """Network metadata for oracle runs without a GPU network (bench.py's reference
    arm): depths, S_net and an empty bias table that oracle.lasnet_forward fills by
    calibrating on its own first forward (it is the oracle that calibrates; this
    module only states the configuration)."""
    return {"depths": tuple(depths), "s_net": tuple(s_net), "bm": {}, "calibrate_seed": int(seed)}


# ----------------------------------------------------------- LAS-RegNetY-800MF --
# torchvision regnet_y_800mf: stem 32; stages (width, depth) = (64, 1), (144, 3),
# (320, 8), (784, 2); group width 16; bottleneck ratio 1; SE ratio 0.25 of the
# block INPUT width; every stage's first block has stride 2 (projection shortcut).
REGNET_Y_800MF = dict(stem=32, widths=(64, 144, 320, 784), depths=(1, 3, 8, 2), group_width=16, se_ratio=0.25)


def pad64(c: int) -> int:
    """Channel count rounded up to the tensor-core K-block of 64 (zero channels)."""
    return -(-c // 64) * 64


def _padded(real: torch.Tensor, shape) -> torch.Tensor:
    out = torch.zeros(shape, dtype=real.dtype)
    out[tuple(slice(0, s) for s in real.shape)] = real
    return out


def make_regnet_block_weights(c_in: int, w_out: int, w_se: int, proj: bool, seed: int, dtype: str = "bf16",
                              group_width: int = 16) -> dict:
    """Y-block weights (BN folded) at REAL widths c_in -> w_out (bottleneck = w_out),
    stored zero-padded to pad64 widths: wa [wb][cin], wb [wb][3][3][16] (grouped),
    se_w1 [w_se][wb], se_w2 [wb][w_se], wc [wout][wb], (proj) wd [wout][cin]; fp32
    biases; masker weight wm [cin] for the dynamic identity blocks."""
    g = _gen(seed)
    dt = _dt(dtype)
    ci, co = pad64(c_in), pad64(w_out)
    wa = torch.randn((w_out, c_in), generator=g) * (2.0 / c_in) ** 0.5
    wb = torch.randn((w_out, 3, 3, group_width), generator=g) * (2.0 / (9 * group_width)) ** 0.5
    s1 = torch.randn((w_se, w_out), generator=g) * (1.0 / w_out) ** 0.5
    s2 = torch.randn((w_out, w_se), generator=g) * (1.0 / w_se) ** 0.5
    wc = torch.randn((w_out, w_out), generator=g) * (2.0 / w_out) ** 0.5 * (1.0 if proj else 0.1)
    b = {k: torch.randn((n,), generator=g) * 0.05 for k, n in (("ba", w_out), ("bb", w_out), ("bc", w_out),
                                                                ("se_b1", w_se), ("se_b2", w_out))}
    out = {
        "wa": _padded(wa, (co, ci)).to(dt).contiguous(), "ba": _padded(b["ba"], (co,)).float().contiguous(),
        "wb": _padded(wb, (co, 3, 3, group_width)).to(dt).contiguous(), "bb": _padded(b["bb"], (co,)).float().contiguous(),
        "se_w1": _padded(s1, (w_se, co)).float().contiguous(), "se_b1": b["se_b1"].float().contiguous(),
        "se_w2": _padded(s2, (co, w_se)).float().contiguous(), "se_b2": _padded(b["se_b2"], (co,)).float().contiguous(),
        "wc": _padded(wc, (co, co)).to(dt).contiguous(), "bc": _padded(b["bc"], (co,)).float().contiguous(),
    }
    if proj:
        wd = torch.randn((w_out, c_in), generator=g) * (2.0 / c_in) ** 0.5
        out["wd"] = _padded(wd, (co, ci)).to(dt).contiguous()
        out["bd"] = _padded(torch.randn((w_out,), generator=g) * 0.05, (co,)).float().contiguous()
    else:
        out["wm"] = _padded((torch.randn((c_in,), generator=g) * (1.0 / c_in) ** 0.5), (ci,)).float().contiguous()
    return out


def make_regnet_weights(cfg=None, classes: int = 1000, seed: int = 21, dtype: str = "bf16") -> dict:
    """Random-init LAS-RegNetY weights (default RegNetY-800MF) at pad64 widths: stem
    [64][3][3][8] (32 real output channels, 3 real input channels), per stage block
    0 (stride 2, projection) and the identity blocks, classifier [classes][pad64(784)]."""
    cfg = cfg or REGNET_Y_800MF
    g = _gen(seed)
    dt = _dt(dtype)
    stem = torch.randn((cfg["stem"], 3, 3, 3), generator=g) * (2.0 / 27) ** 0.5
    w = {"stem_w": _padded(stem, (pad64(cfg["stem"]), 3, 3, 8)).to(dt).contiguous(),
         "stem_b": _padded(torch.randn((cfg["stem"],), generator=g) * 0.05, (pad64(cfg["stem"]),)).float().contiguous()}
    c_in = cfg["stem"]
    for si, (width, depth) in enumerate(zip(cfg["widths"], cfg["depths"])):
        for b in range(depth):
            w_in = c_in if b == 0 else width
            w_se = int(round(cfg["se_ratio"] * w_in))
            w[f"s{si}_b{b}"] = make_regnet_block_weights(w_in, width, w_se, proj=(b == 0),
                                                         seed=seed * 1000 + 100 * si + b, dtype=dtype,
                                                         group_width=cfg["group_width"])
        c_in = width
    fc = torch.randn((classes, c_in), generator=g) * (1.0 / c_in) ** 0.5
    w["fc_w"] = _padded(fc, (classes, pad64(c_in))).to(dt).contiguous()
    w["fc_b"] = torch.zeros((classes,)).float().contiguous()
    return w
