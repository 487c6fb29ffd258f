"""CPU oracle for the LASNet dynamic residual block -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2210_06223_b200`` never imports it and shares no code with it.

This module is a thin ctypes binding over ``lasnet_oracle.c`` (fp64, plain loops,
each function citing the PAPER.md passage it follows).  All tensors cross the
boundary as C-contiguous float64 numpy arrays holding the *exact* values of the
bf16/fp32 tensors the GPU sees (bf16 -> fp64 is exact).

Parity status per function:
  masker_2ch, masker, upsample, compact, static_block, dyn_block_def,
  dyn_block_literal, block_pixel, round_bf16, proj_block, stem, maxpool, head -- all pinned by tests in
  tests/test_oracle_pins.py (library conv2d in fp64, exact rationals, closed
  forms, brute force, textbook routines).  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lasnet_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ROUND_NONE, ROUND_F32, ROUND_BF16 = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (-O2, OpenMP over patches)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        D = ctypes.POINTER(ctypes.c_double)
        U8 = ctypes.POINTER(ctypes.c_uint8)
        I32 = ctypes.POINTER(ctypes.c_int32)
        i = ctypes.c_int
        _lib.oracle_round_bf16.restype = ctypes.c_double
        _lib.oracle_round_bf16.argtypes = [ctypes.c_double]
        _lib.oracle_round_f32.restype = ctypes.c_double
        _lib.oracle_round_f32.argtypes = [ctypes.c_double]
        _lib.oracle_masker_2ch.argtypes = [D, i, i, i, i, i, D, D, U8, D, D]
        _lib.oracle_masker.argtypes = [D, i, i, i, i, i, D, ctypes.c_double, U8, D]
        _lib.oracle_upsample.argtypes = [U8, i, i, i, i, U8]
        _lib.oracle_compact.restype = ctypes.c_int
        _lib.oracle_compact.argtypes = [U8, i, I32]
        _lib.oracle_static_block.argtypes = [D, i, i, i, i, i, i, D, D, D, D, D, D, i, D, D, D]
        _lib.oracle_dyn_block_def.argtypes = [D, i, i, i, i, i, i, D, D, D, D, D, D, U8, i, i, D]
        _lib.oracle_dyn_block_literal.argtypes = [D, i, i, i, i, i, i, D, D, D, D, D, D, I32, i, i, i, D]
        _lib.oracle_block_pixel.restype = ctypes.c_int
        _lib.oracle_block_pixel.argtypes = [D, i, i, i, i, i, D, D, D, D, D, D, U8, i, i, i, i, i, D]
        _lib.oracle_proj_dyn_literal.argtypes = [D, i, i, i, i, i, i, D, D, D, D, D, D, D, D, I32, i, i, i, i, D]
        _lib.oracle_num_threads.restype = ctypes.c_int
        _lib.oracle_set_threads.argtypes = [i]
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def grid(h: int, w: int, s: int):
    """Cell grid of the coarse mask (R7: ceil, clipped edge patches)."""
    return -(-h // s), -(-w // s)


def round_bf16(v: float) -> float:
    return _load().oracle_round_bf16(float(v))


def round_f32(v: float) -> float:
    return _load().oracle_round_f32(float(v))


def masker_2ch(x, Wm, bm, s):
    """Paper-form masker: avgpool -> 1x1 conv (2 ch) -> argmax."""
    lib = _load()
    x, xp = _d(x)
    n, h, w, c = x.shape
    gh, gw = grid(h, w, s)
    Wm, wp = _d(Wm)
    bm, bp = _d(bm)
    mask = np.zeros((n, gh, gw), np.uint8)
    z0 = np.zeros((n, gh, gw))
    z1 = np.zeros((n, gh, gw))
    _, mp = _u8(mask)
    _, z0p = _d(z0)
    _, z1p = _d(z1)
    lib.oracle_masker_2ch(xp, n, h, w, c, s, wp, bp, mp, z0p, z1p)
    return mask, z0, z1


def masker(x, wm, bm, s):
    """Reduced masker (App. B): logit = w . avgpool(x) + b, mask = logit > 0."""
    lib = _load()
    x, xp = _d(x)
    n, h, w, c = x.shape
    gh, gw = grid(h, w, s)
    wm, wp = _d(wm)
    mask = np.zeros((n, gh, gw), np.uint8)
    logit = np.zeros((n, gh, gw))
    _, mp = _u8(mask)
    _, lp = _d(logit)
    lib.oracle_masker(xp, n, h, w, c, s, wp, float(bm), mp, lp)
    return mask, logit


def upsample(mask_cells, h, w, s):
    lib = _load()
    mc, mcp = _u8(mask_cells)
    n = mc.shape[0]
    m = np.zeros((n, h, w), np.uint8)
    _, mp = _u8(m)
    lib.oracle_upsample(mcp, n, h, w, s, mp)
    return m


def compact(mask_cells):
    lib = _load()
    m, mp = _u8(np.asarray(mask_cells).reshape(-1))
    idx = np.zeros(max(m.size, 1), np.int32)
    _, ip = _i32(idx)
    count = lib.oracle_compact(mp, m.size, ip)
    return idx[:count].copy(), count


def _weights(wts):
    out = []
    keep = []
    for k in ("w1", "b1", "w2", "b2", "w3", "b3"):
        a, p = _d(wts[k])
        keep.append(a)
        out.append(p)
    return keep, out


def static_block(x, wts, rmode=ROUND_BF16, return_intermediates=False):
    """Dense bottleneck: h1, h2 with zero padding, y = ReLU(x + conv3(h2))."""
    lib = _load()
    x, xp = _d(x)
    n, h, w, c_in = x.shape
    c_mid = wts["w1"].shape[0]
    c_out = wts["w3"].shape[0]
    keep, wp = _weights(wts)
    y = np.zeros((n, h, w, c_out))
    h1 = np.zeros((n, h, w, c_mid))
    h2 = np.zeros((n, h, w, c_mid))
    _, yp = _d(y)
    _, h1p = _d(h1)
    _, h2p = _d(h2)
    lib.oracle_static_block(xp, n, h, w, c_in, c_mid, c_out, *wp, rmode, yp, h1p, h2p)
    if return_intermediates:
        return y, h1, h2
    return y


def dyn_block_def(x, wts, mask_cells, s, rmode=ROUND_BF16):
    """Definition mode: y = M ? static_block(x) : x."""
    lib = _load()
    x, xp = _d(x)
    n, h, w, c_in = x.shape
    c_mid = wts["w1"].shape[0]
    c_out = wts["w3"].shape[0]
    keep, wp = _weights(wts)
    mc, mcp = _u8(mask_cells)
    y = np.zeros((n, h, w, c_out))
    _, yp = _d(y)
    lib.oracle_dyn_block_def(xp, n, h, w, c_in, c_mid, c_out, *wp, mcp, s, rmode, yp)
    return y


def dyn_block_literal(x, wts, idx, s, rmode=ROUND_BF16, threads: int | None = None):
    """Literal mode: gather halo -> conv1 -> conv2 -> conv3 + residual -> scatter."""
    lib = _load()
    if threads is not None:
        lib.oracle_set_threads(int(threads))
    x, xp = _d(x)
    n, h, w, c_in = x.shape
    c_mid = wts["w1"].shape[0]
    c_out = wts["w3"].shape[0]
    keep, wp = _weights(wts)
    idx = np.asarray(idx, dtype=np.int32).reshape(-1)
    count = int(idx.size)
    idx, ip = _i32(idx if count else np.zeros(1, np.int32))
    y = np.zeros((n, h, w, c_out))
    _, yp = _d(y)
    lib.oracle_dyn_block_literal(xp, n, h, w, c_in, c_mid, c_out, *wp, ip, count, s, rmode, yp)
    return y


def block_pixel(x, wts, mask_cells, s, n, yy, xx, rmode=ROUND_BF16):
    """One output pixel of the block computed on its own (sampled full-size checks)."""
    lib = _load()
    x, xp = _d(x)
    _, h, w, c_in = x.shape
    c_mid = wts["w1"].shape[0]
    c_out = wts["w3"].shape[0]
    keep, wp = _weights(wts)
    mc, mcp = _u8(mask_cells)
    out = np.zeros(c_out)
    _, op = _d(out)
    active = lib.oracle_block_pixel(xp, h, w, c_in, c_mid, c_out, *wp, mcp, s, rmode,
                                    int(n), int(yy), int(xx), op)
    return out, bool(active)


def _round_array(a, rmode):
    if rmode == ROUND_NONE:
        return a
    f = round_bf16 if rmode == ROUND_BF16 else round_f32
    return np.vectorize(f, otypes=[np.float64])(a)


def proj_block(x, wts, stride, rmode=ROUND_BF16, round_shortcut=False):
    """Static projection (first) block of a ResNet stage, BN folded (the
    stride-s first block whose shortcut LASNet keeps dense), written out in
    fp64 numpy with the storage roundings of the stored tensors (h1, h2, y; the
    shortcut x_s Wd^T + bd is an unstored term of y, reading R21):
      h1 = rnd(ReLU(x W1^T + b1))                         at the input resolution
      h2 = rnd(ReLU(sum_{dy,dx} h1p[s*oy+dy, s*ox+dx] W2[:,dy,dx,:]^T + b2)), h1p = h1 zero-padded by 1
      y  = rnd(ReLU(h2 W3^T + b3 + x[:, ::s, ::s] Wd^T + bd))
    x [n][H][W][c_in] (H, W multiples of s) -> y [n][H/s][W/s][c_out]."""
    x = np.asarray(x, np.float64)
    n, hi, wi, c_in = x.shape
    s = int(stride)
    ho, wo = hi // s, wi // s
    w1, b1 = np.asarray(wts["w1"], np.float64), np.asarray(wts["b1"], np.float64)
    w2, b2 = np.asarray(wts["w2"], np.float64), np.asarray(wts["b2"], np.float64)
    w3, b3 = np.asarray(wts["w3"], np.float64), np.asarray(wts["b3"], np.float64)
    wd, bd = np.asarray(wts["wd"], np.float64), np.asarray(wts["bd"], np.float64)
    h1 = _round_array(np.maximum(x @ w1.T + b1, 0.0), rmode)
    h1p = np.zeros((n, hi + 2, wi + 2, h1.shape[-1]))
    h1p[:, 1:-1, 1:-1] = h1
    acc = np.zeros((n, ho, wo, w2.shape[0]))
    for dy in range(3):
        for dx in range(3):
            win = h1p[:, dy:dy + s * ho:s, dx:dx + s * wo:s, :]
            acc += win @ w2[:, dy, dx, :].T
    h2 = _round_array(np.maximum(acc + b2, 0.0), rmode)
    ds = x[:, ::s, ::s, :] @ wd.T + bd
    if round_shortcut:  # the dynamic projection block stores R (reading R22)
        ds = _round_array(ds, rmode)
    return _round_array(np.maximum(h2 @ w3.T + b3 + ds, 0.0), rmode)


def proj_dyn_literal(x, wts, idx, s, stride, rmode=ROUND_BF16, threads: int | None = None):
    """Dynamic projection (first) block, literal mode (C; NEXT-f1, reading R22):
    R = rnd(Wd x_s + bd) dense; y = ReLU(R) everywhere, then for every active cell
    of the output grid: gather the input window (side stride*(S-1)+3), conv1, the
    valid 3x3 at stride `stride`, conv3 + R, ReLU, scatter."""
    lib = _load()
    if threads is not None:
        lib.oracle_set_threads(int(threads))
    x, xp = _d(x)
    n, hi, wi, c_in = x.shape
    c_mid = wts["w1"].shape[0]
    c_out = wts["w3"].shape[0]
    keep, wp = _weights(wts)
    wd, wdp = _d(wts["wd"])
    bd, bdp = _d(wts["bd"])
    idx = np.asarray(idx, dtype=np.int32).reshape(-1)
    count = int(idx.size)
    idx, ip = _i32(idx if count else np.zeros(1, np.int32))
    y = np.zeros((n, hi // stride, wi // stride, c_out))
    _, yp = _d(y)
    lib.oracle_proj_dyn_literal(xp, n, hi, wi, c_in, c_mid, c_out, *wp, wdp, bdp, ip, count, int(s), int(stride),
                                rmode, yp)
    return y


def proj_dyn_def(x, wts, mask_cells, s, stride, rmode=ROUND_BF16):
    """Dynamic projection block, definition mode (numpy): y = M ? static projection
    with the stored shortcut : ReLU(rnd(Wd x_s + bd)), M = upsample(mask_cells, S)
    on the output grid (reading R22)."""
    x = np.asarray(x, np.float64)
    st = int(stride)
    ystat = proj_block(x, wts, st, rmode, round_shortcut=True)
    wd, bd = np.asarray(wts["wd"], np.float64), np.asarray(wts["bd"], np.float64)
    r = _round_array(x[:, ::st, ::st, :] @ wd.T + bd, rmode)
    n, h, w, _ = ystat.shape
    m = upsample(mask_cells, h, w, s).astype(bool)
    return np.where(m[..., None], ystat, np.maximum(r, 0.0))


def stem(x, w, b, rmode=ROUND_BF16):
    """ResNet stem, BN folded: y = rnd(ReLU(conv7x7(x, stride 2, pad 3) + b)).
    x [n][H][W][c] (c = 8: 3 channels + zeros), w [64][7][7][c] OHWI -> y [n][H/2][W/2][64]."""
    x = np.asarray(x, np.float64)
    w, b = np.asarray(w, np.float64), np.asarray(b, np.float64)
    n, hi, wi, c = x.shape
    ho, wo = hi // 2, wi // 2
    xp = np.zeros((n, hi + 6, wi + 6, c))
    xp[:, 3:-3, 3:-3] = x
    acc = np.zeros((n, ho, wo, w.shape[0]))
    for dy in range(7):
        for dx in range(7):
            acc += xp[:, dy:dy + 2 * ho:2, dx:dx + 2 * wo:2, :] @ w[:, dy, dx, :].T
    return _round_array(np.maximum(acc + b, 0.0), rmode)


def maxpool(x):
    """3x3 stride-2 max pool with padding 1 (padding never wins): [n][2h][2w][c] -> [n][h][w][c]."""
    x = np.asarray(x, np.float64)
    n, hi, wi, c = x.shape
    xp = np.full((n, hi + 2, wi + 2, c), -np.inf)
    xp[:, 1:-1, 1:-1] = x
    out = np.full((n, hi // 2, wi // 2, c), -np.inf)
    for dy in range(3):
        for dx in range(3):
            out = np.maximum(out, xp[:, dy:dy + hi:2, dx:dx + wi:2, :])
    return out


def head(x, w, b):
    """Global average pool over the pixels, then the classifier: logits = mean_p x[n,p,:] W^T + b (fp64)."""
    x = np.asarray(x, np.float64)
    n = x.shape[0]
    pooled = x.reshape(n, -1, x.shape[-1]).mean(axis=1)
    return pooled @ np.asarray(w, np.float64).T + np.asarray(b, np.float64)


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_threads(t: int) -> None:
    _load().oracle_set_threads(int(t))


def lasnet_forward(x, weights, meta, calibrate_r=None, return_masks=False, force_masks=None, backbone=False):
    """LAS-ResNet forward composed from the functions above (fp64 accumulation, bf16
    storage rounding at every stored tensor): stem -> max pool -> per stage the
    projection (first) block, then the identity blocks as dynamic blocks (masker
    -> compaction -> literal gather/conv/scatter) ->
    head (global average pool + classifier).  The network of SURVEY 8(f) NEXT-f1 /
    BASELINE configs[2] (ResNet-101 depths 3-4-23-3, S_net 4-4-2-1).
      x        [n][H][W][8] fp64 image (channels 3..7 zero)
      weights  nested dict of fp64 arrays (synth.make_lasnet_weights layout)
      meta     {"depths", "s_net", "bm": {block key: masker bias}, "dyn_proj"} as the GPU network's
               LASResNet.oracle_meta(); with calibrate_r set, each block's bias is
               instead chosen from this forward's own logits so that ~r of its cells
               are active (midway between two neighbouring logits) and written to meta.
    force_masks  {block key: cell mask}: take these decisions instead of the masker's
               (the masker still runs and its own masks are returned) -- lets a test
               follow another implementation's decisions through the whole chain.
    backbone   stop after the last stage and return the four stage outputs.
    Returns logits [n][classes] (or the stage outputs), and the per-block masks
    when return_masks."""
    depths, s_net = meta["depths"], meta["s_net"]
    bms = meta.setdefault("bm", {})
    dyn_proj = meta.get("dyn_proj", True)
    cur = maxpool(stem(x, weights["stem_w"], weights["stem_b"]))
    masks = {}
    feats = []

    def decide(key, xin, wm, s_mask):
        if calibrate_r is not None:
            _, l0 = masker(xin, wm, 0.0, s_mask)
            lg = np.sort(l0.reshape(-1))
            k = int(round(calibrate_r * lg.size))
            if k <= 0:
                bm = -(lg[-1] + 1.0)
            elif k >= lg.size:
                bm = -(lg[0] - 1.0)
            else:
                bm = -0.5 * (lg[lg.size - k - 1] + lg[lg.size - k])
            bms[key] = float(np.float32(bm))
        m, _ = masker(xin, wm, bms[key], s_mask)
        masks[key] = m
        if force_masks is not None and key in force_masks:
            m = np.asarray(force_masks[key], np.uint8)
        return compact(m)[0]

    for si, (depth, s) in enumerate(zip(depths, s_net)):
        stride = 1 if si == 0 else 2
        pw = weights[f"s{si}_proj"]
        if dyn_proj:  # the dynamic first block (reading R22): masker over each cell's stride*S input window
            idx = decide(f"s{si}_proj", cur, pw["wm"], s * stride)
            cur = proj_dyn_literal(cur, pw, idx, s, stride)
        else:
            cur = proj_block(cur, pw, stride)
        for b in range(1, depth):
            key = f"s{si}_b{b}"
            wb = weights[key]
            idx = decide(key, cur, wb["wm"], s)
            cur = dyn_block_literal(cur, wb, idx, s)
        feats.append(cur)
    if backbone:
        return (feats, masks) if return_masks else feats
    logits = head(cur, weights["fc_w"], weights["fc_b"])
    return (logits, masks) if return_masks else logits


# ------------------------------------------------------------ LAS-RegNetY (NEXT-f3) --

def gconv3x3(h, w, b, stride=1, group_width=16):
    """Grouped 3x3 convolution, zero padding 1, stride `stride`, + bias (fp64, no
    activation): the RegNet Y-block's middle conv ("different channel numbers
    and convolution groups"; group width 16).  h [n][H][W][C]; w [C][3][3][gw] (OHWI
    with the gw = group_width input channels of the output channel's group)."""
    h = np.asarray(h, np.float64)
    w, b = np.asarray(w, np.float64), np.asarray(b, np.float64)
    n, H, W, C = h.shape
    gw = group_width
    s = int(stride)
    Ho, Wo = -(-H // s), -(-W // s)
    hp = np.zeros((n, H + 2, W + 2, C))
    hp[:, 1:-1, 1:-1] = h
    out = np.zeros((n, Ho, Wo, C))
    G = C // gw
    for dy in range(3):
        for dx in range(3):
            win = hp[:, dy:dy + s * (Ho - 1) + 1:s, dx:dx + s * (Wo - 1) + 1:s, :]  # [n][Ho][Wo][C]
            wg = w[:, dy, dx, :].reshape(G, gw, gw)                                 # [g][out][in]
            out += np.einsum("nyxgi,goi->nyxgo", win.reshape(n, Ho, Wo, G, gw), wg).reshape(n, Ho, Wo, C)
    return out + b


def se_scale(pooled, wts):
    """Squeeze-and-excitation of a pooled feature (Hu et al.): s = sigmoid(W2
    ReLU(W1 p + b1) + b2), fp64.  pooled [n][C] -> s [n][C]."""
    p = np.asarray(pooled, np.float64)
    z = np.maximum(p @ np.asarray(wts["se_w1"], np.float64).T + np.asarray(wts["se_b1"], np.float64), 0.0)
    t = z @ np.asarray(wts["se_w2"], np.float64).T + np.asarray(wts["se_b2"], np.float64)
    return 1.0 / (1.0 + np.exp(-t))


def regnet_block(x, wts, stride=1, mask_cells=None, s=1, rmode=ROUND_BF16):
    """RegNet Y-block (BN folded), static or dynamic (NEXT-f3):
      h1  = rnd(ReLU(x Wa^T + ba))                          1x1
      h2  = rnd(ReLU(gconv3x3(h1, Wb, stride) + bb))        grouped 3x3, group width 16
      p   = mean of h2 over the computed output pixels      (reading R23: in a dynamic
                                                             block, the ACTIVE pixels only)
      h2s = rnd(h2 * se_scale(p))                           squeeze-and-excitation
      R   = x (identity) or Wd x_s + bd (projection, unstored, reading R21)
      y   = rnd(ReLU(R + h2s Wc^T + bc)) on computed pixels; x on the others
    x [n][H][W][c_in]; mask_cells [n][gh][gw] on the output grid (None: static block,
    every pixel computed); projection when wts has "wd" (stride 1 or 2, static only).
    An image without active cells keeps y = x (no pooled mean is needed)."""
    x = np.asarray(x, np.float64)
    f = {k: np.asarray(v, np.float64) for k, v in wts.items()}
    st = int(stride)
    h1 = _round_array(np.maximum(x @ f["wa"].T + f["ba"], 0.0), rmode)
    h2 = _round_array(np.maximum(gconv3x3(h1, f["wb"], f["bb"], st), 0.0), rmode)
    n, Ho, Wo, C = h2.shape
    if mask_cells is None:
        m = np.ones((n, Ho, Wo), bool)
    else:
        m = upsample(mask_cells, Ho, Wo, s).astype(bool)
    cnt = m.reshape(n, -1).sum(axis=1)
    pooled = (h2 * m[..., None]).reshape(n, -1, C).sum(axis=1) / np.maximum(cnt, 1)[:, None]
    sc = se_scale(pooled, f)
    h2s = _round_array(h2 * sc[:, None, None, :], rmode)
    if "wd" in f:
        R = x[:, ::st, ::st, :] @ f["wd"].T + f["bd"]
    else:
        R = x
    y = _round_array(np.maximum(R + h2s @ f["wc"].T + f["bc"], 0.0), rmode)
    if mask_cells is None:
        return y
    return np.where(m[..., None], y, x)


def regnet_block_literal(x, wts, idx, s, rmode=ROUND_BF16):
    """Dynamic RegNet Y identity block, literal gather -> compute -> scatter (P:89,
    P:163-170) in plain loops over the active patches, in two passes because the
    SE pool needs every active pixel of the image first (reading R23):
      pass 1, per active patch: gather the (S+2)^2 halo window of x, conv1 (0 outside
        the image, R6), valid grouped 3x3 -> S x S h2, accumulate the in-image h2
        into the image's pooled sum;
      SE per image over its active pixels;
      pass 2, per active patch: h2s = rnd(h2 * s), conv3 + residual, ReLU, scatter.
    Small inputs only (Python loops)."""
    x = np.asarray(x, np.float64)
    f = {k: np.asarray(v, np.float64) for k, v in wts.items()}
    n, H, W, _ = x.shape
    C = f["wa"].shape[0]
    gh, gw = grid(H, W, s)
    hs = s + 2
    y = x.copy()
    patches = []
    psum = np.zeros((n, C))
    pcnt = np.zeros(n)
    for cid in np.asarray(idx).reshape(-1):
        img, g = divmod(int(cid), gh * gw)
        gy, gx = divmod(g, gw)
        win = np.zeros((hs, hs, C))
        for wy in range(hs):
            for wx in range(hs):
                sy, sx = gy * s - 1 + wy, gx * s - 1 + wx
                if 0 <= sy < H and 0 <= sx < W:
                    win[wy, wx] = _round_array(np.maximum(x[img, sy, sx] @ f["wa"].T + f["ba"], 0.0), rmode)
        h2 = np.zeros((s, s, C))
        for py in range(s):
            for px in range(s):
                acc = f["bb"].copy()
                for o in range(C):
                    g0 = (o // 16) * 16
                    for dy in range(3):
                        for dx in range(3):
                            acc[o] += f["wb"][o, dy, dx, :] @ win[py + dy, px + dx, g0:g0 + 16]
                h2[py, px] = _round_array(np.maximum(acc, 0.0), rmode)
                if gy * s + py < H and gx * s + px < W:
                    psum[img] += h2[py, px]
                    pcnt[img] += 1
        patches.append((img, gy, gx, h2))
    sc = se_scale(psum / np.maximum(pcnt, 1)[:, None], f)
    for img, gy, gx, h2 in patches:
        for py in range(s):
            for px in range(s):
                yy, xx = gy * s + py, gx * s + px
                if yy < H and xx < W:
                    h2s = _round_array(h2[py, px] * sc[img], rmode)
                    y[img, yy, xx] = _round_array(np.maximum(x[img, yy, xx] + h2s @ f["wc"].T + f["bc"], 0.0), rmode)
    return y


def regnet_stem(x, w, b, rmode=ROUND_BF16):
    """RegNet stem, BN folded: y = rnd(ReLU(conv3x3(x, stride 2, pad 1) + b)).
    x [n][H][W][c]; w [co][3][3][c] OHWI -> y [n][H/2][W/2][co]."""
    x = np.asarray(x, np.float64)
    w, b = np.asarray(w, np.float64), np.asarray(b, np.float64)
    n, hi, wi, c = x.shape
    ho, wo = hi // 2, wi // 2
    xp = np.zeros((n, hi + 2, wi + 2, c))
    xp[:, 1:-1, 1:-1] = x
    acc = np.zeros((n, ho, wo, w.shape[0]))
    for dy in range(3):
        for dx in range(3):
            acc += xp[:, dy:dy + 2 * ho:2, dx:dx + 2 * wo:2, :] @ w[:, dy, dx, :].T
    return _round_array(np.maximum(acc + b, 0.0), rmode)


def regnet_forward(x, weights, meta, calibrate_r=None, force_masks=None, return_masks=False):
    """LAS-RegNetY forward (BASELINE configs[3]; NEXT-f3): RegNet stem -> per stage the
    static first block (stride 2, projection) and the identity Y-blocks as dynamic
    blocks (masker -> compaction -> regnet_block with the mask) ->
    head.  meta: {"depths", "s_net", "bm": {key: bias}}; calibrate_r / force_masks as
    lasnet_forward.  x [n][H][W][8] (channels 3..7 zero)."""
    depths, s_net = meta["depths"], meta["s_net"]
    bms = meta.setdefault("bm", {})
    cur = regnet_stem(x, weights["stem_w"], weights["stem_b"])
    masks = {}
    for si, (depth, s) in enumerate(zip(depths, s_net)):
        cur = regnet_block(cur, weights[f"s{si}_b0"], stride=2)
        for b in range(1, depth):
            key = f"s{si}_b{b}"
            wb = weights[key]
            if calibrate_r is not None:
                _, l0 = masker(cur, wb["wm"], 0.0, s)
                lg = np.sort(l0.reshape(-1))
                k = int(round(calibrate_r * lg.size))
                bm = -(lg[-1] + 1.0) if k <= 0 else (-(lg[0] - 1.0) if k >= lg.size else
                                                      -0.5 * (lg[lg.size - k - 1] + lg[lg.size - k]))
                bms[key] = float(np.float32(bm))
            m, _ = masker(cur, wb["wm"], bms[key], s)
            masks[key] = m
            if force_masks is not None and key in force_masks:
                m = np.asarray(force_masks[key], np.uint8)
            cur = regnet_block(cur, wb, stride=1, mask_cells=m, s=s)
    logits = head(cur, weights["fc_w"], weights["fc_b"])
    return (logits, masks) if return_masks else logits
