"""Pins for the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a library routine
(torch.nn.functional.conv2d in float64, numpy.flatnonzero, numpy.kron),
exact rational arithmetic (fractions.Fraction), closed forms, a bit-level
second implementation of bf16 rounding pinned by torch's fp32->bf16 cast,
or brute force written here in plain Python loops.
"""
from fractions import Fraction
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth


# ---------------------------------------------------------------- helpers ----

def bf16_rne_bits(a: np.ndarray) -> np.ndarray:
    """Second, bit-level implementation of fp64 -> bf16 round-to-nearest-even
    (keep 7 of the 52 fp64 fraction bits; ties to even), normal range only."""
    a = np.asarray(a, np.float64)
    bits = a.view(np.uint64).copy()
    drop = np.uint64(52 - 7)
    lsb = (bits >> drop) & np.uint64(1)
    half = np.uint64(1) << (drop - np.uint64(1))
    bits = bits + half - np.uint64(1) + lsb
    bits &= ~((np.uint64(1) << drop) - np.uint64(1))
    out = bits.view(np.float64)
    return np.where(a == 0, a, out)


def torch_static_block(x, wts, rnd=None):
    """Static bottleneck with torch float64 conv2d (library routine)."""
    r = (lambda t: t) if rnd is None else rnd
    xt = torch.from_numpy(x).permute(0, 3, 1, 2)  # NCHW
    w1 = torch.from_numpy(wts["w1"])[:, :, None, None]
    w2 = torch.from_numpy(wts["w2"]).permute(0, 3, 1, 2)  # OHWI -> OIHW
    w3 = torch.from_numpy(wts["w3"])[:, :, None, None]
    h1 = r(torch.relu(F.conv2d(xt, w1, torch.from_numpy(wts["b1"]))))
    h2 = r(torch.relu(F.conv2d(h1, w2, torch.from_numpy(wts["b2"]), padding=1)))
    y = r(torch.relu(xt + F.conv2d(h2, w3, torch.from_numpy(wts["b3"]))))
    return y.permute(0, 2, 3, 1).contiguous().numpy(), h1.permute(0, 2, 3, 1).numpy(), h2.permute(0, 2, 3, 1).numpy()


def tiny_case(n, h, w, c_in, c_mid, seed, dtype="bf16", relu=True):
    x = synth.to_f64(synth.make_x(n, h, w, c_in, seed=seed, dtype=dtype, relu=relu))
    wts = synth.weights_f64(synth.make_block_weights(c_in, c_mid, c_in, seed=seed + 100, dtype=dtype))
    return x, wts


# ------------------------------------------------------------ rounding -------

def test_round_bf16_matches_torch_cast_on_fp32_values(oracle_mod):
    g = torch.Generator().manual_seed(0)
    v = torch.randn(4000, generator=g) * torch.exp2(torch.randint(-30, 30, (4000,), generator=g).float())
    want = v.to(torch.bfloat16).to(torch.float64).numpy()
    got = np.array([oracle_mod.round_bf16(float(t)) for t in v.to(torch.float64)])
    assert np.array_equal(got, want)


def test_round_bf16_ties_and_subnormals(oracle_mod):
    r = oracle_mod.round_bf16
    assert r(1 + 2 ** -8) == 1.0                      # tie -> even (down)
    assert r(1 + 3 * 2 ** -8) == 1 + 2 ** -6           # tie -> even (up)
    assert r(-(1 + 3 * 2 ** -8)) == -(1 + 2 ** -6)
    assert r(2 ** -134) == 0.0                         # subnormal tie -> even (0)
    assert r(3 * 2 ** -134) == 2 ** -132               # subnormal tie -> even
    assert r(1e-300) == 0.0
    assert r(3.0e38) == 226 * 2.0 ** 120          # finite: 1.765625 * 2^127
    assert r(3.4e38) == float("inf")            # above the RNE overflow threshold
    assert oracle_mod.round_f32(1 + 2 ** -30) == 1.0


def test_bitlevel_rne_helper_agrees_with_torch():
    g = torch.Generator().manual_seed(1)
    v = torch.randn(5000, generator=g, dtype=torch.float32)
    assert np.array_equal(bf16_rne_bits(v.double().numpy()), v.to(torch.bfloat16).double().numpy())


# --------------------------------------------------------------- masker ------

@pytest.mark.parametrize("h,w,s", [(4, 4, 2), (5, 5, 2), (7, 5, 3), (4, 6, 1), (5, 7, 4)])
def test_masker_exact_rational_sign(oracle_mod, h, w, s):
    """logit = sum_c w_c * mean_{p in Omega} x_pc + b computed exactly with Fractions
    (P:109 pooling + 1x1 conv; R1 average; R7 clipped Omega; R3 strict >)."""
    c = 8
    x = synth.to_f64(synth.make_x(2, h, w, c, seed=h * 31 + w, relu=False))
    wm = synth.make_masker_weights(c, seed=7).double().numpy()
    b = 0.01
    mask, logit = oracle_mod.masker(x, wm, b, s)
    gh, gw = -(-h // s), -(-w // s)
    for n in range(2):
        for gy in range(gh):
            for gx in range(gw):
                pix = [(yy, xx) for yy in range(gy * s, min(gy * s + s, h)) for xx in range(gx * s, min(gx * s + s, w))]
                exact = Fraction(b)
                for ci in range(c):
                    tot = sum(Fraction(x[n, yy, xx, ci]) for yy, xx in pix)
                    exact += Fraction(wm[ci]) * tot / len(pix)
                assert mask[n, gy, gx] == (1 if exact > 0 else 0)
                assert abs(Fraction(logit[n, gy, gx]) - exact) <= Fraction(1, 10 ** 12) * (1 + abs(exact))


def test_masker_two_channel_argmax_equals_reduced_sign(oracle_mod):
    """App. B eq.: [x*W]_0 > [x*W]_1  <=>  x*(W_0-W_1) > 0, at >= 1000 cells."""
    c = 32
    x = synth.to_f64(synth.make_x(4, 16, 16, c, seed=11))
    W, bb = synth.make_masker_weights_2ch(c, seed=12)
    W = W.double().numpy()
    bb = bb.double().numpy()
    m2, z0, z1 = oracle_mod.masker_2ch(x, W, bb, 1)
    m1, l1 = oracle_mod.masker(x, W[0] - W[1], bb[0] - bb[1], 1)
    assert m2.size >= 1000
    sure = np.abs(z0 - z1) > 1e-12
    assert sure.sum() >= 1000
    assert np.array_equal(m2[sure], m1[sure])
    np.testing.assert_allclose(l1, z0 - z1, rtol=0, atol=1e-12)


def test_masker_s1_is_per_pixel_matvec(oracle_mod):
    """S = 1: pooling is the identity, logit = x . w + b (numpy matmul)."""
    c = 16
    x = synth.to_f64(synth.make_x(2, 5, 6, c, seed=5, relu=False))
    wm = synth.make_masker_weights(c, seed=6).double().numpy()
    mask, logit = oracle_mod.masker(x, wm, -0.02, 1)
    np.testing.assert_allclose(logit, x @ wm - 0.02, rtol=0, atol=1e-13)
    assert np.array_equal(mask, (x @ wm - 0.02 > 0).astype(np.uint8))


def test_masker_constant_input_closed_form(oracle_mod):
    """x == a everywhere: logit = a * sum(w) + b for every cell, clipped or not."""
    c = 16
    a = 0.75
    x = np.full((1, 7, 9, c), a)
    wm = synth.make_masker_weights(c, seed=9).double().numpy()
    mask, logit = oracle_mod.masker(x, wm, 0.125, 4)
    np.testing.assert_allclose(logit, a * wm.sum() + 0.125, rtol=1e-14, atol=1e-15)
    assert logit.shape == (1, 2, 3)


def test_masker_tie_is_inactive(oracle_mod):
    """R3: logit exactly 0 -> not selected (strict >)."""
    x = np.zeros((1, 4, 4, 16))
    mask, logit = oracle_mod.masker(x, np.ones(16), 0.0, 2)
    assert np.all(logit == 0) and np.all(mask == 0)


# ----------------------------------------------------- compaction, upsample --

@pytest.mark.parametrize("r", [0.0, 0.1, 0.5, 1.0])
def test_compact_equals_flatnonzero(oracle_mod, r):
    m = synth.make_cell_mask(3, 7, 9, r, seed=4)
    idx, count = oracle_mod.compact(m)
    ref = np.flatnonzero(m.reshape(-1))
    assert count == int(m.sum()) == len(ref)
    assert np.array_equal(idx, ref)
    assert np.all(np.diff(idx) > 0)


def test_upsample_matches_kron_and_preserves_rate(oracle_mod):
    m = synth.make_cell_mask(2, 7, 7, 0.5, seed=8)
    for s in (1, 2, 4):
        up = oracle_mod.upsample(m, 7 * s, 7 * s, s)
        ref = np.stack([np.kron(m[i], np.ones((s, s), np.uint8)) for i in range(2)])
        assert np.array_equal(up, ref)
        assert Fraction(int(up.sum()), up.size) == Fraction(int(m.sum()), m.size)


# ---------------------------------------------------------- static block -----

@pytest.mark.parametrize("n,h,w,c_in,c_mid", [(1, 5, 7, 32, 16), (2, 8, 8, 64, 16), (1, 4, 4, 16, 8)])
def test_static_block_matches_torch_conv2d_fp64(oracle_mod, n, h, w, c_in, c_mid):
    x, wts = tiny_case(n, h, w, c_in, c_mid, seed=h + w)
    y, h1, h2 = oracle_mod.static_block(x, wts, rmode=oracle_mod.ROUND_NONE, return_intermediates=True)
    yt, h1t, h2t = torch_static_block(x, wts)
    np.testing.assert_allclose(h1, h1t, rtol=0, atol=1e-12)
    np.testing.assert_allclose(h2, h2t, rtol=0, atol=1e-12)
    np.testing.assert_allclose(y, yt, rtol=0, atol=1e-12)


def test_static_block_bf16_storage_rounding(oracle_mod):
    """bf16 RNE at h1/h2/y (R13) vs torch fp64 conv2d + bit-level RNE."""
    x, wts = tiny_case(2, 6, 7, 32, 16, seed=21)
    y = oracle_mod.static_block(x, wts, rmode=oracle_mod.ROUND_BF16)
    rnd = lambda t: torch.from_numpy(bf16_rne_bits(t.numpy()))
    yt, _, _ = torch_static_block(x, wts, rnd=rnd)
    assert np.mean(y == yt) > 0.999
    ulp = np.abs(yt) * 2.0 ** -7 + 1e-30
    assert np.all(np.abs(y - yt) <= ulp)


def test_static_block_fp32_storage_rounding(oracle_mod):
    x, wts = tiny_case(1, 5, 5, 16, 16, seed=22, dtype="f32")
    y = oracle_mod.static_block(x, wts, rmode=oracle_mod.ROUND_F32)
    rnd = lambda t: t.float().double()
    yt, _, _ = torch_static_block(x, wts, rnd=rnd)
    np.testing.assert_allclose(y, yt, rtol=1e-7, atol=1e-12)


# ------------------------------------------------------------- dyn block -----

SHAPES = [(1, 4, 4, 32, 16, 2), (2, 5, 5, 32, 16, 2), (1, 7, 7, 32, 16, 4), (1, 8, 8, 64, 32, 3),
          (2, 7, 5, 32, 16, 1), (1, 8, 8, 32, 16, 8), (1, 5, 8, 16, 16, 7)]


@pytest.mark.parametrize("n,h,w,c_in,c_mid,s", SHAPES)
def test_literal_equals_definition(oracle_mod, n, h, w, c_in, c_mid, s):
    """Gather/compute/scatter reaches the definition y = M ? static : x exactly."""
    x, wts = tiny_case(n, h, w, c_in, c_mid, seed=s * 7 + h)
    gh, gw = -(-h // s), -(-w // s)
    for r in (0.3, 0.7):
        mc = synth.make_cell_mask(n, gh, gw, r, seed=3)
        idx, _ = oracle_mod.compact(mc)
        y_lit = oracle_mod.dyn_block_literal(x, wts, idx, s)
        y_def = oracle_mod.dyn_block_def(x, wts, mc, s)
        assert np.array_equal(y_lit, y_def)


@pytest.mark.parametrize("n,h,w,c_in,c_mid,s", SHAPES[:4])
def test_all_zero_mask_is_identity_and_all_one_is_static(oracle_mod, n, h, w, c_in, c_mid, s):
    x, wts = tiny_case(n, h, w, c_in, c_mid, seed=5)
    gh, gw = -(-h // s), -(-w // s)
    zeros = np.zeros((n, gh, gw), np.uint8)
    ones = np.ones((n, gh, gw), np.uint8)
    assert np.array_equal(oracle_mod.dyn_block_literal(x, wts, [], s), x)
    idx, _ = oracle_mod.compact(ones)
    assert np.array_equal(oracle_mod.dyn_block_literal(x, wts, idx, s),
                          oracle_mod.static_block(x, wts))
    assert np.array_equal(oracle_mod.dyn_block_def(x, wts, zeros, s), x)


@pytest.mark.parametrize("s", [2, 3, 4])
def test_granularity_equivalence_to_pixel_level(oracle_mod, s):
    """dyn(x, Mc, S) == dyn(x, upsample(Mc, S), 1): S = 1 is pixel-level DynConv."""
    n, h, w = 2, 8, 7
    x, wts = tiny_case(n, h, w, 32, 16, seed=40 + s)
    gh, gw = -(-h // s), -(-w // s)
    mc = synth.make_cell_mask(n, gh, gw, 0.5, seed=s)
    idx, _ = oracle_mod.compact(mc)
    up = oracle_mod.upsample(mc, h, w, s)
    idx1, _ = oracle_mod.compact(up)
    assert np.array_equal(oracle_mod.dyn_block_literal(x, wts, idx, s),
                          oracle_mod.dyn_block_literal(x, wts, idx1, 1))


def test_closed_form_w3_zero(oracle_mod):
    """W3 = 0, b3 = 0 -> y = ReLU(x) on active pixels, x elsewhere."""
    x, wts = tiny_case(1, 6, 6, 32, 16, seed=50, relu=False)
    wts["w3"][:] = 0
    wts["b3"][:] = 0
    mc = synth.make_cell_mask(1, 3, 3, 0.5, seed=1)
    y = oracle_mod.dyn_block_literal(x, wts, oracle_mod.compact(mc)[0], 2)
    up = np.kron(mc[0], np.ones((2, 2), np.uint8)).astype(bool)
    assert np.array_equal(y[0][up], np.maximum(x[0][up], 0))
    assert np.array_equal(y[0][~up], x[0][~up])


def test_closed_form_w1_zero(oracle_mod):
    """W1 = 0, b1 = 0 -> h1 = 0, h2 = round(ReLU(b2)), y = round(ReLU(x + W3 h2 + b3))."""
    x, wts = tiny_case(1, 5, 5, 32, 16, seed=51)
    wts["w1"][:] = 0
    wts["b1"][:] = 0
    h2 = bf16_rne_bits(np.maximum(wts["b2"], 0))
    z = wts["w3"] @ h2 + wts["b3"]
    y = oracle_mod.static_block(x, wts)
    want = bf16_rne_bits(np.maximum(x + z, 0))
    assert np.array_equal(y, want)


def test_single_cell_covering_image_is_static_block(oracle_mod):
    """S = H = W, the single cell active -> the whole-image static block (P:109 extreme)."""
    x, wts = tiny_case(1, 6, 6, 32, 16, seed=52)
    y = oracle_mod.dyn_block_literal(x, wts, [0], 6)
    assert np.array_equal(y, oracle_mod.static_block(x, wts))


def test_block_pixel_matches_definition(oracle_mod):
    x, wts = tiny_case(2, 7, 9, 32, 16, seed=53)
    mc = synth.make_cell_mask(2, 4, 5, 0.5, seed=9)
    y = oracle_mod.dyn_block_def(x, wts, mc, 2)
    rng = np.random.default_rng(0)
    for _ in range(25):
        n, yy, xx = rng.integers(2), rng.integers(7), rng.integers(9)
        out, act = oracle_mod.block_pixel(x, wts, mc, 2, n, yy, xx)
        assert np.array_equal(out, y[n, yy, xx])
        assert act == bool(mc[n, yy // 2, xx // 2])


# ----------------------------------------------------------- brute force -----

def _brute_block(x, wts, mc, s):
    """Whole block in plain Python loops straight from P:86/P:89 (tiny sizes only)."""
    n_img, h, w, c_in = x.shape
    c_mid = wts["w1"].shape[0]
    W1, b1, W2, b2, W3, b3 = (wts[k] for k in ("w1", "b1", "w2", "b2", "w3", "b3"))
    rnd = lambda v: float(bf16_rne_bits(np.array([v]))[0])
    h1 = {}
    for n in range(n_img):
        for yy in range(h):
            for xx in range(w):
                for c in range(c_mid):
                    a = float(b1[c])
                    for ci in range(c_in):
                        a += float(W1[c, ci]) * float(x[n, yy, xx, ci])
                    h1[n, yy, xx, c] = rnd(max(a, 0.0))
    y = x.copy()
    for n in range(n_img):
        for yy in range(h):
            for xx in range(w):
                if not mc[n, yy // s, xx // s]:
                    continue
                h2 = []
                for c in range(c_mid):
                    a = float(b2[c])
                    for dy in range(3):
                        for dx in range(3):
                            sy, sx = yy + dy - 1, xx + dx - 1
                            if 0 <= sy < h and 0 <= sx < w:
                                for ci in range(c_mid):
                                    a += float(W2[c, dy, dx, ci]) * h1[n, sy, sx, ci]
                    h2.append(rnd(max(a, 0.0)))
                for co in range(c_in):
                    a = float(b3[co])
                    for c in range(c_mid):
                        a += float(W3[co, c]) * h2[c]
                    y[n, yy, xx, co] = rnd(max(float(x[n, yy, xx, co]) + a, 0.0))
    return y


@pytest.mark.parametrize("h,w,s", [(4, 4, 2), (5, 4, 3)])
def test_brute_force_exhaustive_masks(oracle_mod, h, w, s):
    """Every coarse mask of a G <= 4 grid, compared with plain-Python loops."""
    x, wts = tiny_case(1, h, w, 8, 4, seed=60 + h)
    gh, gw = -(-h // s), -(-w // s)
    G = gh * gw
    assert G <= 4
    for bits in itertools.product([0, 1], repeat=G):
        mc = np.array(bits, np.uint8).reshape(1, gh, gw)
        idx, _ = oracle_mod.compact(mc)
        got = oracle_mod.dyn_block_literal(x, wts, idx, s)
        want = _brute_block(x, wts, mc, s)
        assert np.array_equal(got, want)  # same summation order: exact


# ------------------------------------------------- projection block (NEXT-f1) --

@pytest.mark.parametrize("stride,h,c_in,c_mid,c_out", [(1, 8, 64, 64, 128), (2, 8, 64, 64, 128), (2, 6, 32, 16, 64)])
def test_proj_block_equals_torch_conv2d_f64(oracle_mod, stride, h, c_in, c_mid, c_out):
    """oracle.proj_block (unrounded) == the same block built from float64
    torch.nn.functional.conv2d (library routine): 1x1, 3x3 stride s pad 1, 1x1,
    and the 1x1 stride-s shortcut."""
    import torch.nn.functional as F

    x = synth.make_x(2, h, h, c_in, seed=stride + h)
    w = synth.make_proj_weights(c_in, c_mid, c_out, seed=5)
    got = oracle_mod.proj_block(synth.to_f64(x), synth.weights_f64(w), stride, rmode=oracle_mod.ROUND_NONE)
    xt = torch.from_numpy(synth.to_f64(x)).permute(0, 3, 1, 2)
    W = {k: torch.from_numpy(v) for k, v in synth.weights_f64(w).items()}
    h1 = F.relu(F.conv2d(xt, W["w1"][:, :, None, None], W["b1"]))
    h2 = F.relu(F.conv2d(h1, W["w2"].permute(0, 3, 1, 2), W["b2"], stride=stride, padding=1))
    ds = F.conv2d(xt, W["wd"][:, :, None, None], W["bd"], stride=stride)
    want = F.relu(F.conv2d(h2, W["w3"][:, :, None, None], W["b3"]) + ds).permute(0, 2, 3, 1).numpy()
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_proj_block_closed_form_zero_conv1(oracle_mod):
    """W1 = 0, b1 = 0 -> h1 = 0, h2 = ReLU(b2) everywhere, so
    y = ReLU(W3 ReLU(b2) + b3 + Wd x_s + bd) per output pixel (rounded as stored)."""
    x = synth.make_x(1, 6, 6, 64, seed=3)
    w = synth.weights_f64(synth.make_proj_weights(64, 64, 128, seed=4))
    w["w1"][:] = 0.0
    w["b1"][:] = 0.0
    y = oracle_mod.proj_block(synth.to_f64(x), w, 2, rmode=oracle_mod.ROUND_NONE)
    xs = synth.to_f64(x)[:, ::2, ::2, :]
    want = np.maximum(w["w3"] @ np.maximum(w["b2"], 0.0) + w["b3"] + xs @ w["wd"].T + w["bd"], 0.0)
    assert np.allclose(y, want, rtol=0, atol=1e-12)


# --------------------------------------------------- stem, pool, head (NEXT-f1) --

def test_stem_pool_head_equal_torch_f64(oracle_mod):
    """oracle.stem / maxpool / head == float64 torch conv2d(7x7, s2, p3) + ReLU,
    max_pool2d(3, s2, p1) and adaptive-avg-pool + linear (library routines)."""
    g = torch.Generator().manual_seed(0)
    x = torch.randn((2, 16, 24, 8), generator=g, dtype=torch.float64)
    x[..., 3:] = 0.0
    w = torch.randn((64, 7, 7, 8), generator=g, dtype=torch.float64) * 0.1
    b = torch.randn((64,), generator=g, dtype=torch.float64) * 0.1
    got = oracle_mod.stem(x.numpy(), w.numpy(), b.numpy(), rmode=oracle_mod.ROUND_NONE)
    want = F.relu(F.conv2d(x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), b, stride=2, padding=3))
    assert np.abs(got - want.permute(0, 2, 3, 1).numpy()).max() < 1e-12
    mp = oracle_mod.maxpool(got)
    want_mp = F.max_pool2d(torch.from_numpy(got).permute(0, 3, 1, 2), 3, stride=2, padding=1)
    assert np.array_equal(mp, want_mp.permute(0, 2, 3, 1).numpy())  # a max selects: exact
    wf = torch.randn((10, 64), generator=g, dtype=torch.float64)
    bf = torch.randn((10,), generator=g, dtype=torch.float64)
    lg = oracle_mod.head(mp, wf.numpy(), bf.numpy())
    want_lg = F.linear(F.adaptive_avg_pool2d(want_mp, 1).flatten(1), wf, bf)
    assert np.abs(lg - want_lg.numpy()).max() < 1e-12


# ------------------------------------ dynamic projection block (NEXT-f1, R22) --

def proj_case(n, hi, c_in, c_mid, c_out, seed, relu=True):
    x = synth.to_f64(synth.make_x(n, hi, hi + 2, c_in, seed=seed, relu=relu))
    w = synth.weights_f64(synth.make_proj_weights(c_in, c_mid, c_out, seed=seed + 1))
    return x, w


def torch_proj_parts(x, w, stride):
    """h2 (unrounded ReLU(3x3 stride-s conv of h1)) and the shortcut R = Wd x_s + bd
    from float64 torch conv2d (library routine); x NHWC -> NCHW tensors."""
    xt = torch.from_numpy(x).permute(0, 3, 1, 2)
    W = {k: torch.from_numpy(v) for k, v in w.items()}
    h1 = torch.relu(F.conv2d(xt, W["w1"][:, :, None, None], W["b1"]))
    h2 = torch.relu(F.conv2d(h1, W["w2"].permute(0, 3, 1, 2), W["b2"], stride=stride, padding=1))
    R = F.conv2d(xt, W["wd"][:, :, None, None], W["bd"], stride=stride)
    return h2, R, W


@pytest.mark.parametrize("stride,s", [(1, 2), (2, 1), (2, 2), (2, 3), (2, 4)])
def test_proj_dyn_literal_equals_torch_masked(oracle_mod, stride, s):
    """Unrounded (fp64) literal dynamic projection block == ReLU(R + M (W3 h2 + b3))
    built from float64 torch conv2d, M the nearest-upsampled cell mask: every
    term (window origin, stride of the 3x3, clipping, shortcut) is fixed by the
    library routine; S = 3 does not divide the 6 x 7 output grid (clipped cells)."""
    x, w = proj_case(2, 12, 32, 16, 64, seed=10 * stride + s)
    h, wd = 12 // stride, 14 // stride
    gh, gw = -(-h // s), -(-wd // s)
    mc = synth.make_cell_mask(2, gh, gw, 0.5, seed=s)
    idx, _ = oracle_mod.compact(mc)
    got = oracle_mod.proj_dyn_literal(x, w, idx, s, stride, rmode=oracle_mod.ROUND_NONE)
    h2, R, W = torch_proj_parts(x, w, stride)
    F3 = F.conv2d(h2, W["w3"][:, :, None, None], W["b3"])
    M = torch.from_numpy(np.kron(mc, np.ones((s, s), np.uint8))[:, :h, :wd].astype(np.float64))[:, None]
    want = torch.relu(R + M * F3).permute(0, 2, 3, 1).numpy()
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("stride,s", [(1, 2), (2, 2), (2, 3)])
def test_proj_dyn_literal_equals_definition(oracle_mod, stride, s):
    """Literal (C, gather/compute/scatter) vs definition (numpy: masked select of the
    static projection block with the stored shortcut) -- two independent writings,
    fp64 (reassociation only) and with bf16 storage rounding."""
    x, w = proj_case(2, 12, 64, 32, 128, seed=40 + s, relu=False)
    h, wd = 12 // stride, 14 // stride
    mc = synth.make_cell_mask(2, -(-h // s), -(-wd // s), 0.6, seed=s + 1)
    idx, _ = oracle_mod.compact(mc)
    a = oracle_mod.proj_dyn_literal(x, w, idx, s, stride, rmode=oracle_mod.ROUND_NONE)
    b = oracle_mod.proj_dyn_def(x, w, mc, s, stride, rmode=oracle_mod.ROUND_NONE)
    assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()
    a = oracle_mod.proj_dyn_literal(x, w, idx, s, stride)
    b = oracle_mod.proj_dyn_def(x, w, mc, s, stride)
    assert np.mean(a == b) > 0.999  # a bf16 tie may flip under fp64 reassociation
    assert np.abs(a - b).max() <= 2 ** -7 * np.abs(b).max()


def test_proj_dyn_all_ones_all_zeros(oracle_mod):
    """All-ones mask == the static projection block with the stored shortcut
    (itself pinned by torch conv2d above); all-zeros mask == ReLU(rnd(R)), R from
    torch conv2d and rounded by the bit-level RNE."""
    stride, s = 2, 2
    x, w = proj_case(1, 8, 32, 16, 64, seed=70)
    h, wd = 4, 5
    gh, gw = 2, 3
    ones = np.ones((1, gh, gw), np.uint8)
    idx, _ = oracle_mod.compact(ones)
    got = oracle_mod.proj_dyn_literal(x, w, idx, s, stride)
    want = oracle_mod.proj_block(x, w, stride, round_shortcut=True)
    assert np.array_equal(got, want)
    got0 = oracle_mod.proj_dyn_literal(x, w, np.zeros(0, np.int32), s, stride)
    _, R, _ = torch_proj_parts(x, w, stride)
    want0 = np.maximum(bf16_rne_bits(R.permute(0, 2, 3, 1).numpy()), 0.0)
    assert np.array_equal(got0, want0)


def test_proj_dyn_identity_shortcut_reduces_to_identity_block(oracle_mod):
    """Stride 1, c_in == c_out, Wd = I, bd = 0: R = rnd(x) = x (bf16 input), so the
    dynamic projection block IS the identity dynamic block (P:86 input fill) --
    pinned against the independent identity-block literal at every cell mask."""
    s = 2
    x = synth.to_f64(synth.make_x(2, 8, 6, 64, seed=80))
    w = synth.weights_f64(synth.make_block_weights(64, 32, 64, seed=81))
    w["wd"] = np.eye(64)
    w["bd"] = np.zeros(64)
    mc = synth.make_cell_mask(2, 4, 3, 0.5, seed=82)
    idx, _ = oracle_mod.compact(mc)
    a = oracle_mod.proj_dyn_literal(x, w, idx, s, 1)
    b = oracle_mod.dyn_block_literal(x, {k: w[k] for k in ("w1", "b1", "w2", "b2", "w3", "b3")}, idx, s)
    assert np.array_equal(a, b)


def test_proj_dyn_granularity_equivalence(oracle_mod):
    """dyn(M_c, S) == dyn(upsample(M_c, S), 1) at stride 2 (S = 1 is the
    pixel-level case): every output pixel does the same arithmetic in the same order."""
    stride, s = 2, 2
    x, w = proj_case(2, 16, 32, 16, 64, seed=90)
    h, wd = 8, 9
    mc = synth.make_cell_mask(2, 4, 5, 0.5, seed=91)
    idx, _ = oracle_mod.compact(mc)
    a = oracle_mod.proj_dyn_literal(x, w, idx, s, stride)
    up = np.kron(mc, np.ones((s, s), np.uint8))[:, :h, :wd]
    idx1, _ = oracle_mod.compact(up)
    b = oracle_mod.proj_dyn_literal(x, w, idx1, 1, stride)
    assert np.array_equal(a, b)


def test_proj_masker_grid_is_output_grid(oracle_mod):
    """The stride-2 masker pools the 2S x 2S input window of each output cell: the
    input-resolution masker at granularity 2S has exactly the output grid, and its
    logits equal the pooled-mean closed form over the clipped input window."""
    x = synth.to_f64(synth.make_x(1, 14, 10, 16, seed=95))
    wm = np.linspace(-1, 1, 16)
    s, st = 3, 2
    m, lg = oracle_mod.masker(x, wm, 0.1, st * s)
    assert m.shape == (1, -(-7 // s), -(-5 // s))
    for gy in range(m.shape[1]):
        for gx in range(m.shape[2]):
            win = x[0, st * s * gy:st * s * gy + st * s, st * s * gx:st * s * gx + st * s, :]
            want = float(win.reshape(-1, 16).mean(axis=0) @ wm) + 0.1
            assert abs(lg[0, gy, gx] - want) <= 1e-12
