"""Parity of the CUDA path (through the C ABI) with the CPU oracle (-m gpu).

Masks and indices: bit-exact.  Activations: max-abs-rel <= 2e-2 (bf16, fp32
accumulation) or 1e-5 (fp32 path), per tensor; inactive pixels: bitwise x.
Sizes span several 128-row tiles with ragged tails; the full-size config-2
launch (the one bench.py times) is checked on sampled pixels.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import (BF16_TOL, F32_TOL, make_case, margin_bias, max_abs_rel, rmode, tol, to_dev)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2210_06223_b200 import build, _lib
    build.build()
    _lib.load()
    oracle.build()


import paper_2210_06223_b200 as L  # noqa: E402


# ------------------------------------------------------------------ step 1 --

MASK_CASES = [
    (1, 14, 14, 256, 2, "f32"),     # config 1
    (2, 13, 11, 64, 4, "bf16"),     # ragged: clipped edge cells
    (3, 9, 10, 128, 5, "bf16"),
    (128, 28, 28, 512, 1, "bf16"),  # config 2, every S
    (128, 28, 28, 512, 2, "bf16"),
    (128, 28, 28, 512, 4, "bf16"),
    (128, 28, 28, 512, 7, "bf16"),
]


@pytest.mark.parametrize("n,h,w,c,s,dtype", MASK_CASES)
def test_mask_bit_exact(n, h, w, c, s, dtype):
    x = synth.make_x(n, h, w, c, seed=s, dtype=dtype)
    wm = synth.make_masker_weights(c, seed=s + 10)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    bm = margin_bias(l0, 0.5)
    m_or, l_or = oracle.masker(xd, synth.to_f64(wm), bm, s)
    m, lg = L.mask(x.cuda(), wm.cuda(), bm, s, logits=True)
    m = m.cpu().numpy()
    assert np.array_equal(m, m_or)
    np.testing.assert_allclose(lg.cpu().numpy(), l_or, rtol=1e-12, atol=1e-12 * np.abs(l_or).max())
    margin = np.abs(l_or).min()
    assert margin > 1e-9 * np.abs(l_or).max()  # no cell inside the rounding band


def test_mask_all_on_all_off():
    x = synth.make_x(2, 8, 8, 64, seed=1)
    wm = synth.make_masker_weights(64, seed=2)
    assert L.mask(x.cuda(), wm.cuda(), 1e6, 2).sum().item() == 2 * 16
    assert L.mask(x.cuda(), wm.cuda(), -1e6, 2).sum().item() == 0


@pytest.mark.parametrize("n,h,w,c,s,dtype", MASK_CASES)
def test_fused_mask_compact_bit_exact(n, h, w, c, s, dtype):
    """Steps 1+2 in one launch: same mask, logits, idx and count as the oracle;
    repeated calls reuse the self-resetting workspace."""
    x = synth.make_x(n, h, w, c, seed=s + 1, dtype=dtype)
    wm = synth.make_masker_weights(c, seed=s + 11)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    blk = L.DynBlock(L.BlockShape(n, h, w, c, 64, s, torch.float32 if dtype == "f32" else torch.bfloat16),
                     synth.make_block_weights(c, 64, c, seed=1, dtype=dtype), wm, 0.0)
    xg = x.cuda()
    for r in (0.5, 0.2, 0.9):
        blk.bm = margin_bias(l0, r)
        blk.mask_compact(xg, want_logits=True)
        m_or, l_or = oracle.masker(xd, synth.to_f64(wm), blk.bm, s)
        idx_or, cnt = oracle.compact(m_or)
        assert np.array_equal(blk.mask_buf.cpu().numpy(), m_or)
        assert int(blk.count.item()) == cnt
        assert np.array_equal(blk.idx[:cnt].cpu().numpy(), idx_or)
        np.testing.assert_allclose(blk.logits.cpu().numpy(), l_or, rtol=1e-12, atol=1e-12 * np.abs(l_or).max())
    assert int(blk.mcws.count_nonzero().item()) == 0  # workspace left zeroed


STREAM_CASES = MASK_CASES + [
    (2, 13, 11, 256, 4, "bf16"),     # ragged, 1 slot per pixel
    (1, 9, 7, 2048, 3, "bf16"),      # 8 slots per pixel
    (3, 10, 12, 1024, 2, "f32"),     # fp32, 8 slots
]


@pytest.mark.parametrize("n,h,w,c,s,dtype", STREAM_CASES)
def test_mask_decisions_only_bit_exact(n, h, w, c, s, dtype):
    """Decisions without logits (the certified fp32 fast path): mask, and with
    step 2 fused idx/count, equal the fp64 oracle's bit for bit; the workspace
    is left zeroed."""
    x = synth.make_x(n, h, w, c, seed=s + 3, dtype=dtype)
    wm = synth.make_masker_weights(c, seed=s + 13)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    xg, wg = x.cuda(), wm.cuda()
    for r in (0.5, 0.1, 0.9):
        bm = margin_bias(l0, r)
        m_or, _ = oracle.masker(xd, synth.to_f64(wm), bm, s)
        idx_or, cnt = oracle.compact(m_or)
        assert np.array_equal(L.mask(xg, wg, bm, s).cpu().numpy(), m_or)
        blk = L.DynBlock(L.BlockShape(n, h, w, c, 64, s, torch.float32 if dtype == "f32" else torch.bfloat16),
                         synth.make_block_weights(c, 64, c, seed=1, dtype=dtype), wm, bm)
        blk.mask_compact(xg)
        assert np.array_equal(blk.mask_buf.cpu().numpy(), m_or)
        assert int(blk.count.item()) == cnt
        assert np.array_equal(blk.idx[:cnt].cpu().numpy(), idx_or)
        assert int(blk.mcws.count_nonzero().item()) == 0


def test_mask_decisions_only_uncertain_cells_fall_back_exactly():
    """Biases placing one cell's logit within fp32 rounding of 0: the masker's
    exact fp64 re-sum decides it as the oracle does."""
    n, h, w, c, s = 4, 12, 12, 512, 3
    x = synth.make_x(n, h, w, c, seed=21)
    wm = synth.make_masker_weights(c, seed=22)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    for k in (0, 5, 17):
        bm = float(np.float32(-l0.reshape(-1)[k]))
        m_or, l_or = oracle.masker(xd, synth.to_f64(wm), bm, s)
        if np.abs(l_or).min() < 1e-12 * np.abs(l_or).max():
            continue  # exact tie at fp64 precision
        assert np.array_equal(L.mask(x.cuda(), wm.cuda(), bm, s).cpu().numpy(), m_or)


# ------------------------------------------------------------------ step 2 --

@pytest.mark.parametrize("ncells,r", [(1, 1.0), (7, 0.5), (4095, 0.3), (4096, 0.5), (4097, 0.9),
                                      (100352, 0.5), (100352, 0.0), (100352, 1.0), (250001, 0.1)])
def test_compact_bit_exact(ncells, r):
    rng = np.random.default_rng(ncells)
    m = (rng.random(ncells) < r).astype(np.uint8)
    idx, count = L.compact(torch.from_numpy(m).cuda())
    want, wc = oracle.compact(m)
    c = int(count.item())
    assert c == wc
    assert np.array_equal(idx[:c].cpu().numpy(), want)


def test_compact_empty():
    m = torch.zeros(0, dtype=torch.uint8, device="cuda")
    idx, count = L.compact(m)
    assert int(count.item()) == 0


# ---------------------------------------------------------------- steps 3-5 --

def run_dyn(x, wts, mc, s, inplace=True):
    xd = x.cuda()
    idx, count = L.compact(torch.from_numpy(mc).cuda())
    if inplace:
        y = xd.clone()
        L.dyn_block(y, to_dev(wts), idx, count, s)
    else:
        y = torch.empty_like(xd)
        L.dyn_block(xd, to_dev(wts), idx, count, s, y=y)
    return y


DYN_CASES = [
    # n, h, w, c_in, c_mid, s, r, dtype
    (2, 14, 14, 256, 64, 2, 0.5, "bf16"),
    (2, 14, 14, 256, 64, 1, 0.3, "bf16"),
    (2, 14, 14, 256, 64, 4, 0.6, "bf16"),
    (2, 14, 14, 256, 64, 7, 0.5, "bf16"),
    (3, 13, 11, 128, 128, 3, 0.5, "bf16"),   # S not dividing H or W: clipped patches
    (2, 10, 10, 128, 64, 4, 1.0, "bf16"),
    (1, 7, 7, 512, 256, 1, 0.5, "bf16"),     # stage-4-like widths, N tile 256
    (4, 28, 28, 512, 128, 4, 0.5, "bf16"),   # config-2 shape, reduced batch
    (1, 14, 14, 256, 64, 2, 25 / 49, "f32"),  # config 1
    (2, 9, 9, 128, 64, 2, 0.5, "f32"),
]


@pytest.mark.parametrize("n,h,w,c_in,c_mid,s,r,dtype", DYN_CASES)
def test_dyn_block_matches_oracle(n, h, w, c_in, c_mid, s, r, dtype):
    x, wts, _ = make_case(n, h, w, c_in, c_mid, s, seed=n * 100 + s, dtype=dtype)
    gh, gw = L.grid(h, w, s)
    mc = synth.make_cell_mask(n, gh, gw, r, seed=s)
    y = run_dyn(x, wts, mc, s).cpu()
    idx, _ = oracle.compact(mc)
    want = oracle.dyn_block_literal(synth.to_f64(x), synth.weights_f64(wts), idx, s, rmode=rmode(dtype))
    got = synth.to_f64(y)
    up = oracle.upsample(mc, h, w, s).astype(bool)
    assert max_abs_rel(got[up], want[up]) <= tol(dtype)
    assert np.array_equal(got[~up], synth.to_f64(x)[~up])  # input fill, bitwise


def test_dyn_block_clustered_mask():
    n, h, w, s = 4, 28, 28, 4
    x, wts, _ = make_case(n, h, w, 256, 64, s, seed=7)
    mc = synth.make_cell_mask(n, 7, 7, 0.4, seed=3, family="clustered")
    y = run_dyn(x, wts, mc, s).cpu()
    want = oracle.dyn_block_def(synth.to_f64(x), synth.weights_f64(wts), mc, s)
    assert max_abs_rel(synth.to_f64(y), want) <= BF16_TOL


def test_in_place_equals_out_of_place():
    x, wts, _ = make_case(2, 14, 14, 256, 64, 2, seed=3)
    mc = synth.make_cell_mask(2, 7, 7, 0.5, seed=4)
    a = run_dyn(x, wts, mc, 2, inplace=True)
    b = run_dyn(x, wts, mc, 2, inplace=False)
    assert torch.equal(a, b)


def test_zero_mask_is_identity_bitwise():
    x, wts, _ = make_case(2, 14, 14, 256, 64, 2, seed=5)
    mc = np.zeros((2, 7, 7), np.uint8)
    y = run_dyn(x, wts, mc, 2)
    assert torch.equal(y.cpu(), x)


def test_all_ones_equals_dense_comparator():
    x, wts, _ = make_case(2, 14, 14, 256, 64, 2, seed=6)
    mc = np.ones((2, 7, 7), np.uint8)
    y = run_dyn(x, wts, mc, 2)
    yd = L.dense_block(x.cuda(), to_dev(wts))
    assert max_abs_rel(synth.to_f64(y.cpu()), synth.to_f64(yd.cpu())) <= 1e-2


def test_granularity_equivalence_on_gpu():
    """dyn(x, Mc, S) vs dyn(x, upsample(Mc, S), 1)."""
    n, h, w, s = 2, 16, 16, 4
    x, wts, _ = make_case(n, h, w, 128, 64, s, seed=8)
    mc = synth.make_cell_mask(n, 4, 4, 0.5, seed=8)
    up = oracle.upsample(mc, h, w, s)
    a = run_dyn(x, wts, mc, s)
    b = run_dyn(x, wts, up, 1)
    assert max_abs_rel(synth.to_f64(a.cpu()), synth.to_f64(b.cpu())) <= 1e-2


@pytest.mark.parametrize("n,h,w,c_in,c_mid,dtype", [(2, 14, 14, 256, 64, "bf16"), (3, 9, 7, 128, 128, "bf16"),
                                                     (1, 14, 14, 256, 64, "f32")])
def test_dense_block_matches_oracle(n, h, w, c_in, c_mid, dtype):
    x, wts, _ = make_case(n, h, w, c_in, c_mid, 1, seed=9, dtype=dtype)
    y = L.dense_block(x.cuda(), to_dev(wts)).cpu()
    want = oracle.static_block(synth.to_f64(x), synth.weights_f64(wts), rmode=rmode(dtype))
    assert max_abs_rel(synth.to_f64(y), want) <= tol(dtype)


def test_five_steps_end_to_end_masker_driven():
    """Full path with the masker deciding: mask -> compact -> dyn block."""
    n, h, w, c, s = 4, 28, 28, 256, 4
    x, wts, wm = make_case(n, h, w, c, 64, s, seed=11)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    bm = margin_bias(l0, 0.5)
    blk = L.DynBlock(L.BlockShape(n, h, w, c, 64, s), wts, wm, bm)
    y = x.cuda().clone()
    blk.forward(y)
    m_or, _ = oracle.masker(xd, synth.to_f64(wm), bm, s)
    assert np.array_equal(blk.mask_buf.cpu().numpy(), m_or)
    idx_or, cnt = oracle.compact(m_or)
    assert int(blk.count.item()) == cnt
    assert np.array_equal(blk.idx[:cnt].cpu().numpy(), idx_or)
    want = oracle.dyn_block_literal(xd, synth.weights_f64(wts), idx_or, s)
    assert max_abs_rel(synth.to_f64(y.cpu()), want) <= BF16_TOL


@pytest.mark.parametrize("s", [1, 2, 4, 7])
def test_full_size_config2_sampled(s):
    """Config 2 at full size (N=128, 28x28x512, C=128) in the launch configuration
    bench.py times; checked on sampled output pixels the oracle computes one by one."""
    n, h, w, c_in, c_mid = 128, 28, 28, 512, 128
    x, wts, wm = make_case(n, h, w, c_in, c_mid, s, seed=20 + s)
    blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), wts, wm, 0.0)
    xg = x.cuda()
    blk.calibrate_bias(xg, 0.5)
    y = xg.clone()
    blk.forward(y)
    torch.cuda.synchronize()
    mc = blk.mask_buf.cpu().numpy()
    xd = synth.to_f64(x)
    m_or, l_or = oracle.masker(xd, synth.to_f64(wm), blk.bm, s)
    assert np.array_equal(mc, m_or)
    wd = synth.weights_f64(wts)
    yc = synth.to_f64(y.cpu())
    rng = np.random.default_rng(s)
    worst = 0.0
    active = 0
    for _ in range(96):
        i, yy, xx = int(rng.integers(n)), int(rng.integers(h)), int(rng.integers(w))
        want, act = oracle.block_pixel(xd, wd, mc, s, i, yy, xx)
        if act:
            active += 1
            worst = max(worst, float(np.abs(yc[i, yy, xx] - want).max() / max(np.abs(want).max(), 1e-30)))
        else:
            assert np.array_equal(yc[i, yy, xx], xd[i, yy, xx])
    assert active > 20
    assert worst <= BF16_TOL


# ------------------------------------------- lasnet_block_forward, both schedules --

FWD_CASES = [
    # n, h, w, c_in, c_mid, s, r
    (2, 14, 14, 256, 64, 2, 0.5),
    (2, 14, 14, 256, 64, 1, 0.3),
    (3, 13, 11, 128, 128, 3, 0.5),   # clipped edge cells
    (2, 14, 14, 256, 64, 7, 0.6),
    (2, 10, 10, 128, 64, 4, 1.0),    # every cell active
    (2, 10, 10, 128, 64, 4, 0.0),    # no cell active
    (1, 7, 7, 512, 256, 1, 0.5),     # c_mid 256: unfused conv2 / conv3 kernels
    (4, 28, 28, 512, 128, 4, 0.5),   # config-2 widths, reduced batch
    (2, 56, 56, 256, 64, 4, 0.5),    # LAS-R101 stage 1 identity block (config 3), reduced batch
    (2, 14, 14, 1024, 256, 2, 0.5),  # stage 3
    (2, 7, 7, 2048, 512, 1, 0.5),    # stage 4
    (2, 19, 17, 256, 64, 5, 0.5),    # direct conv23 patches: 5 per tile, clipped edge cells
    (2, 22, 20, 256, 128, 8, 0.6),   # direct: 2 patches (128 rows) per tile
    (2, 23, 21, 256, 64, 11, 0.7),   # direct: 1 patch of 121 rows per tile
    (2, 13, 11, 256, 256, 3, 0.5),   # conv2 cp.async gather (c_mid 256): clipped cells, 14 patches per tile
    (2, 9, 9, 512, 512, 5, 0.6),     # conv2 gather at c_mid 512, 5 patches (125 rows) per tile
]


@pytest.mark.parametrize("sched", [L.SCHED_SEPARATE, L.SCHED_FUSED])
@pytest.mark.parametrize("n,h,w,c_in,c_mid,s,r", FWD_CASES)
def test_block_forward_matches_oracle(sched, n, h, w, c_in, c_mid, s, r):
    """Steps 1-5 in one call: mask/idx/count bit-exact, y within 2e-2, inactive
    pixels bitwise x -- for the north-star schedule and the paper's Table-1
    schedule (masker fused into a static conv1)."""
    x, wts, wm = make_case(n, h, w, c_in, c_mid, s, seed=n * 31 + s)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    bm = margin_bias(l0, r)
    m_or, _ = oracle.masker(xd, synth.to_f64(wm), bm, s)
    idx_or, cnt = oracle.compact(m_or)
    xg = x.cuda()
    ws = None
    for rep in range(2):  # second call: the self-resetting control words
        y, m, idx, count = L.block_forward(xg.clone(), to_dev(wts), wm.cuda(), bm, s, sched, ws=ws)
        assert np.array_equal(m.cpu().numpy(), m_or)
        assert int(count.item()) == cnt
        assert np.array_equal(idx[:cnt].cpu().numpy(), idx_or)
    want = oracle.dyn_block_literal(xd, synth.weights_f64(wts), idx_or, s)
    got = synth.to_f64(y.cpu())
    up = oracle.upsample(m_or, h, w, s).astype(bool)
    assert max_abs_rel(got[up], want[up]) <= BF16_TOL
    assert np.array_equal(got[~up], xd[~up])


def test_block_forward_fused_equals_separate_and_out_of_place():
    n, h, w, c, s = 4, 28, 28, 256, 4
    x, wts, wm = make_case(n, h, w, c, 64, s, seed=77)
    _, l0 = oracle.masker(synth.to_f64(x), synth.to_f64(wm), 0.0, s)
    bm = margin_bias(l0, 0.5)
    xg, wd, wmg = x.cuda(), to_dev(wts), wm.cuda()
    a = L.block_forward(xg.clone(), wd, wmg, bm, s, L.SCHED_SEPARATE)[0]
    b = L.block_forward(xg.clone(), wd, wmg, bm, s, L.SCHED_FUSED)[0]
    yo = torch.empty_like(xg)
    c2 = L.block_forward(xg, wd, wmg, bm, s, L.SCHED_FUSED, y=yo)[0]
    assert torch.equal(xg.cpu(), x)          # out of place leaves x untouched
    assert torch.equal(b, c2)                # in place == out of place
    assert max_abs_rel(synth.to_f64(a.cpu()), synth.to_f64(b.cpu())) <= 1e-2


def test_block_forward_fused_uncertain_cells_fall_back_exactly():
    """A masker bias placing logits right at the fp32 bound: the exact re-sum
    path decides those cells; decisions still equal the fp64 oracle's."""
    n, h, w, c, s = 2, 8, 8, 64, 2
    x, wts, wm = make_case(n, h, w, c, 64, s, seed=5)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    # bias = -(one cell's logit) rounded to fp32: that cell sits within ~1e-8 of 0
    bm = float(np.float32(-l0.reshape(-1)[3]))
    m_or, l_or = oracle.masker(xd, synth.to_f64(wm), bm, s)
    if np.abs(l_or).min() < 1e-12 * np.abs(l_or).max():
        pytest.skip("exact tie at fp64 precision")
    y, m, idx, count = L.block_forward(x.cuda(), to_dev(wts), wm.cuda(), bm, s, L.SCHED_FUSED)
    assert np.array_equal(m.cpu().numpy(), m_or)


@pytest.mark.parametrize("s", [1, 2, 4, 7])
def test_full_size_config2_fused_sampled(s):
    """Config 2 at full size through the paper's schedule (the bench launch)."""
    n, h, w, c_in, c_mid = 128, 28, 28, 512, 128
    x, wts, wm = make_case(n, h, w, c_in, c_mid, s, seed=40 + s)
    blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), wts, wm, 0.0, schedule=L.SCHED_FUSED)
    xg = x.cuda()
    blk.calibrate_bias(xg, 0.5)
    y = xg.clone()
    blk.forward(y)
    torch.cuda.synchronize()
    mc = blk.mask_buf.cpu().numpy()
    xd = synth.to_f64(x)
    m_or, _ = oracle.masker(xd, synth.to_f64(wm), blk.bm, s)
    assert np.array_equal(mc, m_or)
    idx_or, cnt = oracle.compact(m_or)
    assert int(blk.count.item()) == cnt and np.array_equal(blk.idx[:cnt].cpu().numpy(), idx_or)
    wd = synth.weights_f64(wts)
    yc = synth.to_f64(y.cpu())
    rng = np.random.default_rng(s + 100)
    worst, active = 0.0, 0
    for _ in range(96):
        i, yy, xx = int(rng.integers(n)), int(rng.integers(h)), int(rng.integers(w))
        want, act = oracle.block_pixel(xd, wd, mc, s, i, yy, xx)
        if act:
            active += 1
            worst = max(worst, float(np.abs(yc[i, yy, xx] - want).max() / max(np.abs(want).max(), 1e-30)))
        else:
            assert np.array_equal(yc[i, yy, xx], xd[i, yy, xx])
    assert active > 20
    assert worst <= BF16_TOL


@pytest.mark.parametrize("sched", [None, L.SCHED_FUSED])
def test_cuda_graph_replay_equals_eager(sched):
    """The block captured in a CUDA graph (bench.py's timed path) gives the same
    bytes as eager launches: mask, idx, count and y."""
    n, h, w, c_in, c_mid, s = 4, 28, 28, 512, 128, 4
    x, wts, wm = make_case(n, h, w, c_in, c_mid, s, seed=77)
    blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), wts, wm, 0.0, schedule=sched)
    blk.calibrate_bias(synth.make_x(n, h, w, c_in, seed=78).cuda(), 0.5)
    xg = x.cuda()
    y_e = xg.clone()
    blk.forward(y_e)
    m_e, c_e = blk.mask_buf.clone(), int(blk.count.item())
    idx_e = blk.idx[:c_e].clone()
    y_g = xg.clone()
    g = blk.capture(y_g, warmup=0)
    y_g.copy_(xg)
    blk.mask_buf.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(blk.mask_buf, m_e) and int(blk.count.item()) == c_e
    assert torch.equal(blk.idx[:c_e], idx_e)
    assert torch.equal(y_g, y_e)


@pytest.mark.parametrize("sched", [None, L.SCHED_FUSED])
def test_stream_host_pipeline_equals_per_batch_forward(sched):
    """DynBlock.stream_host (bench.py's e2e serving loop: H2D, block and D2H of
    consecutive batches overlapped on three streams, two device buffers) returns
    for every batch the same bytes as a plain forward of that batch."""
    n, h, w, c_in, c_mid, s = 4, 28, 28, 512, 128, 4
    _, wts, wm = make_case(n, h, w, c_in, c_mid, s, seed=81)
    blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), wts, wm, 0.0, schedule=sched)
    blk.calibrate_bias(synth.make_x(n, h, w, c_in, seed=82).cuda(), 0.5)
    xs = [synth.make_x(n, h, w, c_in, seed=90 + i).pin_memory() for i in range(5)]
    ys = [torch.empty_like(x).pin_memory() for x in xs]
    devs = [torch.empty_like(xs[0], device="cuda") for _ in range(2)]
    blk.stream_host(xs, ys, devs, len(xs))
    torch.cuda.synchronize()
    for x, y in zip(xs, ys):
        want = x.cuda()
        blk.forward(want)
        assert torch.equal(y, want.cpu())


def test_fused_schedule_bn256_repeated_graph_replays_stable():
    """conv1 with 256-column tiles runs 3 pipeline stages (odd): every masker warp
    must consume every stage (a K-parity split read stages before they were
    refilled -- wrong partials / faults in ~1 of 10 chained runs).  Repeated graph
    replays of chained stage-3 blocks give identical bytes, and the masks equal
    the fp64 oracle's."""
    n, h, w, c_in, c_mid, s = 32, 14, 14, 1024, 256, 2
    x = synth.make_x(n, h, w, c_in, seed=91)
    blks = []
    y = x.cuda()
    for b in range(3):
        wts = synth.make_block_weights(c_in, c_mid, c_in, seed=92 + 2 * b)
        wm = synth.make_masker_weights(c_in, seed=93 + 2 * b)
        blk = L.DynBlock(L.BlockShape(n, h, w, c_in, c_mid, s), wts, wm, 0.0, schedule=L.SCHED_FUSED)
        blk.calibrate_bias(y, 0.5)
        xin = synth.to_f64(y.cpu())
        blk.forward(y)
        m_or, _ = oracle.masker(xin, synth.to_f64(wm), blk.bm, s)
        assert np.array_equal(blk.mask_buf.cpu().numpy(), m_or)
        blks.append(blk)
    ref = y.clone()
    x0 = x.cuda()
    g = torch.cuda.CUDAGraph()
    y.copy_(x0)
    with torch.cuda.graph(g):
        for b in blks:
            b.forward(y)
    for _ in range(10):
        y.copy_(x0)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y, ref)


@pytest.mark.parametrize("env", ["LASNET_PDL=0", "LASNET_NO_FUSE=1", "LASNET_TC_PAIR=0", "LASNET_C2_GATHER=0",
                                 "LASNET_SMALL=0", "LASNET_MASK_MAXITEMS=8", "LASNET_GATHER=1",
                                 "LASNET_DECIDE_2K=1", "LASNET_C23_BALANCE=0", "LASNET_TMA_Y=0"])
def test_library_variants(env):
    """The opt-in library variants (read once per process: run in a subprocess)
    give oracle-exact masks/idx and in-tolerance activations for both schedules
    and the dense comparator."""
    import os
    import subprocess
    import sys

    k, v = env.split("=")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "variant_check.py")], env=dict(os.environ, **{k: v}),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("sched", [L.SCHED_SEPARATE, L.SCHED_FUSED])
def test_batch_sharding_is_bitwise_invariant(sched):
    """images are independent, so running a batch split over two
    'ranks' (two calls on halves) gives the same bytes as one call on the whole
    batch -- the data-parallel sharding of bench.py --gpus N changes nothing."""
    n, h, w, c_in, c_mid, s = 8, 28, 28, 512, 128, 4
    x, wts, wm = make_case(n, h, w, c_in, c_mid, s, seed=33)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    bm = margin_bias(l0, 0.5)
    y_all, m_all, _, _ = L.block_forward(x.cuda(), to_dev(wts), wm.cuda(), bm, s, sched)
    for lo, hi in ((0, 3), (3, 8)):
        y_p, m_p, _, _ = L.block_forward(x[lo:hi].contiguous().cuda(), to_dev(wts), wm.cuda(), bm, s, sched)
        assert torch.equal(m_p, m_all[lo:hi])
        assert torch.equal(y_p, y_all[lo:hi])


PROJ_CASES = [
    # n, h_in, c_in, c_mid, c_out, stride  (LAS-R101 first blocks, reduced batch/size)
    (2, 14, 64, 64, 256, 1),     # stage 1 (stride 1, 64 -> 256)
    (2, 14, 256, 128, 512, 2),   # stage 2
    (2, 14, 512, 256, 1024, 2),  # stage 3 (c_mid 256: conv1 with 256-column tiles)
    (3, 8, 128, 64, 128, 2),
    (1, 14, 1024, 512, 2048, 2),  # stage 4
]


@pytest.mark.parametrize("n,h,c_in,c_mid,c_out,stride", PROJ_CASES)
def test_proj_block_matches_oracle(n, h, c_in, c_mid, c_out, stride):
    """Static projection (first) block through lasnet_proj_block vs the fp64 oracle
    with the same storage roundings."""
    x = synth.make_x(n, h, h, c_in, seed=h + stride)
    wts = synth.make_proj_weights(c_in, c_mid, c_out, seed=7)
    y = L.proj_block(x.cuda(), to_dev(wts), stride)
    want = oracle.proj_block(synth.to_f64(x), synth.weights_f64(wts), stride)
    got = synth.to_f64(y.cpu())
    assert got.shape == want.shape
    assert max_abs_rel(got, want) <= BF16_TOL


PROJ_DYN_CASES = [
    # n, h_in, w_in, c_in, c_mid, c_out, stride, s, r   (LAS-R101 first blocks, reduced batch; ragged grids)
    (2, 16, 16, 64, 64, 256, 1, 4, 0.5),      # stage 1 (stride 1, 64 -> 256, fused conv23)
    (2, 28, 28, 256, 128, 512, 2, 4, 0.5),    # stage 2 (stride 2, fused conv23 over parity views)
    (2, 28, 28, 512, 256, 1024, 2, 2, 0.5),   # stage 3 (c_mid 256: unfused conv2 / conv3)
    (1, 14, 14, 1024, 512, 2048, 2, 1, 0.5),  # stage 4 (S = 1)
    (2, 20, 26, 128, 64, 256, 2, 3, 0.6),     # S does not divide the 10 x 13 output: clipped cells
    (2, 16, 16, 128, 128, 256, 2, 4, 1.0),    # every cell active
    (2, 16, 16, 128, 128, 256, 2, 4, 0.0),    # none active: y = ReLU(R)
    (8, 56, 56, 256, 128, 512, 2, 4, 0.5),    # multi-round persistent tiles
]


@pytest.mark.parametrize("n,hi,wi,c_in,c_mid,c_out,stride,s,r", PROJ_DYN_CASES)
def test_proj_dyn_block_matches_oracle(n, hi, wi, c_in, c_mid, c_out, stride, s, r):
    """The dynamic first block (NEXT-f1, reading R22) through lasnet_block_forward
    with the shortcut weights: mask / idx / count bit-exact vs the oracle masker at
    granularity stride*S on the input, y vs the literal oracle (active pixels
    ReLU(R + F), the others ReLU(R)) within 2e-2; signed input."""
    x = synth.make_x(n, hi, wi, c_in, seed=hi + s, relu=False)
    wts = synth.make_proj_weights(c_in, c_mid, c_out, seed=7 + s)
    wm = synth.make_masker_weights(c_in, seed=8 + s)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s * stride)
    bm = margin_bias(l0, r)
    m_or, _ = oracle.masker(xd, synth.to_f64(wm), bm, s * stride)
    idx_or, cnt = oracle.compact(m_or)
    y, m, idx, count = L.proj_block_forward(x.cuda(), to_dev(wts), wm.cuda(), bm, s, stride)
    assert np.array_equal(m.cpu().numpy(), m_or)
    assert int(count.item()) == cnt and np.array_equal(idx[:cnt].cpu().numpy(), idx_or)
    want = oracle.proj_dyn_literal(xd, synth.weights_f64(wts), idx_or, s, stride)
    got = synth.to_f64(y.cpu())
    assert got.shape == want.shape
    assert max_abs_rel(got, want) <= BF16_TOL


@pytest.mark.parametrize("n,h,w", [(2, 16, 24), (1, 32, 16), (2, 224, 224), (1, 32, 672)])
def test_stem_maxpool_head_match_oracle(n, h, w):
    """Stem (tcgen05, 7x7 stride 2 over 4 column-residue window views), max pool and
    head against the fp64 oracle; the 224x224 case is the ImageNet stem."""
    g = torch.Generator().manual_seed(n + h)
    x = torch.randn((n, h, w, 8), generator=g).clamp(-3, 3)
    x[..., 3:] = 0.0
    x = x.to(torch.bfloat16)
    wt = (torch.randn((64, 7, 7, 8), generator=g) * 0.1)
    wt[..., 3:] = 0.0
    wt = wt.to(torch.bfloat16)
    b = (torch.randn((64,), generator=g) * 0.1).float()
    x_pad = torch.zeros((n, h, w + 8, 8), dtype=torch.bfloat16)
    x_pad[:, :, 4:4 + w] = x
    y = L.stem(x_pad.cuda(), wt.cuda(), b.cuda())
    want = oracle.stem(synth.to_f64(x), synth.to_f64(wt), synth.to_f64(b))
    got = synth.to_f64(y.cpu())
    assert max_abs_rel(got, want) <= BF16_TOL
    mp = L.maxpool(y)
    assert np.array_equal(synth.to_f64(mp.cpu()), oracle.maxpool(got))  # exact on the same input
    wf = (torch.randn((1000, 64), generator=g) * 0.1).to(torch.bfloat16)
    bf = (torch.randn((1000,), generator=g) * 0.1).float()
    lg = L.head(mp, wf.cuda(), bf.cuda()).cpu().numpy()
    want_lg = oracle.head(synth.to_f64(mp.cpu()), synth.to_f64(wf), synth.to_f64(bf))
    assert np.abs(lg - want_lg).max() <= 1e-4 * max(1.0, np.abs(want_lg).max())


NET_CASES = [
    # n, hw, s_net, backbone
    (2, 64, (4, 4, 2, 1), False),
    (4, 224, (4, 4, 2, 1), False),          # the measured ImageNet shape (configs[2])
    (1, (256, 672), (4, 4, 2, 1), True),     # COCO-shaped backbone (configs[4]): W = 168 > 128 at stage 1
    (1, (256, 672), (4, 4, 7, 1), True),     # S_net 4-4-7-1: clipped S = 7 cells on 16 x 42
]


@pytest.mark.parametrize("n,hw,s_net,backbone", NET_CASES)
def test_lasnet_network_layerwise_matches_oracle(n, hw, s_net, backbone):
    """LAS-ResNet-101 run layer by layer through the library (64x64: stages of
    16/8/4/2 px; 224x224: the measured ImageNet shape, stages 56/28/14/7 px,
    multi-round persistent tiles; 256x672: a COCO-shaped backbone with
    column-blocked dense tiles and clipped cells); each layer's output is checked
    against the fp64 oracle applied to the same GPU input (teacher forcing): stem,
    pool, every first block (dynamic: mask bit-exact), every dynamic block (mask
    bit-exact, activations in tolerance, inactive pixels bitwise), head; then the
    oracle's own end-to-end forward (oracle.lasnet_forward with the GPU network's
    masker biases and decisions) against the GPU logits / stage outputs."""
    H, W = (hw, hw) if isinstance(hw, int) else hw
    wts = synth.make_lasnet_weights(seed=5)
    net = L.LASResNet(n, wts, hw=hw, s_net=s_net, backbone=backbone)
    x = synth.make_image_batch(n, hw, seed=6).cuda()
    net.forward(synth.make_image_batch(n, hw, seed=7).cuda(), calibrate_r=0.5)  # biases from a separate batch
    torch.cuda.synchronize()
    y = L.stem(x, net.stem_w, net.stem_b)
    xin = synth.to_f64(x.cpu())[:, :, 4:4 + W, :]
    assert max_abs_rel(synth.to_f64(y.cpu()), oracle.stem(xin, synth.to_f64(net.stem_w.cpu()),
                                                           synth.to_f64(net.stem_b.cpu()))) <= BF16_TOL
    p = L.maxpool(y)
    assert np.array_equal(synth.to_f64(p.cpu()), oracle.maxpool(synth.to_f64(y.cpu())))
    cur = p
    for si, (proj, dyn) in enumerate(net.stages):
        xin = synth.to_f64(cur.cpu())
        out = proj.forward(cur)
        stride = 1 if si == 0 else 2
        if getattr(proj, "dynamic", False):  # the dynamic first block (reading R22)
            m_or, _ = oracle.masker(xin, synth.to_f64(proj.wm.cpu()), proj.bm, proj.s * stride)
            assert np.array_equal(proj.mask_buf.cpu().numpy(), m_or), f"stage {si} projection mask"
            idx_or, cnt = oracle.compact(m_or)
            assert int(proj.count.item()) == cnt
            want = oracle.proj_dyn_literal(xin, synth.weights_f64(proj.wts), idx_or, proj.s, stride)
        else:
            want = oracle.proj_block(xin, synth.weights_f64(proj.wts), stride)
        assert max_abs_rel(synth.to_f64(out.cpu()), want) <= BF16_TOL, f"stage {si} projection"
        for bi, blk in enumerate(dyn):
            xin = synth.to_f64(out.cpu())
            blk.forward(out)
            m_or, _ = oracle.masker(xin, synth.to_f64(blk.wm.cpu()), blk.bm, blk.shape.s)
            assert np.array_equal(blk.mask_buf.cpu().numpy(), m_or), f"stage {si} block {bi} mask"
            idx_or, cnt = oracle.compact(m_or)
            assert int(blk.count.item()) == cnt, f"stage {si} block {bi} count"
            want = oracle.dyn_block_literal(xin, synth.weights_f64({k: v.cpu() for k, v in blk.wts.items()}), idx_or,
                                            blk.shape.s)
            got = synth.to_f64(out.cpu())
            up = oracle.upsample(m_or, blk.shape.h, blk.shape.w, blk.shape.s).astype(bool)
            assert max_abs_rel(got[up], want[up]) <= BF16_TOL, f"stage {si} block {bi}"
            assert np.array_equal(got[~up], xin[~up]), f"stage {si} block {bi} inactive pixels"
        cur = out
    if not backbone:
        lg = L.head(cur, net.fc_w, net.fc_b).cpu().numpy()
        want_lg = oracle.head(synth.to_f64(cur.cpu()), synth.to_f64(net.fc_w.cpu()), synth.to_f64(net.fc_b.cpu()))
        assert np.abs(lg - want_lg).max() <= 1e-4 * max(1.0, np.abs(want_lg).max())
    # the captured graph reproduces the eager forward
    out_eager = net.forward(x)
    out_eager = [t.clone() for t in out_eager] if backbone else out_eager.clone()
    g = net.capture(x)
    g.replay()
    torch.cuda.synchronize()
    if backbone:
        assert all(torch.equal(a, b) for a, b in zip(net.features, out_eager))
    else:
        assert torch.equal(net.logits, out_eager)
    # end to end: the oracle's own forward from the image with the same masker biases, following the
    # GPU network's decisions (force_masks) so that one 1-ulp bf16 difference upstream cannot flip a
    # near-threshold cell and diverge the two chains; its own (free-running) decisions are counted
    meta = net.oracle_meta()
    keys = sorted(meta["bm"], key=_block_order)
    gpu_masks = {k: b.mask_buf.cpu().numpy() for k, b in zip(keys, net.blocks())}
    want_e2e, masks = oracle.lasnet_forward(xin_img(x, W), synth.weights_f64_nested(wts), meta, return_masks=True,
                                            force_masks=gpu_masks, backbone=backbone)
    diff_cells = sum(int((masks[k] != gpu_masks[k]).sum()) for k in keys)
    total_cells = sum(b.ncells for b in net.blocks())
    # free-running decisions of the fp64 chain agree on >= 99% of the cells
    assert diff_cells <= max(1, total_cells // 100), f"{diff_cells} of {total_cells} decisions differ end to end"
    if backbone:
        for si, (a, b) in enumerate(zip(out_eager, want_e2e)):
            assert max_abs_rel(synth.to_f64(a.cpu()), b) <= BF16_TOL, f"stage {si} features"
    else:
        assert max_abs_rel(out_eager.cpu().numpy(), want_e2e) <= BF16_TOL


def xin_img(x, hw):
    return synth.to_f64(x.cpu())[:, :, 4:4 + hw, :]


def _block_order(key):
    si, b = key[1:].split("_")
    return int(si), 0 if b == "proj" else int(b[1:])


def test_network_batch_sharding_is_bitwise_invariant():
    """sharding the global batch over ranks changes nothing -- the logits
    of two half-batch networks (what two ranks compute before the all-gather) equal
    the whole-batch network's bit for bit, with the same masker biases."""
    wts = synth.make_lasnet_weights(seed=9)
    x = synth.make_image_batch(4, 64, seed=10).cuda()
    full = L.LASResNet(4, wts, hw=64)
    full.forward(synth.make_image_batch(4, 64, seed=11).cuda(), calibrate_r=0.5)
    lg_full = full.forward(x).clone()
    parts = []
    for lo, hi in ((0, 2), (2, 4)):
        half = L.LASResNet(2, wts, hw=64)
        for a, b in zip(half.blocks(), full.blocks()):
            a.bm = b.bm
        parts.append(half.forward(x[lo:hi].contiguous()).clone())
    assert torch.equal(torch.cat(parts), lg_full)


# ------------------------- single-launch fp32 small-batch block (small_block.cu) --

SMALL_CASES = [
    # n, h, w, c, c_mid, s, r
    (1, 14, 14, 256, 64, 2, 25 / 49),  # config 1
    (2, 13, 11, 128, 64, 3, 0.5),      # clipped edge cells
    (3, 9, 9, 128, 64, 1, 0.4),        # S = 1: pixel-level
    (1, 14, 14, 256, 64, 4, 1.0),      # every cell active
    (1, 14, 14, 256, 64, 2, 0.0),      # no cell active
    (4, 14, 14, 64, 64, 7, 0.5),       # narrow widths
]


@pytest.mark.parametrize("n,h,w,c,c_mid,s,r", SMALL_CASES)
def test_small_block_matches_oracle(n, h, w, c, c_mid, s, r):
    """fp32 small batches run the whole block as ONE cooperative launch (masker,
    compaction, conv1 once per pixel of the dilated union of the active cells,
    conv2, conv3 + scatter-add): mask/idx/count bit-exact, y within 1e-5, inactive
    pixels bitwise x; the dense comparator likewise against the static block."""
    x, wts, wm = make_case(n, h, w, c, c_mid, s, seed=900 + n + s, dtype="f32")
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    bm = margin_bias(l0, r)
    m_or, _ = oracle.masker(xd, synth.to_f64(wm), bm, s)
    idx_or, cnt = oracle.compact(m_or)
    xg, wd = x.cuda(), to_dev(wts)
    import ctypes
    from paper_2210_06223_b200 import _lib
    d = L.make_desc(n, h, w, c, c_mid, c, s, torch.float32)
    ws = torch.zeros(_lib.load().lasnet_block_forward_workspace_bytes(ctypes.byref(d), L.SCHED_SEPARATE),
                     dtype=torch.uint8, device="cuda")
    for rep in range(3):  # repeated calls on one workspace: the barrier words are left zero
        y, m, idx, count = L.block_forward(xg.clone(), wd, wm.cuda(), bm, s, L.SCHED_SEPARATE, ws=ws)
        assert L.last_launch_count() == 1
        assert np.array_equal(m.cpu().numpy(), m_or)
        assert int(count.item()) == cnt
        assert np.array_equal(idx[:cnt].cpu().numpy(), idx_or)
    want = oracle.dyn_block_literal(xd, synth.weights_f64(wts), idx_or, s, rmode=oracle.ROUND_F32)
    got = synth.to_f64(y.cpu())
    up = oracle.upsample(m_or, h, w, s).astype(bool)
    if up.any():
        assert max_abs_rel(got[up], want[up]) <= 1e-5
    assert np.array_equal(got[~up], xd[~up])
    yd = L.dense_block(xg, wd)
    assert L.last_launch_count() == 1
    wdense = oracle.static_block(xd, synth.weights_f64(wts), rmode=oracle.ROUND_F32)
    assert max_abs_rel(synth.to_f64(yd.cpu()), wdense) <= 1e-5


def test_maxpool_odd_output_and_head_ragged_shapes():
    """The 2 x 2-block max pool at odd output sizes (a block's second row / column past the
    edge), exact vs the oracle; the tensor-core head at ragged shapes (images not a multiple of
    16, classes not a multiple of 32, c % 16 == 8: the last K-step half-empty) within 1e-4."""
    g = torch.Generator().manual_seed(77)
    for (n, ho, wo, c) in [(1, 7, 9, 64), (3, 5, 3, 16), (2, 1, 1, 8)]:
        x = torch.randn((n, 2 * ho, 2 * wo, c), generator=g).to(torch.bfloat16)
        got = synth.to_f64(L.maxpool(x.cuda()).cpu())
        assert np.array_equal(got, oracle.maxpool(synth.to_f64(x))), (n, ho, wo, c)
    for (n, hw, c, classes) in [(5, 9, 72, 37), (17, 4, 24, 100), (1, 1, 8, 1)]:
        x = torch.randn((n, hw, 1, c), generator=g).abs().to(torch.bfloat16)
        wf = (torch.randn((classes, c), generator=g) * 0.1).to(torch.bfloat16)
        bf = (torch.randn((classes,), generator=g) * 0.1).float()
        lg = L.head(x.cuda(), wf.cuda(), bf.cuda()).cpu().numpy()
        want = oracle.head(synth.to_f64(x), synth.to_f64(wf), synth.to_f64(bf))
        assert np.abs(lg - want).max() <= 1e-4 * max(1.0, np.abs(want).max()), (n, hw, c, classes)
