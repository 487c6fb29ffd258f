"""Pins of the LAS-RegNetY oracle (oracle.gconv3x3 / se_scale / regnet_block /
regnet_block_literal / regnet_stem) against things other
than itself: float64 torch.nn.functional.conv2d with groups (library routine),
the SE closed form, the masked-select definition vs the two-pass literal loops,
and the zero-padded widths vs the real widths.  -m "not gpu"."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth


def real_block(c_in, w_out, w_se, proj, seed):
    w = synth.make_regnet_block_weights(c_in, w_out, w_se, proj, seed)
    return {k: synth.to_f64(v) for k, v in w.items()}


def torch_block(x, f, stride, w_out, c_in):
    """The Y-block at REAL widths from float64 torch ops (conv2d groups, mean, sigmoid)."""
    xt = torch.from_numpy(x[..., :c_in]).permute(0, 3, 1, 2)
    T = {k: torch.from_numpy(v) for k, v in f.items()}
    wa = T["wa"][:w_out, :c_in, None, None]
    h1 = F.relu(F.conv2d(xt, wa, T["ba"][:w_out]))
    wb = T["wb"][:w_out].permute(0, 3, 1, 2)  # [out][16][3][3]
    h2 = F.relu(F.conv2d(h1, wb, T["bb"][:w_out], stride=stride, padding=1, groups=w_out // 16))
    p = h2.mean(dim=(2, 3))
    z = F.relu(p @ T["se_w1"][:, :w_out].T + T["se_b1"])
    s = torch.sigmoid(z @ T["se_w2"][:w_out].T + T["se_b2"][:w_out])
    h2s = h2 * s[:, :, None, None]
    c = F.conv2d(h2s, T["wc"][:w_out, :w_out, None, None], T["bc"][:w_out])
    if "wd" in T:
        R = F.conv2d(xt, T["wd"][:w_out, :c_in, None, None], T["bd"][:w_out], stride=stride)
    else:
        R = xt
    return F.relu(R + c).permute(0, 2, 3, 1).numpy()


@pytest.mark.parametrize("stride", [1, 2])
def test_gconv_equals_torch_grouped_conv2d(oracle_mod, stride):
    g = torch.Generator().manual_seed(stride)
    h = torch.randn((2, 9, 7, 48), generator=g, dtype=torch.float64)
    w = torch.randn((48, 3, 3, 16), generator=g, dtype=torch.float64)
    b = torch.randn((48,), generator=g, dtype=torch.float64)
    got = oracle_mod.gconv3x3(h.numpy(), w.numpy(), b.numpy(), stride)
    want = F.conv2d(h.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), b, stride=stride, padding=1, groups=3)
    assert np.abs(got - want.permute(0, 2, 3, 1).numpy()).max() < 1e-12


@pytest.mark.parametrize("c_in,w_out,w_se,proj,stride", [(64, 64, 16, False, 1), (144, 144, 36, False, 1),
                                                          (64, 144, 16, True, 2), (32, 64, 8, True, 2)])
def test_regnet_block_equals_torch_at_real_widths(oracle_mod, c_in, w_out, w_se, proj, stride):
    """Static Y-block, unrounded, padded widths (zero channels) == the real-width block
    built from torch conv2d(groups) + SE: the padding changes nothing."""
    f = real_block(c_in, w_out, w_se, proj, seed=c_in + w_out)
    ci = synth.pad64(c_in)
    x = np.zeros((2, 8, 10, ci))
    x[..., :c_in] = synth.to_f64(synth.make_x(2, 8, 10, c_in, seed=3))
    got = oracle_mod.regnet_block(x, f, stride, rmode=oracle_mod.ROUND_NONE)
    want = torch_block(x, f, stride, w_out, c_in)
    assert np.abs(got[..., :w_out] - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
    assert np.all(got[..., w_out:] == 0.0)


def test_se_closed_form(oracle_mod):
    """se_w1 = 0, se_b1 = 0 -> z = 0 -> s = sigmoid(se_b2) whatever the pooled input."""
    f = real_block(64, 64, 16, False, seed=5)
    f["se_w1"][:] = 0.0
    f["se_b1"][:] = 0.0
    s = oracle_mod.se_scale(np.random.default_rng(0).standard_normal((3, 64)), f)
    assert np.allclose(s, 1.0 / (1.0 + np.exp(-f["se_b2"]))[None, :], rtol=0, atol=1e-15)


def test_dynamic_all_ones_is_static_and_all_zeros_is_identity(oracle_mod):
    f = real_block(64, 64, 16, False, seed=7)
    x = synth.to_f64(synth.make_x(2, 8, 8, 64, seed=8))
    ones = np.ones((2, 4, 4), np.uint8)
    assert np.array_equal(oracle_mod.regnet_block(x, f, 1, mask_cells=ones, s=2), oracle_mod.regnet_block(x, f, 1))
    zeros = np.zeros((2, 4, 4), np.uint8)
    assert np.array_equal(oracle_mod.regnet_block(x, f, 1, mask_cells=zeros, s=2), x)


@pytest.mark.parametrize("h,w,s", [(8, 8, 2), (7, 9, 3), (6, 6, 1)])
def test_literal_equals_definition(oracle_mod, h, w, s):
    """Two-pass literal loops (gather, conv, SE pooled over the ACTIVE pixels, scatter)
    == the masked-select definition (reading R23), exactly in fp64 and with bf16
    storage rounding (the same roundings at the same points)."""
    f = real_block(32 if False else 64, 64, 16, False, seed=h + w + s)
    x = synth.to_f64(synth.make_x(2, h, w, 64, seed=s))
    gh, gw = -(-h // s), -(-w // s)
    mc = synth.make_cell_mask(2, gh, gw, 0.5, seed=s)
    idx, _ = oracle_mod.compact(mc)
    for rm in (oracle_mod.ROUND_NONE, oracle_mod.ROUND_BF16):
        a = oracle_mod.regnet_block_literal(x, f, idx, s, rmode=rm)
        b = oracle_mod.regnet_block(x, f, 1, mask_cells=mc, s=s, rmode=rm)
        if rm == oracle_mod.ROUND_NONE:
            assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()
        else:
            assert np.mean(a == b) > 0.999 and np.abs(a - b).max() <= 2 ** -7 * np.abs(b).max()


def test_se_pools_only_active_pixels(oracle_mod):
    """Changing x only inside INACTIVE cells (away from the active cells' halos)
    leaves the active outputs unchanged: the SE mean is over active pixels only."""
    f = real_block(64, 64, 16, False, seed=11)
    x = synth.to_f64(synth.make_x(1, 12, 12, 64, seed=12))
    mc = np.zeros((1, 6, 6), np.uint8)
    mc[0, 0, 0] = 1
    y0 = oracle_mod.regnet_block(x, f, 1, mask_cells=mc, s=2)
    x2 = x.copy()
    x2[0, 8:, 8:, :] += 1.0
    y1 = oracle_mod.regnet_block(x2, f, 1, mask_cells=mc, s=2)
    assert np.array_equal(y0[0, :2, :2], y1[0, :2, :2])


def test_regnet_stem_equals_torch(oracle_mod):
    g = torch.Generator().manual_seed(0)
    x = torch.randn((2, 16, 24, 8), generator=g, dtype=torch.float64)
    x[..., 3:] = 0
    w = torch.randn((64, 3, 3, 8), generator=g, dtype=torch.float64)
    b = torch.randn((64,), generator=g, dtype=torch.float64)
    got = oracle_mod.regnet_stem(x.numpy(), w.numpy(), b.numpy(), rmode=oracle_mod.ROUND_NONE)
    want = F.relu(F.conv2d(x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), b, stride=2, padding=1))
    assert np.abs(got - want.permute(0, 2, 3, 1).numpy()).max() < 1e-12
