"""LAS-RegNetY on the GPU vs the fp64 oracle (-m gpu):
the Y-block (grouped 3x3 on mma.sync, SE pooled over the active pixels =
reading R23, conv3 + scatter-add), dynamic and static, identity and stride-2
projection, the RegNet stem, and the whole LAS-RegNetY-800MF layer by layer.
Masks / idx / counts bit-exact; activations max-abs-rel <= 2e-2; inactive
pixels bitwise x."""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import BF16_TOL, margin_bias, max_abs_rel

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


def block_case(n, h, w, c_real, w_se, seed, proj=False, c_in_real=None):
    wts = synth.make_regnet_block_weights(c_in_real or c_real, c_real, w_se, proj, seed)
    c_in = synth.pad64(c_in_real or c_real)
    x = torch.zeros((n, h, w, c_in), dtype=torch.bfloat16)
    x[..., :c_in_real or c_real] = synth.make_x(n, h, w, c_in_real or c_real, seed=seed + 1)
    return x, wts


DYN_CASES = [
    # n, h, w, c_real, w_se, s, r
    (2, 14, 14, 144, 36, 2, 0.5),    # stage 2 (padded to 192), S = 2
    (2, 28, 28, 144, 36, 4, 0.5),
    (4, 14, 14, 320, 80, 2, 0.5),    # stage 3 (320: a partial masker slot)
    (2, 7, 7, 784, 196, 1, 0.5),     # stage 4 (padded to 832)
    (2, 13, 11, 64, 16, 3, 0.6),     # ragged grid, clipped cells
    (3, 14, 14, 144, 36, 2, 1.0),    # every cell active
    (2, 14, 14, 144, 36, 2, 0.0),    # none active
    (32, 14, 14, 320, 80, 2, 0.5),   # many patches (multi-round tiles)
]


@pytest.mark.parametrize("sched", [L.SCHED_SEPARATE, L.SCHED_FUSED])
@pytest.mark.parametrize("n,h,w,c,w_se,s,r", DYN_CASES)
def test_regnet_dynamic_block_matches_oracle(n, h, w, c, w_se, s, r, sched):
    x, wts = block_case(n, h, w, c, w_se, seed=h + c + s)
    xd = synth.to_f64(x)
    wm = wts["wm"]
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    bm = margin_bias(l0, r)
    m_or, _ = oracle.masker(xd, synth.to_f64(wm), bm, s)
    idx_or, cnt = oracle.compact(m_or)
    blk = L.RegNetBlock(n, h, w, x.shape[-1], x.shape[-1], 1, wts, s=s, dynamic=True, schedule=sched)
    blk.bm = bm
    for rep in range(2):  # second call: the self-resetting control words
        y = x.cuda()
        blk.forward(y)
    torch.cuda.synchronize()
    assert np.array_equal(blk.mask_buf.cpu().numpy(), m_or)
    assert int(blk.count.item()) == cnt and np.array_equal(blk.idx[:cnt].cpu().numpy(), idx_or)
    want = oracle.regnet_block(xd, synth.weights_f64(wts), 1, mask_cells=m_or, s=s)
    got = synth.to_f64(y.cpu())
    up = oracle.upsample(m_or, h, w, s).astype(bool)
    if up.any():
        assert max_abs_rel(got[up], want[up]) <= BF16_TOL
    assert np.array_equal(got[~up], xd[~up])


@pytest.mark.parametrize("n,h,c_in,c_out,w_se,stride", [(2, 16, 32, 64, 8, 2), (2, 28, 64, 144, 16, 2),
                                                        (2, 14, 144, 320, 36, 2), (2, 14, 320, 784, 80, 2),
                                                        (2, 14, 144, 144, 36, 1)])
def test_regnet_static_block_matches_oracle(n, h, c_in, c_out, w_se, stride):
    proj = c_in != c_out or stride != 1
    x, wts = block_case(n, h, h, c_out, w_se, seed=h + c_in, proj=proj, c_in_real=c_in)
    blk = L.RegNetBlock(n, h, h, x.shape[-1], synth.pad64(c_out), stride, wts)
    y = blk.forward(x.cuda())
    want = oracle.regnet_block(synth.to_f64(x), synth.weights_f64(wts), stride)
    assert max_abs_rel(synth.to_f64(y.cpu()), want) <= BF16_TOL


def test_regnet_stem_matches_oracle():
    w = synth.make_regnet_weights()
    x = synth.make_image_batch(2, (32, 48), seed=3)
    net_y = torch.empty((2, 16, 24, 64), dtype=torch.bfloat16, device="cuda")
    lib = L._lib.load()
    from paper_2210_06223_b200.block import _p, _stream
    xg, wg, bg = x.cuda(), w["stem_w"].cuda(), w["stem_b"].cuda()  # kept alive until the kernel has run
    L._lib.check("stem", lib.lasnet_regnet_stem(2, 16, 24, 32, _p(xg), _p(wg), _p(bg), _p(net_y), _stream()))
    torch.cuda.synchronize()
    want = oracle.regnet_stem(synth.to_f64(x)[:, :, 4:52, :], synth.to_f64(w["stem_w"]), synth.to_f64(w["stem_b"]))
    assert max_abs_rel(synth.to_f64(net_y.cpu()), want) <= BF16_TOL
    assert torch.count_nonzero(net_y[..., 32:]) == 0


@pytest.mark.parametrize("n,hw", [(2, 64), (2, 224)])
def test_las_regnet_layerwise_matches_oracle(n, hw):
    """LAS-RegNetY-800MF layer by layer (teacher forcing: the oracle on each layer's
    GPU input), then the oracle's own forward with the GPU's decisions vs the logits."""
    wts = synth.make_regnet_weights(seed=5)
    net = L.LASRegNet(n, wts, hw=hw)
    x = synth.make_image_batch(n, hw, seed=6).cuda()
    net.forward(synth.make_image_batch(n, hw, seed=7).cuda(), calibrate_r=0.5)
    torch.cuda.synchronize()
    lib = L._lib.load()
    from paper_2210_06223_b200.block import _p, _stream
    stem = torch.empty_like(net.stem_y)
    L._lib.check("stem", lib.lasnet_regnet_stem(n, hw // 2, hw // 2, 32, _p(x), _p(net.stem_w), _p(net.stem_b),
                                                 _p(stem), _stream()))
    xin = synth.to_f64(x.cpu())[:, :, 4:4 + hw, :]
    assert max_abs_rel(synth.to_f64(stem.cpu()),
                       oracle.regnet_stem(xin, synth.to_f64(net.stem_w.cpu()), synth.to_f64(net.stem_b.cpu()))) <= BF16_TOL
    cur = stem
    for si, (first, dyn) in enumerate(net.stages):
        xin = synth.to_f64(cur.cpu())
        out = first.forward(cur)
        want = oracle.regnet_block(xin, synth.weights_f64({k: v.cpu() for k, v in first.wts.items()}), 2)
        assert max_abs_rel(synth.to_f64(out.cpu()), want) <= BF16_TOL, f"stage {si} first block"
        for bi, blk in enumerate(dyn):
            xin = synth.to_f64(out.cpu())
            blk.forward(out)
            m_or, _ = oracle.masker(xin, synth.to_f64(blk.wm.cpu()), blk.bm, blk.s)
            assert np.array_equal(blk.mask_buf.cpu().numpy(), m_or), f"stage {si} block {bi} mask"
            want = oracle.regnet_block(xin, synth.weights_f64({k: v.cpu() for k, v in blk.wts.items()}), 1,
                                       mask_cells=m_or, s=blk.s)
            got = synth.to_f64(out.cpu())
            up = oracle.upsample(m_or, blk.h, blk.w, blk.s).astype(bool)
            assert max_abs_rel(got[up], want[up]) <= BF16_TOL, f"stage {si} block {bi}"
            assert np.array_equal(got[~up], xin[~up])
        cur = out
    lg = net.forward(x).clone()
    g = net.capture(x)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(net.logits, lg)
    meta = net.oracle_meta()
    gpu_masks = {f"s{si}_b{bi + 1}": b.mask_buf.cpu().numpy() for si, (_, dyn) in enumerate(net.stages)
                 for bi, b in enumerate(dyn)}
    want, masks = oracle.regnet_forward(xin_img(x, hw), synth.weights_f64_nested(wts), meta, force_masks=gpu_masks,
                                        return_masks=True)
    diff = sum(int((masks[k] != gpu_masks[k]).sum()) for k in gpu_masks)
    total = sum(b.ncells for b in net.blocks())
    assert diff <= max(1, total // 100)
    assert max_abs_rel(lg.cpu().numpy(), want) <= BF16_TOL


def xin_img(x, hw):
    return synth.to_f64(x.cpu())[:, :, 4:4 + hw, :]
