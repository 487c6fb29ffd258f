"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and host-side validation rejects bad arguments before any
CUDA call (nothing is launched on error, include/lasnet.h)."""
import ctypes
import os
import re

import pytest

from paper_2210_06223_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lasnet.h")).read()
    return sorted(set(re.findall(r"\b(lasnet_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_status_strings_and_version(lib):
    assert lib.lasnet_abi_version() == 2
    for code, name in _lib.STATUS.items():
        assert lib.lasnet_status_str(code).decode().startswith(name)


def desc(**kw):
    d = dict(n=2, h=14, w=14, c_in=256, c_mid=64, c_out=256, stride=1, s=2, dtype=_lib.LASNET_BF16)
    d.update(kw)
    return _lib.BlockDesc(*(d[k] for k in ("n", "h", "w", "c_in", "c_mid", "c_out", "stride", "s", "dtype")))


def test_workspace_sizes_are_pure_host_math(lib):
    d = desc()
    cap = 2 * 7 * 7
    # h1 [cap][(S+2)^2][c_mid] + h2 [cap][S^2][c_mid], bf16, 256-B aligned
    want = lambda b: (b + 255) // 256 * 256
    assert lib.lasnet_dyn_workspace_bytes(ctypes.byref(d), cap) == want(cap * 16 * 64 * 2) + want(cap * 4 * 64 * 2)
    assert lib.lasnet_dense_workspace_bytes(ctypes.byref(d)) == 2 * want(2 * 14 * 14 * 64 * 2)
    assert lib.lasnet_compact_workspace_bytes(4096) == 8
    assert lib.lasnet_compact_workspace_bytes(4097) == 16
    bad = desc(s=0)
    assert lib.lasnet_dyn_workspace_bytes(ctypes.byref(bad), cap) == 0


FAKE = ctypes.c_void_p(0x10000)  # never dereferenced: validation fails first


def test_mask_validation(lib):
    d = desc()
    assert lib.lasnet_mask(None, FAKE, FAKE, 0.0, FAKE, None, None) == 1
    assert lib.lasnet_mask(ctypes.byref(d), None, FAKE, 0.0, FAKE, None, None) == 1
    assert lib.lasnet_mask(ctypes.byref(desc(s=0)), FAKE, FAKE, 0.0, FAKE, None, None) == 3
    assert lib.lasnet_mask(ctypes.byref(desc(dtype=7)), FAKE, FAKE, 0.0, FAKE, None, None) == 3
    assert lib.lasnet_mask(ctypes.byref(desc(h=0)), FAKE, FAKE, 0.0, FAKE, None, None) == 2
    assert lib.lasnet_mask(ctypes.byref(desc(stride=2)), FAKE, FAKE, 0.0, FAKE, None, None) == 4
    assert lib.lasnet_mask(ctypes.byref(desc(c_in=12)), FAKE, FAKE, 0.0, FAKE, None, None) == 4
    assert lib.lasnet_mask(ctypes.byref(d), ctypes.c_void_p(0x10008), FAKE, 0.0, FAKE, None, None) == 4


def test_compact_validation(lib):
    assert lib.lasnet_compact(FAKE, -1, FAKE, FAKE, FAKE, 8, None) == 2
    assert lib.lasnet_compact(FAKE, 10, FAKE, None, FAKE, 8, None) == 1
    assert lib.lasnet_compact(None, 10, FAKE, FAKE, FAKE, 8, None) == 1
    assert lib.lasnet_compact(FAKE, 5000, FAKE, FAKE, FAKE, 8, None) == 6
    assert lib.lasnet_compact(FAKE, 10, FAKE, FAKE, None, 0, None) == 6


def test_dyn_block_validation(lib):
    d = desc()
    w = _lib.BlockWeights(0x10000, 0x10000, 0x10000, 0x10000, 0x10000, 0x10000, None, None)
    wnull = _lib.BlockWeights(0x10000, None, 0x10000, 0x10000, 0x10000, 0x10000, None, None)
    wds = _lib.BlockWeights(0x10000, 0x10000, 0x10000, 0x10000, 0x10000, 0x10000, 0x10000, 0x10000)
    cap = 98
    big = 1 << 30
    call = lambda dd, ww, x, y, cap=cap, ws=FAKE, wsb=big: lib.lasnet_dyn_block(
        ctypes.byref(dd), ctypes.byref(ww), x, y, FAKE, FAKE, cap, ws, wsb, None)
    assert call(d, wnull, FAKE, FAKE) == 1
    assert call(d, wds, FAKE, FAKE) == 4
    assert call(d, w, None, FAKE) == 1
    assert call(desc(s=-1), w, FAKE, FAKE) == 3
    assert call(d, w, FAKE, FAKE, cap=-1) == 2
    assert call(d, w, FAKE, FAKE, cap=99) == 2                     # cap > n*gh*gw
    assert call(desc(c_mid=48), w, FAKE, FAKE) == 4                # not a multiple of 64
    assert call(desc(c_out=128), w, FAKE, FAKE) == 4               # non-identity residual
    assert call(d, w, FAKE, ctypes.c_void_p(0x10000 + 4096)) == 5  # partial overlap
    assert call(d, w, FAKE, FAKE, ws=None) == 6
    assert call(d, w, FAKE, FAKE, wsb=16) == 6


def test_dense_block_validation(lib):
    d = desc()
    w = _lib.BlockWeights(0x10000, 0x10000, 0x10000, 0x10000, 0x10000, 0x10000, None, None)
    assert lib.lasnet_dense_block(ctypes.byref(d), ctypes.byref(w), FAKE, None, FAKE, 1 << 30, None) == 1
    assert lib.lasnet_dense_block(ctypes.byref(d), ctypes.byref(w), FAKE, ctypes.c_void_p(0x10010), FAKE,
                                  1 << 30, None) == 5
    assert lib.lasnet_dense_block(ctypes.byref(d), ctypes.byref(w), FAKE, FAKE, FAKE, 10, None) == 6


def test_block_forward_validation(lib):
    d = desc()
    w = _lib.BlockWeights(0x10000, 0x10000, 0x10000, 0x10000, 0x10000, 0x10000, None, None)
    big = 1 << 30
    call = lambda dd, sched, x=FAKE, y=FAKE, wm=FAKE, ws=FAKE, wsb=big: lib.lasnet_block_forward(
        ctypes.byref(dd), ctypes.byref(w), x, y, wm, 0.0, sched, None, FAKE, FAKE, ws, wsb, None)
    for sched in (_lib.SCHED_SEPARATE, _lib.SCHED_FUSED):
        assert call(d, sched, x=None) == 1
        assert call(d, sched, wm=None) == 1
        assert call(desc(s=0), sched) == 3
        assert call(desc(c_out=128), sched) == 4
        assert call(d, sched, y=ctypes.c_void_p(0x10000 + 4096)) == 5
        assert call(d, sched, ws=None) == 6
        assert call(d, sched, wsb=64) == 6
    assert call(d, 2) == 3                                              # unknown schedule
    assert call(desc(dtype=_lib.LASNET_F32), _lib.SCHED_FUSED) == 4    # fused masker: bf16 only


def test_block_forward_workspace_and_schedule_choice(lib):
    d = desc(n=128, h=28, w=28, c_in=512, c_mid=128, c_out=512, s=4)
    px, cells = 128 * 28 * 28, 128 * 7 * 7
    fused = lib.lasnet_block_forward_workspace_bytes(ctypes.byref(d), _lib.SCHED_FUSED)
    # mpart + dense h1 dominate (conv2 reads its halos straight from the dense h1
    # at c_mid <= 128, s >= 4: no gathered copy); control words are small
    assert fused >= px * 16 + px * 128 * 2
    assert fused < px * 16 + px * 128 * 2 + 64 * 1024
    # s = 1: conv2 reads a gathered copy of the 3x3 halos of every cell
    d1 = desc(n=128, h=28, w=28, c_in=512, c_mid=128, c_out=512, s=1)
    f1 = lib.lasnet_block_forward_workspace_bytes(ctypes.byref(d1), _lib.SCHED_FUSED)
    assert px * 16 + px * 128 * 2 + px * 9 * 128 * 2 <= f1 < px * 16 + px * 128 * 2 + px * 9 * 128 * 2 + 256 * 1024
    assert lib.lasnet_block_forward_workspace_bytes(ctypes.byref(d), 5) == 0
    # the latency predictor (P:158-160 r_th; tests/test_predictor.py): at r = 0.5 the fused masker wins
    assert lib.lasnet_choose_schedule(ctypes.byref(d), 0.5) == _lib.SCHED_FUSED
    assert lib.lasnet_choose_schedule(ctypes.byref(d), 0.01) in (_lib.SCHED_SEPARATE, _lib.SCHED_FUSED)
    f32 = desc(dtype=_lib.LASNET_F32)
    assert lib.lasnet_choose_schedule(ctypes.byref(f32), 0.9) == _lib.SCHED_SEPARATE


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib._lib_backup = _lib._lib
        try:
            _lib._lib = None
            _lib.load(str(tmp_path / "nope.so"))
        finally:
            _lib._lib = _lib._lib_backup


def test_network_layer_entry_points_validate_before_launch(lib):
    """lasnet_proj_block / lasnet_stem / lasnet_maxpool / lasnet_head reject bad
    arguments on the host with the documented status (nothing launched)."""
    ST = {v: k for k, v in _lib.STATUS.items()}
    z = ctypes.c_void_p(0)
    # projection block: missing shortcut weights -> ERR_NULL; fp32 -> UNSUPPORTED; c_out % 128 -> UNSUPPORTED
    d = desc(c_in=256, c_mid=64, c_out=512, stride=2, h=7, w=7)
    w_no_ds = _lib.BlockWeights(FAKE.value, FAKE.value, FAKE.value, FAKE.value, FAKE.value, FAKE.value, None, None)
    w_ok = _lib.BlockWeights(*([FAKE.value] * 8))
    assert lib.lasnet_proj_block(ctypes.byref(d), ctypes.byref(w_no_ds), FAKE, FAKE, FAKE, 1 << 30, z) == \
        ST["LASNET_ERR_NULL"]
    d32 = desc(c_in=256, c_mid=64, c_out=512, stride=2, h=7, w=7, dtype=_lib.LASNET_F32)
    assert lib.lasnet_proj_block(ctypes.byref(d32), ctypes.byref(w_ok), FAKE, FAKE, FAKE, 1 << 30, z) == \
        ST["LASNET_ERR_UNSUPPORTED"]
    dbad = desc(c_in=256, c_mid=64, c_out=320, stride=2, h=7, w=7)
    assert lib.lasnet_proj_block(ctypes.byref(dbad), ctypes.byref(w_ok), FAKE, FAKE, FAKE, 1 << 30, z) == \
        ST["LASNET_ERR_UNSUPPORTED"]
    dst3 = desc(stride=3)
    assert lib.lasnet_proj_block(ctypes.byref(dst3), ctypes.byref(w_ok), FAKE, FAKE, FAKE, 1 << 30, z) == \
        ST["LASNET_ERR_DOMAIN"]
    far = ctypes.c_void_p(FAKE.value + (1 << 32))  # a y that does not overlap x
    assert lib.lasnet_proj_block(ctypes.byref(d), ctypes.byref(w_ok), FAKE, far, FAKE, 0, z) == \
        ST["LASNET_ERR_WORKSPACE"]
    # overlapping x / y -> ERR_ALIAS
    assert lib.lasnet_proj_block(ctypes.byref(d), ctypes.byref(w_ok), FAKE, ctypes.c_void_p(FAKE.value + 64), FAKE,
                                 1 << 30, z) == ST["LASNET_ERR_ALIAS"]
    assert lib.lasnet_proj_workspace_bytes(ctypes.byref(d)) > 0
    # stem: w % 4 -> UNSUPPORTED, null -> NULL, no workspace -> WORKSPACE
    assert lib.lasnet_stem(2, 112, 110, FAKE, FAKE, FAKE, FAKE, FAKE, 1 << 20, z) == ST["LASNET_ERR_UNSUPPORTED"]
    assert lib.lasnet_stem(2, 112, 112, None, FAKE, FAKE, FAKE, FAKE, 1 << 20, z) == ST["LASNET_ERR_NULL"]
    assert lib.lasnet_stem(2, 112, 112, FAKE, FAKE, FAKE, FAKE, FAKE, 16, z) == ST["LASNET_ERR_WORKSPACE"]
    assert lib.lasnet_stem_workspace_bytes() == 64 * 448 * 2
    # max pool: c % 8 -> UNSUPPORTED; head: bad sizes -> SHAPE, small workspace -> WORKSPACE
    assert lib.lasnet_maxpool(2, 56, 56, 60, FAKE, FAKE, z) == ST["LASNET_ERR_UNSUPPORTED"]
    assert lib.lasnet_head(2, 49, 0, 1000, FAKE, FAKE, FAKE, FAKE, FAKE, 1 << 20, z) == ST["LASNET_ERR_SHAPE"]
    assert lib.lasnet_head(2, 49, 2048, 1000, FAKE, FAKE, FAKE, FAKE, FAKE, 8, z) == ST["LASNET_ERR_WORKSPACE"]
    assert lib.lasnet_head_workspace_bytes(2, 2048) == 2 * 2048 * 4
