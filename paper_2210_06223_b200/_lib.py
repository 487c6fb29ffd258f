"""ctypes binding of liblasnet.so (include/lasnet.h).  Argument marshalling only.

There is no fallback: if the CUDA library is missing or fails to load, every
entry point raises.  Tensors are passed as raw device pointers; torch only
supplies memory and the current stream.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblasnet.so")

LASNET_F32, LASNET_BF16 = 0, 1
STATUS = {
    0: "LASNET_OK", 1: "LASNET_ERR_NULL", 2: "LASNET_ERR_SHAPE", 3: "LASNET_ERR_DOMAIN",
    4: "LASNET_ERR_UNSUPPORTED", 5: "LASNET_ERR_ALIAS", 6: "LASNET_ERR_WORKSPACE", 7: "LASNET_ERR_CUDA",
}

# every symbol include/lasnet.h declares
EXPORTS = [
    "lasnet_mask", "lasnet_mask_compact", "lasnet_mask_compact_workspace_bytes", "lasnet_compact", "lasnet_compact_workspace_bytes", "lasnet_dyn_block",
    "lasnet_dyn_workspace_bytes", "lasnet_dense_block", "lasnet_dense_workspace_bytes",
    "lasnet_status_str", "lasnet_abi_version", "lasnet_last_launch_count", "lasnet_set_kernel_events",
    "lasnet_block_forward", "lasnet_block_forward_workspace_bytes", "lasnet_choose_schedule",
    "lasnet_proj_block", "lasnet_proj_workspace_bytes", "lasnet_stem", "lasnet_stem_workspace_bytes",
    "lasnet_maxpool", "lasnet_head", "lasnet_head_workspace_bytes", "lasnet_kernel_event_name",
    "lasnet_kernel_event_count", "lasnet_hw_b200", "lasnet_kernel_type_name", "lasnet_predict_latency",
    "lasnet_regnet_block", "lasnet_regnet_workspace_bytes", "lasnet_regnet_stem",
]

# lasnet_schedule (SCHED_DENSE: predictor only, the static block)
SCHED_SEPARATE, SCHED_FUSED, SCHED_DENSE = 0, 1, 2
K_COUNT = 18


class HW(ctypes.Structure):
    """lasnet_hw: the predictor's hardware model."""
    _fields_ = [("sms", ctypes.c_int32), ("hbm_gbs", ctypes.c_double), ("l2_gbs", ctypes.c_double),
                ("tc_tflops", ctypes.c_double), ("launch_us", ctypes.c_double), ("eff", ctypes.c_double * K_COUNT),
                ("t0_us", ctypes.c_double * K_COUNT)]


class BlockDesc(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("n", "h", "w", "c_in", "c_mid", "c_out", "stride", "s", "dtype")]


class BlockWeights(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in ("w1", "b1", "w2", "b2", "w3", "b3", "wd", "bd")]


class RegnetWeights(ctypes.Structure):
    _fields_ = [("wa", ctypes.c_void_p), ("ba", ctypes.c_void_p), ("wb", ctypes.c_void_p), ("bb", ctypes.c_void_p),
                ("se_w1", ctypes.c_void_p), ("se_b1", ctypes.c_void_p), ("se_w2", ctypes.c_void_p),
                ("se_b2", ctypes.c_void_p), ("w_se", ctypes.c_int32), ("wc", ctypes.c_void_p), ("bc", ctypes.c_void_p),
                ("wd", ctypes.c_void_p), ("bd", ctypes.c_void_p)]


class LasnetError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} -> {STATUS.get(code, code)}")
        self.code = code


_lib = None


def load(path: str = LIB_PATH):
    """Load liblasnet.so.  Raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"liblasnet.so not found at {path}; build it with `python -m paper_2210_06223_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
    D = ctypes.POINTER(BlockDesc)
    Wt = ctypes.POINTER(BlockWeights)
    lib.lasnet_mask.argtypes = [D, vp, vp, ctypes.c_float, vp, vp, vp]
    lib.lasnet_mask.restype = ctypes.c_int
    lib.lasnet_mask_compact.argtypes = [D, vp, vp, ctypes.c_float, vp, vp, vp, vp, vp, sz, vp]
    lib.lasnet_mask_compact.restype = ctypes.c_int
    lib.lasnet_mask_compact_workspace_bytes.argtypes = [D]
    lib.lasnet_mask_compact_workspace_bytes.restype = sz
    lib.lasnet_compact.argtypes = [vp, i32, vp, vp, vp, sz, vp]
    lib.lasnet_compact.restype = ctypes.c_int
    lib.lasnet_compact_workspace_bytes.argtypes = [i32]
    lib.lasnet_compact_workspace_bytes.restype = sz
    lib.lasnet_dyn_block.argtypes = [D, Wt, vp, vp, vp, vp, i32, vp, sz, vp]
    lib.lasnet_dyn_block.restype = ctypes.c_int
    lib.lasnet_dyn_workspace_bytes.argtypes = [D, i32]
    lib.lasnet_dyn_workspace_bytes.restype = sz
    lib.lasnet_dense_block.argtypes = [D, Wt, vp, vp, vp, sz, vp]
    lib.lasnet_dense_block.restype = ctypes.c_int
    lib.lasnet_dense_workspace_bytes.argtypes = [D]
    lib.lasnet_dense_workspace_bytes.restype = sz
    lib.lasnet_block_forward.argtypes = [D, Wt, vp, vp, vp, ctypes.c_float, i32, vp, vp, vp, vp, sz, vp]
    lib.lasnet_block_forward.restype = ctypes.c_int
    lib.lasnet_block_forward_workspace_bytes.argtypes = [D, i32]
    lib.lasnet_block_forward_workspace_bytes.restype = sz
    lib.lasnet_choose_schedule.argtypes = [D, ctypes.c_double]
    lib.lasnet_choose_schedule.restype = i32
    lib.lasnet_proj_block.argtypes = [D, Wt, vp, vp, vp, sz, vp]
    lib.lasnet_proj_block.restype = ctypes.c_int
    lib.lasnet_proj_workspace_bytes.argtypes = [D]
    lib.lasnet_proj_workspace_bytes.restype = sz
    lib.lasnet_stem.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, sz, vp]
    lib.lasnet_stem.restype = ctypes.c_int
    lib.lasnet_stem_workspace_bytes.argtypes = []
    lib.lasnet_stem_workspace_bytes.restype = sz
    lib.lasnet_maxpool.argtypes = [i32, i32, i32, i32, vp, vp, vp]
    lib.lasnet_maxpool.restype = ctypes.c_int
    lib.lasnet_head.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp, vp, sz, vp]
    lib.lasnet_head.restype = ctypes.c_int
    lib.lasnet_head_workspace_bytes.argtypes = [i32, i32]
    lib.lasnet_head_workspace_bytes.restype = sz
    lib.lasnet_status_str.argtypes = [ctypes.c_int]
    lib.lasnet_status_str.restype = ctypes.c_char_p
    lib.lasnet_abi_version.restype = i32
    lib.lasnet_last_launch_count.restype = i32
    lib.lasnet_set_kernel_events.argtypes = [ctypes.POINTER(ctypes.c_void_p), i32]
    lib.lasnet_set_kernel_events.restype = ctypes.c_int
    lib.lasnet_kernel_event_name.argtypes = [i32]
    lib.lasnet_kernel_event_name.restype = ctypes.c_char_p
    lib.lasnet_kernel_event_count.restype = i32
    lib.lasnet_hw_b200.argtypes = [ctypes.POINTER(HW)]
    lib.lasnet_hw_b200.restype = None
    lib.lasnet_kernel_type_name.argtypes = [i32]
    lib.lasnet_kernel_type_name.restype = ctypes.c_char_p
    lib.lasnet_predict_latency.argtypes = [D, i32, ctypes.c_double, ctypes.POINTER(HW), ctypes.POINTER(i32),
                                           ctypes.POINTER(ctypes.c_double), i32, ctypes.POINTER(i32)]
    lib.lasnet_predict_latency.restype = ctypes.c_double
    RW = ctypes.POINTER(RegnetWeights)
    lib.lasnet_regnet_block.argtypes = [D, RW, vp, vp, vp, ctypes.c_float, i32, vp, vp, vp, vp, sz, vp]
    lib.lasnet_regnet_block.restype = ctypes.c_int
    lib.lasnet_regnet_workspace_bytes.argtypes = [D, i32]
    lib.lasnet_regnet_workspace_bytes.restype = sz
    lib.lasnet_regnet_stem.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp, vp]
    lib.lasnet_regnet_stem.restype = ctypes.c_int
    _lib = lib
    return lib


def check(fn: str, code: int) -> None:
    if code != 0:
        raise LasnetError(fn, code)
