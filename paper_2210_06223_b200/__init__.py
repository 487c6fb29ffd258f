"""B200-native LASNet coarse-grained spatially-dynamic residual block (arXiv 2210.06223).

Product path: include/lasnet.h C ABI implemented by liblasnet.so (sm_100a
kernels in csrc/), bound by ctypes in _lib.py, with the Python API in block.py.
There is no CPU fallback: calls raise if the CUDA library is missing.
"""
from ._lib import SCHED_DENSE, SCHED_FUSED, SCHED_SEPARATE
from .net import LASResNet, ProjBlock
from .regnet import LASRegNet, RegNetBlock
from .block import (BlockShape, DynBlock, ProjDynBlock, block_forward, proj_block_forward, predict_latency, hw_b200, choose_schedule, compact, dense_block, dyn_block, grid,
                    head, last_launch_count, make_desc, make_weights, mask, maxpool, proj_block, stem)

__all__ = ["LASRegNet", "RegNetBlock", "SCHED_DENSE", "predict_latency", "hw_b200", "BlockShape", "DynBlock", "ProjDynBlock", "proj_block_forward", "SCHED_FUSED", "SCHED_SEPARATE", "block_forward", "choose_schedule", "compact",
           "dense_block", "dyn_block", "grid", "last_launch_count", "make_desc", "make_weights", "mask", "proj_block",
           "stem", "maxpool", "head", "LASResNet", "ProjBlock"]
