"""Build the in-tree CUDA library liblasnet.so for sm_100a with nvcc.

The .so is built next to this file (git-ignored, travels to the GPU box with
the gpurun snapshot).  Usage: ``python -m paper_2210_06223_b200.build``.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblasnet.so")
SOURCES = ["lasnet_capi.cu", "mask_compact.cu", "conv_tc.cu", "conv23_tc.cu", "conv_simt.cu", "decide_gather.cu",
           "proj_block.cu", "net_layers.cu", "predictor.cu",
           "regnet.cu", "small_block.cu"]
HEADERS = ["rowmap.cuh", "sm100_ptx.cuh", "launch.cuh", "predictor_b200.inc", "regnet.cuh", "small_block.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# A/B experiments only: extra nvcc flags (e.g. -DLASNET_C23_STAGES=2); the product build sets none
EXTRA = os.environ.get("LASNET_EXTRA_NVCC", "").split()
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "lasnet.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace=True builds liblasnet_trace.so with the per-role timeline of CTA 0
    (debug only; the product library never has it)."""
    lib = LIB if not trace else LIB.replace(".so", "_trace.so")
    if not force and not trace and not _stale():
        return LIB
    bdir = os.path.join(HERE, "build" if not trace else "build_trace")
    os.makedirs(bdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *EXTRA, *(["-DLASNET_TRACE"] if trace else []), "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, r

    from concurrent.futures import ThreadPoolExecutor

    objs = []
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        for src, obj, r in ex.map(compile_one, SOURCES):
            if verbose or r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}")
            objs.append(obj)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", lib, *objs]
    subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
