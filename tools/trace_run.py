"""Per-role timeline of CTA 0 for each conv kernel of the bench workload (trace build)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2210_06223_b200 import _lib, build  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

path = build.build(trace=True)
lib = _lib.load(path)
lib.lasnet_trace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
lib.lasnet_trace_clear.argtypes = [ctypes.c_int]
lib.lasnet_ktrace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
n, h, w, c, cm, s = 128, 28, 28, 512, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 4
if len(sys.argv) > 2:  # n,h,w,c,cm (e.g. 256,14,14,1024,256 for the LAS-R101 stage-3 block)
    n, h, w, c, cm = (int(v) for v in sys.argv[2].split(","))
sched = L.SCHED_FUSED if len(sys.argv) > 3 and sys.argv[3] == "fused" else None
x = synth.make_x(n, h, w, c, seed=0).cuda()
blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, s), synth.make_block_weights(c, cm, c, seed=1),
                 synth.make_masker_weights(c, seed=2), 0.0, schedule=sched)
blk.calibrate_bias(synth.make_x(n, h, w, c, seed=1000).cuda(), 0.5)
y = x.clone()
y2 = torch.empty_like(x)
lib.lasnet_mtrace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
for _ in range(3):
    y.copy_(x)
    lib.lasnet_mtrace_clear()
    blk.mask_compact(y)
    torch.cuda.synchronize()
    mt = (ctypes.c_ulonglong * 4)()
    lib.lasnet_mtrace_read(mt)
    print(f"== mask_compact: last decision {(mt[1] - mt[0]) / 1e3:.2f} us, compaction start {(mt[2] - mt[0]) / 1e3:.2f}, "
          f"done {(mt[3] - mt[0]) / 1e3:.2f} us after the first CTA started")
if hasattr(lib, "lasnet_trace23_read"):
    lib.lasnet_trace23_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    for _ in range(2):
        y.copy_(x)
        blk.forward(y)
    torch.cuda.synchronize()
    lib.lasnet_trace23_clear()
    y.copy_(x)
    blk.forward(y)
    torch.cuda.synchronize()
    b23 = (ctypes.c_ulonglong * 512)()
    lib.lasnet_trace23_read(b23)
    t = np.array(b23, dtype=np.int64).reshape(64, 8)
    t0 = t[t[:, 0] > 0][:, 0].min() if (t[:, 0] > 0).any() else 0
    print("== conv23 (fused conv2+conv3), CTA0; us: conv2 start | acc2 ready | H2 staged | conv3 MMAs done | stored")
    for i in range(64):
        if t[i, 0]:
            print(f"   {i:4d} " + " ".join(f"{(v - t0) / 1e3:7.2f}" if v else "    nan" for v in t[i, :5]))
    if hasattr(lib, "lasnet_trace23c_read"):
        lib.lasnet_trace23c_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
        bc = (ctypes.c_ulonglong * 1024)()
        lib.lasnet_trace23c_read(bc)
        tc = np.array(bc, dtype=np.int64).reshape(64, 16)
        print("   chunk  W3issue accFree W3land  commit | resLand accRdy stored  tmemLd  mathDn  ldsDn")
        for c in range(64):
            if tc[c, 0]:
                print(f"   {c:5d} " + " ".join(f"{(v - t0) / 1e3:7.2f}" if v else "    nan" for v in tc[c, :10]))
names = {0: "conv1_dyn", 1: "conv2_dyn", 2: "conv3_dyn", 3: "conv1_dense", 4: "conv2_dense", 5: "conv3_dense",
         6: "conv1_mask", 8: "conv2_gather"}
for mode in (0, 1, 2, 3, 4, 5, 6, 8):
    for _ in range(2):
        y.copy_(x)
        blk.forward(y)
        blk.dense(x, y2)
    torch.cuda.synchronize()
    lib.lasnet_trace_clear(mode)
    y.copy_(x)
    blk.forward(y)
    blk.dense(x, y2)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 512)()
    lib.lasnet_trace_read(buf, 512)
    t = np.array(buf, dtype=np.int64).reshape(64, 8)
    valid = t[:, 0] > 0
    t0 = t[valid][:, 0].min() if valid.any() else 0
    print(f"== {names[mode]} (S={s}): CTA0 tiles={int(valid.sum())}; us rel. to first producer start")
    print("   tile  prod0  prodK  mmaFree mmaDone epiRdy epiStg stored")
    for i in range(64):
        if t[i, 0] == 0:
            continue
        row = [(v - t0) / 1e3 if v > 0 else float('nan') for v in t[i, :7]]
        print(f"   {i:4d} " + " ".join(f"{v:7.2f}" for v in row))
    if mode in (0, 2, 3, 6, 8):
        kb = (ctypes.c_ulonglong * 512)()
        lib.lasnet_ktrace_read(kb)
        k = np.array(kb, dtype=np.int64).reshape(128, 4)
        print("   kblk  gather   tma   mmaFull  gthrWaitDone (us rel.)  lat(full-issue)")
        for i in range(0, 48):
            if k[i, 1] == 0:
                continue
            iss = max(k[i, 0], k[i, 1]) if k[i, 0] else k[i, 1]
            print(f"   {i:4d} " + " ".join(f"{(v - t0) / 1e3:7.2f}" if v else "    nan" for v in k[i, :4])
                  + f"   {(k[i, 2] - iss) / 1e3:6.2f}")
