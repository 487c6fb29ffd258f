"""Per-role timeline of CTA 0 of the fused conv23 at the LAS-R101 stage-3 shape
(N=256, 14x14x1024, c_mid 256, S=2, r=0.5; 2-SM pairs), trace build."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2210_06223_b200 import _lib, build  # noqa: E402

path = build.build(trace=True)
lib = _lib.load(path)
import paper_2210_06223_b200 as L  # noqa: E402

n, h, w, c, cm, s = 256, 14, 14, 1024, 256, 2
if len(sys.argv) > 1:
    n, h, w, c, cm, s = (int(v) for v in sys.argv[1].split(","))
x = synth.make_x(n, h, w, c, seed=0).cuda()
blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, s), synth.make_block_weights(c, cm, c, seed=1),
                 synth.make_masker_weights(c, seed=2), 0.0, schedule=L.SCHED_FUSED)
blk.calibrate_bias(synth.make_x(n, h, w, c, seed=1000).cuda(), 0.5)
y = x.clone()
lib.lasnet_trace23_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
lib.lasnet_trace23c_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
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
t0 = t[t[:, 0] > 0][:, 0].min()
print("== conv23, CTA0; us: conv2 start | acc2 ready | H2 staged | conv3 MMAs done | stored")
for i in range(64):
    if t[i, 0]:
        print(f"   {i:4d} " + " ".join(f"{(v - t0) / 1e3:7.2f}" if v else "    nan" for v in t[i, :5]))
bc = (ctypes.c_ulonglong * 1024)()
lib.lasnet_trace23c_read(bc)
tc = np.array(bc, dtype=np.int64).reshape(64, 16)
print("   chunk  W3issue accFree W3land  commit | resLand accRdy stored  tmemLd  mathDn  ldsDn")
for ch in range(64):
    if tc[ch, 0] or tc[ch, 4]:
        print(f"   {ch:5d} " + " ".join(f"{(v - t0) / 1e3:7.2f}" if v else "    nan" for v in tc[ch, :10]))
