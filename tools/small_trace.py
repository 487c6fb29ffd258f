"""Phase timeline of the single-launch small-batch block (trace build), config 1."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2210_06223_b200 import _lib, build  # noqa: E402

lib = _lib.load(build.build(trace=True))
import paper_2210_06223_b200 as L  # noqa: E402

n, h, w, c, cm, s = 1, 14, 14, 256, 64, 2
x = synth.make_x(n, h, w, c, seed=0, dtype="f32").cuda()
wts = synth.make_block_weights(c, cm, c, seed=1, dtype="f32")
blk = L.DynBlock(L.BlockShape(n, h, w, c, cm, s, torch.float32), wts, synth.make_masker_weights(c, seed=2), 0.0,
                 schedule=L.SCHED_SEPARATE)
blk.calibrate_bias(x, 25 / 49)
y, y2 = x.clone(), torch.empty_like(x)
lib.lasnet_small_trace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
for name, fn in (("dynamic", lambda: blk.forward(y)), ("dense", lambda: blk.dense(x, y2))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    lib.lasnet_small_trace_read(buf)
    t = np.array(buf, dtype=np.int64)
    t0 = t[0]
    print(name, "CTA0 :", " ".join(f"{(v - t0) / 1e3:6.2f}" if v else "   nan" for v in t[:8]))
    print(name, "last :", " ".join(f"{(v - t0) / 1e3:6.2f}" if v else "   nan" for v in t[8:]))
