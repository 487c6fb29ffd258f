"""Run one small block through both schedules under the library options given in
the environment (LASNET_* knobs are read once per process) and check it against
the fp64 oracle: masks/idx/count bit-exact, activations within the bf16
tolerance.  Invoked by tests/test_gpu_parity.py::test_library_variants."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402
from parity_util import BF16_TOL, make_case, margin_bias, max_abs_rel, to_dev  # noqa: E402

oracle.build()
for (n, h, w, c_in, c_mid, s) in [(4, 28, 28, 512, 128, 4), (3, 13, 11, 256, 64, 3)]:
    x, wts, wm = make_case(n, h, w, c_in, c_mid, s, seed=61)
    xd = synth.to_f64(x)
    _, l0 = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
    bm = margin_bias(l0, 0.5)
    m_or, _ = oracle.masker(xd, synth.to_f64(wm), bm, s)
    idx_or, cnt = oracle.compact(m_or)
    want = oracle.dyn_block_def(xd, synth.weights_f64(wts), m_or, s, rmode=oracle.ROUND_BF16)
    for sched in (L.SCHED_SEPARATE, L.SCHED_FUSED):
        y, m, idx, count = L.block_forward(x.cuda(), to_dev(wts), wm.cuda(), bm, s, sched)
        assert np.array_equal(m.cpu().numpy(), m_or), "mask"
        assert int(count.item()) == cnt and np.array_equal(idx[:cnt].cpu().numpy(), idx_or), "idx"
        err = max_abs_rel(synth.to_f64(y.cpu()), want)
        assert err <= BF16_TOL, f"activations {err}"
    yd = L.dense_block(x.cuda(), to_dev(wts))
    wd = oracle.static_block(xd, synth.weights_f64(wts), rmode=oracle.ROUND_BF16)
    assert max_abs_rel(synth.to_f64(yd.cpu()), wd) <= BF16_TOL, "dense"
print("variant ok")
