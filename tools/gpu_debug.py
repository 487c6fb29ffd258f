"""Quick GPU diagnostics: run each step once on small inputs and print the error
against the oracle (no asserts), so one gpurun call shows where things break."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402
from paper_2210_06223_b200 import build  # noqa: E402
from parity_util import max_abs_rel, to_dev  # noqa: E402


def step(name, fn):
    t = time.time()
    try:
        out = fn()
        torch.cuda.synchronize()
        print(f"[{name}] ok {time.time() - t:.2f}s {out if out is not None else ''}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"[{name}] FAIL {type(e).__name__}: {e}", flush=True)


def main():
    build.build()
    oracle.build()
    print(torch.cuda.get_device_name(), flush=True)
    n, h, w, c_in, c_mid, s = 2, 14, 14, 256, 64, 2
    x = synth.make_x(n, h, w, c_in, seed=0)
    wts = synth.make_block_weights(c_in, c_mid, c_in, seed=1)
    wm = synth.make_masker_weights(c_in, seed=2)
    xd, wd = synth.to_f64(x), synth.weights_f64(wts)

    def t_mask():
        m = L.mask(x.cuda(), wm.cuda(), 0.0, s).cpu().numpy()
        mo, _ = oracle.masker(xd, synth.to_f64(wm), 0.0, s)
        return f"mismatch={int((m != mo).sum())} active={int(m.sum())}"

    def t_compact():
        m = (np.random.default_rng(0).random(10000) < 0.5).astype(np.uint8)
        idx, cnt = L.compact(torch.from_numpy(m).cuda())
        c = int(cnt.item())
        ref = np.flatnonzero(m)
        return f"count={c} ref={len(ref)} eq={np.array_equal(idx[:c].cpu().numpy(), ref)}"

    def t_dense(dtype):
        xx = synth.make_x(n, h, w, c_in, seed=0, dtype=dtype)
        ww = synth.make_block_weights(c_in, c_mid, c_in, seed=1, dtype=dtype)
        y = L.dense_block(xx.cuda(), to_dev(ww)).cpu()
        want = oracle.static_block(synth.to_f64(xx), synth.weights_f64(ww),
                                   rmode=oracle.ROUND_BF16 if dtype == "bf16" else oracle.ROUND_F32)
        return f"err={max_abs_rel(synth.to_f64(y), want):.3e}"

    def t_dyn(dtype, ss, r):
        xx = synth.make_x(n, h, w, c_in, seed=0, dtype=dtype)
        ww = synth.make_block_weights(c_in, c_mid, c_in, seed=1, dtype=dtype)
        gh, gw = L.grid(h, w, ss)
        mc = synth.make_cell_mask(n, gh, gw, r, seed=3)
        idx, cnt = L.compact(torch.from_numpy(mc).cuda())
        y = xx.cuda().clone()
        L.dyn_block(y, to_dev(ww), idx, cnt, ss)
        io, _ = oracle.compact(mc)
        want = oracle.dyn_block_literal(synth.to_f64(xx), synth.weights_f64(ww), io, ss,
                                        rmode=oracle.ROUND_BF16 if dtype == "bf16" else oracle.ROUND_F32)
        got = synth.to_f64(y.cpu())
        return f"err={max_abs_rel(got, want):.3e} nan={int(np.isnan(got).sum())}"

    step("mask", t_mask)
    step("compact", t_compact)
    step("dense_f32", lambda: t_dense("f32"))
    step("dyn_f32", lambda: t_dyn("f32", 2, 0.5))
    step("dense_bf16", lambda: t_dense("bf16"))
    for ss in (1, 2, 4, 7):
        step(f"dyn_bf16_s{ss}", lambda ss=ss: t_dyn("bf16", ss, 0.5))


if __name__ == "__main__":
    main()
