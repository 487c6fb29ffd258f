import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import synth, oracle
import paper_2210_06223_b200 as L
from parity_util import max_abs_rel, to_dev
oracle.build()
for (n, hi, c_in, c_mid, c_out, st) in [(1, 56, 256, 128, 512, 2), (1, 28, 512, 256, 1024, 2), (1, 32, 128, 64, 256, 2), (1, 24, 128, 64, 256, 2), (1, 20, 128, 64, 256, 2), (2, 18, 128,64,256,2)]:
    x = synth.make_x(n, hi, hi, c_in, seed=1)
    w = synth.make_proj_weights(c_in, c_mid, c_out, seed=2)
    y = L.proj_block(x.cuda(), to_dev(w), st).cpu()
    want = oracle.proj_block(synth.to_f64(x), synth.weights_f64(w), st)
    got = synth.to_f64(y)
    err = np.abs(got - want).max(axis=(0, 2, 3)) / np.abs(want).max()
    print((n, hi, c_in, c_mid, c_out, st), max_abs_rel(got, want), 'bad rows', np.nonzero(err > 0.02)[0][:20])
