import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import synth, paper_2210_06223_b200 as L
from parity_util import make_case, to_dev
n, h, w, c_in, c_mid, s = 1, 7, 7, 512, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 1
x, wts, _ = make_case(n, h, w, c_in, c_mid, s, seed=101)
gh, gw = L.grid(h, w, s)
mc = synth.make_cell_mask(n, gh, gw, 0.5, seed=s)
idx, cnt = L.compact(torch.from_numpy(mc).cuda())
y = x.cuda().clone()
L.dyn_block(y, to_dev(wts), idx, cnt, s)
torch.cuda.synchronize()
print("ok", s)
