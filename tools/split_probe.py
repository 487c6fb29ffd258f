"""Does running the LAS-R101 forward as two half batches on two streams (one CUDA
graph, fork/join) fill the persistent kernels' partial last rounds?  Times the
whole-batch graph against the split graph (same weights, same masker biases) and
checks the logits are bitwise equal."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

N = 256
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 2
weights = synth.make_lasnet_weights(seed=1)
full = L.LASResNet(N, weights, hw=224)
full.forward(synth.make_image_batch(N, 224, seed=5000).cuda(), calibrate_r=0.5)
parts = [L.LASResNet(N // ns, weights, hw=224) for _ in range(ns)]
src = list(full.blocks())
for p in parts:
    for a, b in zip(p.blocks(), src):
        a.bm = b.bm
x = synth.make_image_batch(N, 224, seed=1).cuda()
xs = [x[i * (N // ns):(i + 1) * (N // ns)] for i in range(ns)]


def run_split(dense=False):
    cur = torch.cuda.current_stream()
    outs = []
    for i, p in enumerate(parts):
        s = streams[i]
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            outs.append(p.forward(xs[i], dense=dense))
    for s in streams:
        cur.wait_stream(s)
    return outs


streams = [torch.cuda.Stream() for _ in range(ns)]
res = {}
for dense in (False, True):
    gf = full.capture(x, dense=dense)
    run_split(dense)
    torch.cuda.synchronize()
    gs = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gs):
        run_split(dense)
    for name, g in (("full", gf), ("split", gs)):
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[(name, dense)] = e0.elapsed_time(e1) / 20
    gf.replay()
    gs.replay()
    torch.cuda.synchronize()
    same = all(torch.equal(full.logits[i * (N // ns):(i + 1) * (N // ns)], parts[i].logits) for i in range(ns))
    print(f"dense={dense}: full {res[('full', dense)]:.3f} ms  split x{ns} {res[('split', dense)]:.3f} ms  "
          f"logits bitwise equal: {same}")
print(f"speedup vs dense: full {res[('full', True)] / res[('full', False)]:.3f}  "
      f"split {res[('split', True)] / res[('split', False)]:.3f}")
