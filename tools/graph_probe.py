"""Stress probe: chained identity blocks of consecutive LAS-R101 stages, set up eagerly
(each block calibrated on the activations it sees), captured per stage in one CUDA
graph and replayed.  It found the odd-stage-count masker race.

  python tools/graph_probe.py N STAGE:BLOCKS:FLUSH[:SCHED] ...   e.g. 256 s2:3:1:f s3:22:1:f
  (SCHED f = masker-fused, s = masker-separate, n = step-by-step calls)"""
import sys
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
stages = {"s1": (56, 256, 64, 4), "s2": (28, 512, 128, 4), "s3": (14, 1024, 256, 2), "s4": (7, 2048, 512, 1)}
n = int(sys.argv[1])
for spec in sys.argv[2:]:
    name, nb, fl, sc = (spec.split(":") + ["f"])[:4]
    sched = {"f": L.SCHED_FUSED, "s": L.SCHED_SEPARATE, "n": None}[sc]
    h, c, cm, s = stages[name]
    nb, fl = int(nb), int(fl)
    x = synth.make_x(n, h, h, c, seed=1).cuda()
    y = x.clone()
    blks = []
    for b in range(nb):
        blk = L.DynBlock(L.BlockShape(n, h, h, c, cm, s), synth.make_block_weights(c, cm, c, seed=b + 1),
                         synth.make_masker_weights(c, seed=b + 2), 0.0, schedule=sched)
        blk.calibrate_bias(y, 0.5)
        torch.cuda.synchronize()
        blk.forward(y)
        try:
            torch.cuda.synchronize()
        except Exception as e:
            print("FAULT in eager forward of", name, "block", b, str(e)[:80], flush=True)
            raise
        c_now = int(blk.count.item())
        if not 0 <= c_now <= blk.shape.ncells:
            print("BAD COUNT", name, b, c_now, flush=True)
        blks.append(blk)

    def fwd():
        for b in blks:
            b.forward(y)

    y.copy_(x)
    for _ in range(2):
        fwd()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fwd()
    for _ in range(3):
        y.copy_(x)
        if fl:
            flush.sum()
        g.replay()
    torch.cuda.synchronize()
    print("graph ok", name, n, nb, fl, flush=True)
    del blks, g, x, y
    torch.cuda.empty_cache()
