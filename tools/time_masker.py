"""Time masker variants on the config-2 shape: lasnet_mask alone, lasnet_compact
alone, and the fused lasnet_mask_compact, L2 flushed (256 MB read) before each."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402

n, h, w, c = 128, 28, 28, 512
x = synth.make_x(n, h, w, c, seed=0).cuda()
flush = torch.ones(32 << 20, dtype=torch.int64, device="cuda")


def timeit(fn, reps=10):
    ts = []
    for _ in range(reps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for s in (1, 2, 4, 7):
    blk = L.DynBlock(L.BlockShape(n, h, w, c, 128, s), synth.make_block_weights(c, 128, c, seed=1),
                     synth.make_masker_weights(c, seed=2), 0.0)
    blk.calibrate_bias(x, 0.5)
    t_mask = timeit(lambda: blk.mask(x))
    t_comp = timeit(lambda: blk.compact())
    t_fused = timeit(lambda: blk.mask_compact(x))
    print(f"S={s}: mask {t_mask:7.1f} us  compact {t_comp:6.1f} us  fused {t_fused:7.1f} us  "
          f"(x read at {x.numel() * 2 / t_mask / 1e3:.0f} GB/s by mask)", flush=True)
