"""One LAS-R101 stem launch (N=256, 224x224) under cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import sys
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2210_06223_b200 as L  # noqa: E402
w = synth.make_lasnet_weights(seed=1)
x = synth.make_image_batch(256, 224, seed=1).cuda()
sw, sb = w["stem_w"].cuda(), w["stem_b"].cuda()
y = L.stem(x, sw, sb)
torch.cuda.synchronize()
torch.cuda.profiler.start()
y = L.stem(x, sw, sb)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
