import sys, torch, statistics
sys.path.insert(0, ".")
import synth, paper_2210_06223_b200 as L
n=256
x = synth.make_image_batch(n, 224, seed=0).cuda()
w = synth.make_lasnet_weights(seed=11)
sw, sb = w["stem_w"].cuda(), w["stem_b"].cuda()
y = L.stem(x, sw, sb)
def t(fn, k=20):
    st=torch.cuda.current_stream(); ev=[]
    for _ in range(3): fn()
    for _ in range(k):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); a.record(st); fn(); b.record(st); ev.append((a,b))
    torch.cuda.synchronize(); return statistics.median(a.elapsed_time(b) for a,b in ev)
print("stem ms", t(lambda: L.stem(x, sw, sb)), "maxpool ms", t(lambda: L.maxpool(y)))
