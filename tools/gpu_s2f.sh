#!/bin/bash
# Wide (c_mid 256) fused conv23 on pairs: parity + network A/B (LASNET_C23_WIDE=0/1).
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "256 or 1024 or network or stage3 or dense or variants or proj" 2>&1 | tail -4
for V in 0 1; do
LASNET_C23_WIDE=$V timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-block --no-regnet --detail gpurun_out/det_w$V.json > gpurun_out/bench_w$V.json 2> gpurun_out/bench_w$V.err
echo "WIDE=$V rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_w$V.json'))
k=d['kernels']
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['dense_identity_ms_per_step'], {n: k[n]['ms'] for n in list(k)[:7]})
" || tail -5 gpurun_out/bench_w$V.err
done
python tools/stage_kernels.py gpurun_out/det_w1.json | grep -E " 2 |forward"
