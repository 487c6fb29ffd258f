#!/bin/bash
# CTA-pair conv_tc: parity (GPU suite minus sanitizer) + network A/B over LASNET_TC_PAIR.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -15
for V in 0 1 3 7; do
LASNET_TC_PAIR=$V timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-block --no-regnet --detail gpurun_out/det_p$V.json > gpurun_out/bench_p$V.json 2> gpurun_out/bench_p$V.err
echo "PAIR=$V rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_p$V.json'))
k=d['kernels']
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['dense_identity_ms_per_step'], {n: (k[n]['ms'], k[n]['frac']) for n in k}, d['eager_breakdown_ms'])
" || tail -5 gpurun_out/bench_p$V.err
done
