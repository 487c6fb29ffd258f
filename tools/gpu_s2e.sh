#!/bin/bash
# A-operand L2 prefetch distance A/B (dense conv1 / conv1+masker / dense conv3), pairs for conv2 only.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "network or dense" 2>&1 | tail -2
LASNET_A_PF=4 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "network or dense" 2>&1 | tail -2
for V in 0 2 4 8 16; do
LASNET_A_PF=$V timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-block --no-regnet --detail gpurun_out/det_pf$V.json > gpurun_out/bench_pf$V.json 2> gpurun_out/bench_pf$V.err
echo "PF=$V rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_pf$V.json'))
k=d['kernels']
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['dense_identity_ms_per_step'], {n: k[n]['ms'] for n in list(k)[:7]})
" || tail -5 gpurun_out/bench_pf$V.err
done
python tools/stage_kernels.py gpurun_out/det_pf0.json gpurun_out/det_pf8.json | grep -E " 2 |forward"
