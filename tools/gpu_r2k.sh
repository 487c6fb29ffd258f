#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "stem_maxpool_head" --timeout 300 2>&1 | tail -1
for V in "" "LASNET_CONV1_BN=128"; do
env $V timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-regnet --no-block > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err
echo "$V"; python -c "
import json; d=json.load(open('gpurun_out/bench_k.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['kernels']['head'], d['kernels']['conv1_mask'], d['eager_breakdown_ms'])
"
done
