#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -30 gpurun_out/build.log
timeout -s KILL 600 python tools/regnet_breakdown.py > gpurun_out/regnet_breakdown.txt 2>&1; cat gpurun_out/regnet_breakdown.txt
timeout -s KILL 1800 python -m pytest tests/test_gpu_regnet.py -m gpu -q --timeout 900 -k layerwise > gpurun_out/pytest_r2g.log 2>&1
tail -5 gpurun_out/pytest_r2g.log | cut -c1-400
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-block --no-coco --no-regnet --detail gpurun_out/bench_detail_r2g.json > gpurun_out/bench_r2g.json 2> gpurun_out/bench_r2g.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r2g.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['kernels']['conv2_dyn'], d['eager_breakdown_ms'])
"
LASNET_CONV2_BN=128 timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-block --no-coco --no-regnet > gpurun_out/bench_r2g128.json 2> gpurun_out/bench_r2g128.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r2g128.json'))
print('BN128', d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['kernels']['conv2_dyn'], d['eager_breakdown_ms'])
"
