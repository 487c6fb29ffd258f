#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_regnet.py -m gpu -q --timeout 900 -k "dense or proj or network or static or all_ones or variants" 2>&1 | tail -3
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-block > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err
python -c "
import json; d=json.load(open('gpurun_out/bench_m.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['dense_identity_ms_per_step'], d['kernels']['shortcut'], d['eager_breakdown_ms'], d['regnet'])
"
