#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "stem or network" --timeout 900 2>&1 | tail -2
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-block > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err
python -c "
import json; d=json.load(open('gpurun_out/bench_l.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['kernels']['head'], d['kernels']['stem_conv'], d['regnet'])
"
