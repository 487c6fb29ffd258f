#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -30 gpurun_out/build.log
timeout -s KILL 1800 python -m pytest tests/test_gpu_regnet.py -m gpu -q --timeout 900 > gpurun_out/pytest_r2i.log 2>&1
tail -5 gpurun_out/pytest_r2i.log | cut -c1-400
timeout -s KILL 600 python tools/regnet_breakdown.py > gpurun_out/regnet_breakdown3.txt 2>&1; head -16 gpurun_out/regnet_breakdown3.txt; grep -A10 "^dense" gpurun_out/regnet_breakdown3.txt
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err
tail -c 1000 gpurun_out/bench_r2i.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r2i.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['regnet'], d['config1'], d['block']['ms_per_step'], d['block']['speedup_vs_dense'])
"
