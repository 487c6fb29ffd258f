#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1
timeout -s KILL 300 python tools/dbg_proj.py > gpurun_out/dbg_proj.log 2>&1; cat gpurun_out/dbg_proj.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --detail gpurun_out/bench_detail_r2b.json > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
tail -c 2000 gpurun_out/bench_r2b.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r2b.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['roofline'], d['network_roofline'])
print(json.dumps(d['kernels'])[:2000]); print(d['eager_breakdown_ms']); print(d.get('block',{}).get('ms_per_step'), d.get('e2e'), d.get('cpu_baseline'))
"
timeout -s KILL 1800 python -m pytest tests/test_sanitizer.py -m gpu -q --timeout 1700 > gpurun_out/pytest_san.log 2>&1
tail -30 gpurun_out/pytest_san.log
