#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1
timeout -s KILL 300 python tools/dbg_proj.py > gpurun_out/dbg_proj.log 2>&1; cat gpurun_out/dbg_proj.log
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 \
  -k "proj or network or stem" > gpurun_out/pytest_r2c.log 2>&1
tail -40 gpurun_out/pytest_r2c.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --detail gpurun_out/bench_detail_r2c.json > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
tail -c 2000 gpurun_out/bench_r2c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r2c.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['dense_identity_ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['network_roofline']['frac_schedule'])
print(json.dumps(d['kernels'])[:2500]); print(d['eager_breakdown_ms']); print(d['stats']['r_patch_per_block'])
"
