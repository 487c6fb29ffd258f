#!/bin/bash
# Round-2 check: new full-size / signed / balanced / network-224 parity, sanitizer tier, bench line.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q --timeout 900 \
  -k "full_tensor or signed or balanced or network" > gpurun_out/pytest_r2a.log 2>&1
tail -30 gpurun_out/pytest_r2a.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --detail gpurun_out/bench_detail_r2a.json > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
tail -c 3000 gpurun_out/bench_r2a.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r2a.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['roofline'], d['network_roofline'])
print(json.dumps(d['kernels'])[:2000]); print(d['eager_breakdown_ms']); print(d.get('block',{}).get('ms_per_step'), d.get('e2e'), d.get('cpu_baseline'))
"
timeout -s KILL 1800 python -m pytest tests/test_sanitizer.py -m gpu -q --timeout 1700 > gpurun_out/pytest_san.log 2>&1
tail -30 gpurun_out/pytest_san.log
