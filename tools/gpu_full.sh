#!/bin/bash
# Full GPU check: all -m gpu tests, smoke, and both schedules' bench lines (+ no-PDL A/B).
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > /dev/null
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout -s KILL 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
for sch in fused separate; do
  timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --schedule $sch > gpurun_out/bench_$sch.json 2> gpurun_out/bench_$sch.err
done
LASNET_PDL=1 timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --schedule fused > gpurun_out/bench_nopdl.json 2> gpurun_out/bench_nopdl.err
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
for sch in fused separate nopdl; do python - <<PY
import json
try:
    d=json.load(open("gpurun_out/bench_$sch.json"))
    print("$sch", d["value"], d["ms_per_step"], d["kernels_ms"], "dense", d["dense_ms_per_step"], "speedup", d["speedup_vs_dense"], "roof", d["roofline"]["kernel"], d["roofline"]["frac"], "block", d["block_roofline"]["frac_time"])
except Exception as e:
    print("$sch failed", e); print(open("gpurun_out/bench_$sch.err").read()[-3000:])
PY
done
