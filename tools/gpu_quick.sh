#!/bin/bash
# Quick GPU iteration: selected parity tests + bench lines for both schedules.
# usage: tools/gpu_quick.sh "<pytest -k expr>" [extra bench args]
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > /dev/null
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "${1:-block_forward}" 2>&1 | tail -15 > gpurun_out/pytest_quick.log
for sch in fused separate; do
  timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --schedule $sch $2 > gpurun_out/bench_$sch.json 2> gpurun_out/bench_$sch.err
done
cat gpurun_out/pytest_quick.log
for sch in fused separate; do python - <<PY
import json
try:
    d=json.load(open("gpurun_out/bench_$sch.json"))
    print("$sch", d["value"], d["ms_per_step"], d["kernels_ms"], "dense", d["dense_ms_per_step"], "speedup", d["speedup_vs_dense"], "roof", d["roofline"]["kernel"], d["roofline"]["frac"], "block", d["block_roofline"]["frac_time"], d["block_roofline"].get("schedule_roofline"))
except Exception as e:
    print("$sch failed", e); print(open("gpurun_out/bench_$sch.err").read()[-3000:])
PY
done
