#!/bin/bash
# GPU check + A/B of an env toggle: all -m gpu tests, then bench lines for both
# schedules with and without the toggle.  usage: tools/gpu_ab.sh "ENV=1" [bench args]
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > /dev/null
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for sch in fused separate; do
  for tog in "" "$1"; do
    env $tog timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --schedule $sch $2 > gpurun_out/ab.json 2> gpurun_out/ab.err
    python - "$sch" "$tog" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/ab.json"))
    print(sys.argv[1], sys.argv[2] or "default", d["ms_per_step"], {k: round(v*1e3, 1) for k, v in d["kernels_ms"].items()},
          "dense", d["dense_ms_per_step"], "x", d["speedup_vs_dense"], "block", d["block_roofline"]["frac_time"])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e); print(open("gpurun_out/ab.err").read()[-2000:])
PY
  done
done
