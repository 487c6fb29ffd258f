#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_regnet.py -m gpu -x -q 2>&1 | tail -2
for V in "" "LASNET_REG_GATHER=1"; do
  env $V timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-block > gpurun_out/b_r.json 2> gpurun_out/b_r.err
  python -c "
import json; d=json.load(open('gpurun_out/b_r.json')); r=d['regnet']; print('[$V]', r['ms_per_forward'], r['images_per_s'], r['speedup_vs_dense'])" || tail -3 gpurun_out/b_r.err
done
