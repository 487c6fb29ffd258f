#!/bin/bash
# conv23 opt-in variants on the S = 1 / 2 sweep points (the gathered conv23 path).
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for V in "" "LASNET_C23_PAIR=1" "LASNET_C23_CLUSTER=2" "LASNET_C23_CLUSTER=4"; do
  for S in 1 2; do
    env $V timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-regnet --s $S --schedule fused > gpurun_out/b_$S.json 2> gpurun_out/b_$S.err
    python -c "
import json; d=json.load(open('gpurun_out/b_$S.json')); b=d['block']; print('[$V] S=$S', b['ms_per_step'], b['kernels_ms'])" || tail -3 gpurun_out/b_$S.err
  done
done
