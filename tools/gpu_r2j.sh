#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"conv_tc_kernel|conv23_kernel|decide_kernel|masker_compact_kernel|compact_idx" -o gpurun_out/full_block_r2 -f \
   python tools/block_once.py > gpurun_out/ncu_full_block_r2.log 2>&1
echo full-block rc=$?
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-regnet --no-block --detail gpurun_out/bench_detail_r2j.json > gpurun_out/bench_r2j.json 2> gpurun_out/bench_r2j.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r2j.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['kernels']['head'], d['roofline'])
"
