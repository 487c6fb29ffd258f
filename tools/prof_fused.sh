#!/bin/bash
# ncu evidence for the masker-fused schedule: launch list (time + DRAM bytes) and
# one --set full capture of each of its kernels. usage: tools/prof_fused.sh TAG
TAG=${1:-f1}
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > /dev/null
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --schedule fused > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
   -k regex:"conv_tc_kernel|conv23_kernel|decide|gather" -s 4 -c 4 -o gpurun_out/full_${TAG} \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --schedule fused > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}.log
