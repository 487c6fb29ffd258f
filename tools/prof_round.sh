#!/bin/bash
# Round evidence: ncu launch list of the bench command + one --set full capture
# of each kernel of the dynamic step and of the dense comparator (1 GPU).
TAG=${1:-r1}
mkdir -p gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on \
   -k regex:"conv_tc_kernel|conv23_kernel|masker_compact_kernel" -s 3 -c 6 -o gpurun_out/full_${TAG} \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
