#!/bin/bash
# ncu --set full capture of the conv kernels of the bench workload (1 GPU).
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tc_kernel|masker_kernel|compact_kernel" -s 4 -c 8 -o gpurun_out/prof_${1:-r1} python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_${1:-r1}.log 2>&1
tail -3 gpurun_out/prof_${1:-r1}.log
