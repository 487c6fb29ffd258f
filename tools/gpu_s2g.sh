#!/bin/bash
# ncu --set full of the stage-3 wide conv23 (dynamic + dense).
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"conv23_kernel" -o gpurun_out/s3_wide python tools/stage3_once.py > gpurun_out/ncu_s3_wide.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_s3_wide.log
