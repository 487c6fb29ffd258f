#!/bin/bash
# ncu --set full of the stage-3 block's conv_tc kernels, without / with CTA pairs.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for V in 0 9; do
LASNET_TC_PAIR=$V timeout -s KILL 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"conv_tc_kernel|decide|compact_gather" -o gpurun_out/s3_p$V python tools/stage3_once.py > gpurun_out/ncu_s3_p$V.log 2>&1
echo "p$V rc=$?"; tail -2 gpurun_out/ncu_s3_p$V.log
done
ls -la gpurun_out/*.ncu-rep
