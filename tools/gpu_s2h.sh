#!/bin/bash
# A-stationary conv3: parity under LASNET_C3_GROUP in {2, 4, 8}, then network A/B.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for G in 2 4 8; do
  echo "G=$G"; LASNET_C3_GROUP=$G timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "stage3 or 1024 or 2048 or dense or network or variants" 2>&1 | tail -2
done
bash tools/gpu_ab_net.sh - LASNET_C3_GROUP=2 LASNET_C3_GROUP=4 LASNET_C3_GROUP=8
