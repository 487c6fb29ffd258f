#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
LASNET_TC_PAIR=9 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "fused or network or stage3 or full_tensor" 2>&1 | tail -2
bash tools/gpu_ab_net.sh - LASNET_TC_PAIR=9
