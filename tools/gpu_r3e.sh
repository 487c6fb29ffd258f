#!/bin/bash
# decide CTA size A/B (builds the library twice): 256 (default) then 128 threads, network bench + e2e check
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or Fused" 2>&1 | tail -2
BENCH_ARGS="--no-coco --no-regnet" bash tools/gpu_ab_net.sh -
sed -i 's/^constexpr int kDecThreads = 256;/constexpr int kDecThreads = 128;/' paper_2210_06223_b200/csrc/decide_gather.cu
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
echo "== 128-thread decide"
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or Fused" 2>&1 | tail -2
BENCH_ARGS="--no-coco --no-regnet" bash tools/gpu_ab_net.sh -
