#!/bin/bash
# conv23 variants: conv2 ring depth x H2 buffers (parity of each variant on the full-size block test)
mkdir -p gpurun_out
for V in "3 1" "2 2" "2 1"; do
  set -- $V
  LASNET_EXTRA_NVCC="-DLASNET_C23_STAGES=$1 -DLASNET_C23_H2BUFS=$2" python -c "from paper_2210_06223_b200 import build; build.build(force=True)" > gpurun_out/build_ab.log 2>&1 || tail -20 gpurun_out/build_ab.log
  timeout -s KILL 600 python tools/block_ab.py "st$1_h2$2" 2>&1 | tail -1
  timeout -s KILL 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "full_tensor and 4" --timeout 300 2>&1 | tail -1
done
python -c "from paper_2210_06223_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "stem_maxpool_head or network_batch" --timeout 300 2>&1 | tail -1
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-regnet --no-block > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
python -c "
import json; d=json.load(open('gpurun_out/bench_ab.json'))
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['kernels']['head'])
"
