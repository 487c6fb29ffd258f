#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -k "proj_dyn" 2>&1 | tail -2
for V in "" "LASNET_PROJ_MASK_FUSED=1"; do
env $V timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-block --no-regnet > gpurun_out/bench_n.json 2> gpurun_out/bench_n.err
echo "$V"; python -c "
import json; d=json.load(open('gpurun_out/bench_n.json'))
k=d['kernels']
print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], {n: k[n]['ms'] for n in ('mask','compact','mask_compact') if n in k}, d['eager_breakdown_ms'])
"
done
