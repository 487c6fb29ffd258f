#!/bin/bash
# Build-variant A/B: bash tools/gpu_ab_build.sh "<nvcc -D flags>|<env>" ...  ('-' = none).
# Rebuilds liblasnet.so per variant (forced), one network bench line each; restores the
# default build at the end.  PYTEST_K: parity subset on the default build first.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build --force > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
if [ -n "$PYTEST_K" ]; then
  timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "$PYTEST_K" 2>&1 | tail -4
fi
i=0
for V in "$@"; do
  B="${V%%|*}"; E="${V#*|}"
  [ "$B" = "-" ] && B=""; [ "$E" = "-" ] && E=""
  LASNET_EXTRA_NVCC="$B" python -m paper_2210_06223_b200.build --force > gpurun_out/build_v$i.log 2>&1 || tail -5 gpurun_out/build_v$i.log
  env $E timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-coco --no-regnet ${BENCH_ARGS:---no-block} --detail gpurun_out/det_v$i.json > gpurun_out/bench_v$i.json 2> gpurun_out/bench_v$i.err
  echo "[$B | $E] rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_v$i.json'))
k=d['kernels']
print(d['value'], d['ms_per_step'], 'x%.3f' % d['speedup_vs_dense'], 'dense', d['dense_identity_ms_per_step'], {n: k[n]['ms'] for n in list(k)[:6]})
b=d.get('block')
if b: print('  block', b['ms_per_step'], b['kernels_ms'], 'dense', b.get('dense_ms_per_step'))
" || tail -5 gpurun_out/bench_v$i.err
  i=$((i+1))
done
python -m paper_2210_06223_b200.build --force > /dev/null 2>&1
