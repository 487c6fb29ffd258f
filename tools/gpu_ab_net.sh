#!/bin/bash
# Network A/B: bash tools/gpu_ab_net.sh "ENV=1 ENV2=0" "ENV=0" ...  (one bench line per variant;
# the first quoted arg may be "-" for the default).  Set PYTEST_K to run a parity subset first.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
if [ -n "$PYTEST_K" ]; then
  timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "$PYTEST_K" 2>&1 | tail -4
fi
i=0
for V in "$@"; do
  [ "$V" = "-" ] && V=""
  env $V timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline ${BENCH_ARGS:---no-coco --no-block --no-regnet} --detail gpurun_out/det_ab$i.json > gpurun_out/bench_ab$i.json 2> gpurun_out/bench_ab$i.err
  echo "[$V] rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_ab$i.json'))
k=d['kernels']
print(d['value'], d['ms_per_step'], 'x%.3f' % d['speedup_vs_dense'], 'dense', d['dense_identity_ms_per_step'], {n: k[n]['ms'] for n in list(k)[:7]})
b=d.get('block')
if b: print('  block', b['ms_per_step'], b['kernels_ms'], 'dense', b.get('dense_ms_per_step'))
if d.get('regnet'): print('  regnet', d['regnet'].get('ms_per_forward'), d['regnet'].get('speedup_vs_dense'))
if d.get('coco_backbone'): print('  coco', {k: (v.get('ms_per_forward'), v.get('speedup_vs_dense')) for k, v in d['coco_backbone'].items() if isinstance(v, dict)})
if d.get('config1'): print('  config1', d['config1'].get('us_per_block'), d['config1'].get('dense_us'))
" || tail -5 gpurun_out/bench_ab$i.err
  i=$((i+1))
done
