python -m paper_2210_06223_b200.build >/dev/null
for m in 0 1; do LASNET_DG_DEBUG=$m python bench.py --steps 20 --warmup 5 --no-cpu-baseline --schedule fused 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg $m', d['kernels_ms'], d['ms_per_step'])"; done
