#!/bin/bash
# Driver-like round-end sequence on one GPU: build, GPU tests, smoke, default bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python bench.py > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_check.json')); print(d['value'], d['ms_per_step'], d['speedup_vs_dense'], d['e2e']['value'], d['block']['ms_per_step'], d['clocks'])"
