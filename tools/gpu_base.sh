#!/bin/bash
# Baseline session run: build, GPU tests (with durations), smoke, default bench.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
nproc > gpurun_out/nproc.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q --durations=25 2>&1 | tail -60 > gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout -s KILL 900 python bench.py --detail gpurun_out/bench_detail.json > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -8 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; head -c 3000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
