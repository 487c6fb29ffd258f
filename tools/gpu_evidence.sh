#!/bin/bash
# Round evidence in one call: ncu launch lists + full captures (tools/prof_r2.sh), then the
# default bench line (no profiler) and the GPU test suite.
mkdir -p gpurun_out
bash tools/prof_r2.sh > gpurun_out/prof.log 2>&1
tail -3 gpurun_out/prof.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_final.json
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
