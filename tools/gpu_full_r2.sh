#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1
timeout -s KILL 3000 python -m pytest tests -m gpu -q --timeout 1500 > gpurun_out/pytest_full.log 2>&1
tail -30 gpurun_out/pytest_full.log | cut -c1-400
