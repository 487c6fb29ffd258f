#!/bin/bash
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for ns in 2 3 4; do timeout -s KILL 300 python tools/split_probe.py $ns 2>&1 | tail -3; done
echo "PDL=0"; LASNET_PDL=0 timeout -s KILL 300 python tools/split_probe.py 2 2>&1 | tail -3
