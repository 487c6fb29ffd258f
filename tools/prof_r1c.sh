#!/bin/bash
# Round evidence for both schedules: launch list (time + DRAM bytes) of the bench
# command and one --set full capture of each kernel.  usage: tools/prof_r1c.sh TAG
TAG=${1:-r1c}
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > /dev/null
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_${TAG}.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --network 0 --schedule fused > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
   --log-file gpurun_out/launches_${TAG}_sep.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --network 0 --schedule separate > gpurun_out/ncu_launch_${TAG}_sep.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
   -k regex:"conv_tc_kernel|conv23_kernel|decide|gather|compact_idx|masker" -s 8 -c 8 -o gpurun_out/full_${TAG} \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --network 0 --schedule fused > gpurun_out/ncu_full_${TAG}.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
   -k regex:"masker_compact|conv_tc_kernel" -s 4 -c 2 -o gpurun_out/full_${TAG}_sep \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --network 0 --schedule separate > gpurun_out/ncu_full_${TAG}_sep.log 2>&1
cat gpurun_out/pytest_${TAG}.log; tail -2 gpurun_out/ncu_full_${TAG}.log
