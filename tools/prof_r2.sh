#!/bin/bash
# Round-2 evidence: (1) the launch list of the bench command, (2) a launch list with DRAM
# bytes of one eager LAS-R101 forward (every kernel named via the library's events),
# (3) ncu --set full of the network's main kernels at their stage-3 shapes and of the
# block workload's conv23 / conv1_mask.  One GPU.
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_r2.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweep --no-coco --no-regnet > gpurun_out/ncu_bench_r2.log 2>&1
echo bench-launches rc=$?
timeout -s KILL 900 ncu --metrics $M --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_net_r2.csv \
   python tools/net_once.py --names gpurun_out/net_once_names.json > gpurun_out/ncu_net_r2.log 2>&1
echo net-launches rc=$?
timeout -s KILL 900 ncu --metrics $M --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_regnet_r2.csv \
   python tools/net_once.py --regnet --n 512 --names gpurun_out/regnet_once_names.json > gpurun_out/ncu_regnet_r2.log 2>&1
echo regnet-launches rc=$?
# full captures: stage-3 kernels of the network (launch-skip past stages 0-1)
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"conv_tc_kernel|conv23_kernel|decide_kernel|compact_gather_kernel|masker_compact_kernel" \
   --launch-skip 30 -c 10 -o gpurun_out/full_net_r2 python tools/net_once.py --names gpurun_out/net_once_names_full.json > gpurun_out/ncu_full_net_r2.log 2>&1
echo full-net rc=$?
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"conv_tc_kernel|conv23_kernel|decide_kernel|masker_compact_kernel" -o gpurun_out/full_block_r2 \
   python tools/block_once.py > gpurun_out/ncu_full_block_r2.log 2>&1
echo full-block rc=$?
ls -la gpurun_out/*.ncu-rep
