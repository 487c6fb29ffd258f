#!/bin/bash
# conv1_mask masker-coupling probes at the stage-3 shape (launch lists under env variants) + dense conv1
mkdir -p gpurun_out
python -m paper_2210_06223_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
M=gpu__time_duration.sum
i=0
for V in "$@"; do
[ "$V" = "-" ] && V="A=1"
env $V timeout -s KILL 300 ncu --metrics $M --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/ll$i.csv python tools/stage3_once.py $ARGS > /dev/null 2>&1
echo "[$V]"; python -c "
import csv
r=list(csv.reader(open('gpurun_out/ll$i.csv')))
r=[x for x in r if len(x)>5]
h=r[0]; iK=h.index('Kernel Name'); iM=h.index('Metric Name'); iV=h.index('Metric Value')
print('  '.join(x[iK][:28].replace('void ','')+' '+x[iV] for x in r[1:] if x[iM]=='gpu__time_duration.sum'))
"
i=$((i+1))
done
