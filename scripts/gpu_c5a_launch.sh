#!/bin/bash
mkdir -p gpurun_out/c5a
O=gpurun_out/c5a
for C in C5a C4; do
A="bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
TRD_GRAPH=0 timeout 300 python $A > $O/plain_$C.log 2>&1 && \
TRD_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$C.csv python $A > $O/ncu_$C.log 2>&1
python scripts/launch_share.py $O/launches_$C.csv > $O/share_$C.txt 2>&1
echo "$C"; head -40 $O/share_$C.txt
done
