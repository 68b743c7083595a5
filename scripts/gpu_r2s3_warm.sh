#!/bin/bash
# session 3: warm-cache launch lists (ncu --cache-control none) of the latency configs
mkdir -p gpurun_out/s3
O=gpurun_out/s3
for C in C4 C5a; do
  A="bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/warm_$C.csv python $A > $O/warm_ncu_$C.log 2>&1
  python scripts/launch_share.py $O/warm_$C.csv > $O/warm_share_$C.txt 2>&1
  grep "trd::\|CUB\|TOTAL" $O/warm_share_$C.txt | head -40
done
