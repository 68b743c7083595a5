#!/bin/bash
# session 3: where the latency-bound configs spend a sweep (bench lines + serialised launch lists)
mkdir -p gpurun_out/s3
O=gpurun_out/s3
for C in C4 C5a; do
  timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py $O/bench_$C.log 2>/dev/null | head -1 | cut -c1-200)"
  A="bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$C.csv python $A > $O/ncu_$C.log 2>&1
  python scripts/launch_share.py $O/launches_$C.csv > $O/share_$C.txt 2>&1
  head -45 $O/share_$C.txt
done
