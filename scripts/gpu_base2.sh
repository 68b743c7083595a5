#!/bin/bash
# round-2 baseline: one bench line per config, launch lists of C4 and C5a
mkdir -p gpurun_out
bash scripts/gpu_allcfg.sh base
for C in C4 C5a; do
  A="bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 300 python $A > gpurun_out/${C}_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${C}_launches.csv python $A > gpurun_out/${C}_ncu.log 2>&1
  python scripts/launch_share.py gpurun_out/${C}_launches.csv > gpurun_out/${C}_share.txt 2>&1
done
