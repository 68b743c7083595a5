#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config C5b --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/st_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none -k "regex:stage_bits|stage_vals" -c 4 -o gpurun_out/st_full $CMD > gpurun_out/st_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/st_full.ncu-rep --page details --csv > gpurun_out/st_details.csv 2>/dev/null
