#!/bin/bash
# one ncu --set full capture of a pass kernel (C5b) + source page export
mkdir -p gpurun_out
T=${1:-n1}; K=${2:-tc_pass1}
CMD="python bench.py --config C5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/${T}_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s 2 -c 1 -o gpurun_out/${T} $CMD > gpurun_out/${T}_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${T}.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_src.csv 2>/dev/null
ncu -i gpurun_out/${T}.ncu-rep --page details --csv > gpurun_out/${T}_details.csv 2>/dev/null
ncu -i gpurun_out/${T}.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
ls -la gpurun_out/${T}*
