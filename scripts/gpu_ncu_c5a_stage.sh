#!/bin/bash
# ncu --set full of the C5a staging kernels (sampled sketch, fibre windows)
mkdir -p gpurun_out
CMD="python bench.py --config C5a --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
for K in stage_bits stage_vals; do
  TRD_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s 3 -c 1 -o gpurun_out/c5a_$K $CMD > gpurun_out/c5a_${K}_ncu.log 2>&1; echo "$K ncu=$?"
  ncu -i gpurun_out/c5a_$K.ncu-rep --page details --csv > gpurun_out/c5a_${K}_details.csv 2>/dev/null
done
