#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpu_tests.sh 1500
bash scripts/gpu_bench_all.sh r2e
for G in 0 1; do
  TRD_GRAPH=$G timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2e_C1_g$G.log 2>&1
  echo "C1 graph=$G $(python scripts/show_bench.py gpurun_out/r2e_C1_g$G.log 2>/dev/null | head -1 | cut -c1-200)"
done
for C in C1 C4; do
  A="bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_${C}_launches.csv python $A > gpurun_out/r2e_${C}_ncu.log 2>&1
  python scripts/launch_share.py gpurun_out/r2e_${C}_launches.csv > gpurun_out/r2e_${C}_share.txt 2>&1
done
