#!/bin/bash
# tcgen05 rate microbenchmark + per-role cycle accounting of the pass-1 kernel (C5b, C4)
mkdir -p gpurun_out
timeout 120 ./scripts/microbench/tc_rate > gpurun_out/tc_rate.log 2>&1; echo rate=$?
cat gpurun_out/tc_rate.log
for NOEPI in 0 1; do
  if [ $NOEPI = 1 ]; then export TRD_TC_NOEPI=1; fi
  TRD_TC_TIMING=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/timing_c5b_$NOEPI.log 2>&1; echo rc=$?
  grep -A16 "tc timing" gpurun_out/timing_c5b_$NOEPI.log | head -18
  python scripts/show_bench.py gpurun_out/timing_c5b_$NOEPI.log | head -3
done
