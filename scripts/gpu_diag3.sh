#!/bin/bash
# pass-kernel timing under TRD_TC_EXP experiments (results invalid; timing only)
mkdir -p gpurun_out
for E in ${EXPS:-1 7}; do
  TRD_TC_EXP=$E timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/d3_exp$E.log 2>&1
  echo "exp=$E rc=$? $(python scripts/show_bench.py gpurun_out/d3_exp$E.log 2>/dev/null | head -1 | grep -o 'p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
  grep -A7 "tc exp" gpurun_out/d3_exp$E.log | head -8
done
