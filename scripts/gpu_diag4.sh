#!/bin/bash
# C5b pass-kernel timing: ring unit (TRD_UNIT) x TRD_TC_EXP experiments (timing only)
mkdir -p gpurun_out
for UN in ${UNITS:-2 1}; do
for E in ${EXPS:-0 1 6}; do
  TRD_UNIT=$UN TRD_TC_EXP=$E timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/d4_u${UN}_e$E.log 2>&1
  echo "unit=$UN exp=$E rc=$? $(python scripts/show_bench.py gpurun_out/d4_u${UN}_e$E.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
done
done
