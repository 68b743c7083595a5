#!/bin/bash
mkdir -p gpurun_out
./scripts/microbench/tc_rate x > gpurun_out/tc_rate_sbo.log 2>&1; cat gpurun_out/tc_rate_sbo.log
for E in 0 32; do
  TRD_UNIT=1 TRD_TC_EXP=$E timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/d5_u1_e$E.log 2>&1
  echo "unit=1 exp=$E rc=$? $(python scripts/show_bench.py gpurun_out/d5_u1_e$E.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
done
