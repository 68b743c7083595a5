#!/bin/bash
# tcgen05 data-dependence microbenchmark + pass-kernel timing with the epilogue disabled
mkdir -p gpurun_out
timeout 120 ./scripts/microbench/tc_data > gpurun_out/tc_data.log 2>&1; echo data=$?
cat gpurun_out/tc_data.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/d2_c5b.log 2>&1; echo rc=$?
python scripts/show_bench.py gpurun_out/d2_c5b.log 2>/dev/null | head -2
TRD_TC_EXP=1 timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/d2_c5b_exp1.log 2>&1; echo rc=$?
python scripts/show_bench.py gpurun_out/d2_c5b_exp1.log 2>/dev/null | head -2
