#!/bin/bash
mkdir -p gpurun_out
for UN in ${UNITS:-1 2}; do
for E in ${EXPS:-8}; do
TRD_UNIT=$UN TRD_TC_EXP=$E timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/trace_u${UN}_exp$E.log 2>&1; echo rc=$?
grep -A50 "tc trace" gpurun_out/trace_u${UN}_exp$E.log | head -52
done
done
