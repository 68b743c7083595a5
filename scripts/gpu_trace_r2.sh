#!/bin/bash
# pass-1 per-tile event trace (experiments build) and epilogue-free timing, C5b
mkdir -p gpurun_out
export TRD_LIB_PATH=$PWD/abtest/libtrd_exp.so
TRD_GRAPH=0 TRD_TC_EXP=8 timeout 300 python bench.py --config C5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/tr_C5b.log 2>&1; echo "trace rc=$?"
grep -A30 "tc trace\]" gpurun_out/tr_C5b.log | head -32
for E in 0 1 4 5; do
  TRD_TC_EXP=$E timeout 300 python bench.py --config C5b --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/exp_$E.log 2>&1
  echo "exp=$E rc=$? $(python scripts/show_bench.py gpurun_out/exp_$E.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
done
