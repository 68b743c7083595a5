#!/bin/bash
# pass-kernel floors: timing experiments of the experiments build (results invalid), C5b
mkdir -p gpurun_out
export TRD_LIB_PATH=$PWD/abtest/libtrd_exp.so
for E in ${EXPS:-0 2 4 6 1 3 5 7 16}; do
  TRD_TC_EXP=$E timeout 300 python bench.py --config ${CFG:-C5b} --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/xd_$E.log 2>&1
  echo "exp=$E rc=$? $(python scripts/show_bench.py gpurun_out/xd_$E.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
done
