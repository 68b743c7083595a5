#!/bin/bash
# A/B: abtest/libtrd_head.so (previous commit) vs the in-tree library, C5b, same box
mkdir -p gpurun_out
for R in 1 2; do
for L in head cur; do
  if [ $L = head ]; then export TRD_LIB_PATH=$PWD/abtest/libtrd_head.so; else unset TRD_LIB_PATH; fi
  for UN in ${UNITS:-1}; do
  TRD_UNIT=$UN timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ab_${L}_u$UN.log 2>&1
  echo "lib=$L unit=$UN rc=$? $(python scripts/show_bench.py gpurun_out/ab_${L}_u$UN.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
  done
done
done
