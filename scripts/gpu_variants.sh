#!/bin/bash
# C5b timing of kernel variants built into abtest/libtrd_<v>.so (plus the in-tree library)
mkdir -p gpurun_out
for L in cur ${VARIANTS}; do
  if [ $L = cur ]; then unset TRD_LIB_PATH; else export TRD_LIB_PATH=$PWD/abtest/libtrd_$L.so; fi
  for UN in ${UNITS:-1 2}; do
    TRD_UNIT=$UN timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline ${BARGS} > gpurun_out/var_${L}_u$UN.log 2>&1
    echo "lib=$L unit=$UN rc=$? $(python scripts/show_bench.py gpurun_out/var_${L}_u$UN.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
  done
done
