#!/bin/bash
mkdir -p gpurun_out
run() { # lib unit exp
  if [ $1 = cur ]; then unset TRD_LIB_PATH; else export TRD_LIB_PATH=$PWD/abtest/libtrd_$1.so; fi
  TRD_UNIT=$2 TRD_TC_EXP=$3 timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/e6_$1_u$2_e$3.log 2>&1
  echo "lib=$1 unit=$2 exp=$3 rc=$? $(python scripts/show_bench.py gpurun_out/e6_$1_u$2_e$3.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
}
run v1 1 0; run v1 2 0; run v2 1 0; run v2 2 0
run cur 1 1; run cur 1 3; run cur 2 1; run cur 2 3
run v3 1 1; run v3 2 1
