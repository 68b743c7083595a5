#!/bin/bash
mkdir -p gpurun_out
run() { # lib exp
  if [ $1 = cur ]; then unset TRD_LIB_PATH; else export TRD_LIB_PATH=$PWD/abtest/libtrd_$1.so; fi
  TRD_TC_EXP=$2 timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/p2e_$1_$2.log 2>&1
  echo "lib=$1 exp=$2 rc=$? $(python scripts/show_bench.py gpurun_out/p2e_$1_$2.log 2>/dev/null | head -1 | grep -o 'p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
}
run cur 0; run cur 4; run cur 2; run cur 1; run nsu4 0; run nsu4 4
