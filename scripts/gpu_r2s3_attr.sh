#!/bin/bash
# session 3: pass-1 epilogue attribution (experiments builds, results invalid): TRD_P1_X bit 0 no
# weight stores, 1 no P stores, 2 no exp, 3 no S reads; C5b pass-1 time and the per-tile trace
mkdir -p gpurun_out/s3
O=gpurun_out/s3
for X in exp x1 x2 x4 x8 x15; do
  export TRD_LIB_PATH=$PWD/abtest/libtrd_$X.so
  timeout 300 python bench.py --config C5b --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $O/attr_$X.log 2>&1
  echo "$X rc=$? $(python scripts/show_bench.py $O/attr_$X.log 2>/dev/null | head -1 | grep -o 'p1/sweep=[0-9.]*ms p2/sweep=[0-9.]*ms')"
  TRD_GRAPH=0 TRD_TC_EXP=8 timeout 300 python bench.py --config C5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/attr_tr_$X.log 2>&1
  grep -A14 "tc trace\]" $O/attr_tr_$X.log | tail -6
done
