#!/bin/bash
# session 3: TMEM P -- NE = 3 epilogue warpgroups (A/B library) and per-tile traces of both
mkdir -p gpurun_out/s3
O=gpurun_out/s3
TRD_LIB_PATH=$PWD/abtest/libtrd_ne3.so timeout 300 python bench.py --config C5b --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/tp3_C5b.log 2>&1
echo "NE3 C5b rc=$? $(python scripts/show_bench.py $O/tp3_C5b.log 2>/dev/null | head -1 | cut -c1-220)"
for L in exp exp3; do
  TRD_LIB_PATH=$PWD/abtest/libtrd_$L.so TRD_GRAPH=0 TRD_TC_EXP=8 timeout 300 python bench.py --config C5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/tr_$L.log 2>&1; echo "trace $L rc=$?"
  grep -A40 "tc trace\]" $O/tr_$L.log | head -42
done
