#!/bin/bash
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 300 python bench.py --config C5b --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/tp4_C5b.log 2>&1
echo "C5b rc=$? $(python scripts/show_bench.py $O/tp4_C5b.log 2>/dev/null | head -1 | cut -c1-220)"
TRD_LIB_PATH=$PWD/abtest/libtrd_exp.so TRD_GRAPH=0 TRD_TC_EXP=8 timeout 300 python bench.py --config C5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/tr4.log 2>&1; echo "trace rc=$?"
grep -A30 "tc trace\]" $O/tr4.log | head -32
