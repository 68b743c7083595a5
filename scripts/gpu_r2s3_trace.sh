#!/bin/bash
# session 3: pass-1 per-tile trace of CTA 0 (experiments build), C5b
mkdir -p gpurun_out/s3
export TRD_LIB_PATH=$PWD/abtest/libtrd_exp.so
TRD_GRAPH=0 TRD_TC_EXP=8 timeout 300 python bench.py --config C5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s3/tr_C5b.log 2>&1; echo "trace rc=$?"
grep -A80 "tc trace\]" gpurun_out/s3/tr_C5b.log | head -82
