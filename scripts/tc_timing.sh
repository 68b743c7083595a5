#!/bin/bash
mkdir -p gpurun_out
TRD_TC_TIMING=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/timing_c5b.log 2>&1; echo rc=$?
grep -A10 "tc timing" gpurun_out/timing_c5b.log | head -24
