#!/bin/bash
mkdir -p gpurun_out
TRD_TC_TIMING=1 TRD_TC_NOEPI=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/timing_noepi.log 2>&1; echo rc=$?
grep -A16 "tc timing" gpurun_out/timing_noepi.log | head -18
python scripts/show_bench.py gpurun_out/timing_noepi.log | head -1
