#!/bin/bash
# staging cost in the e2e path (C5b): per-stage timeline of the host-resident context
mkdir -p gpurun_out
TRD_TIMELINE=1 timeout 600 python bench.py --config C5b --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/st_C5b.log 2>&1
echo "rc=$?"; grep -A25 "trd timeline" gpurun_out/st_C5b.log | grep "stage\|pass\|lft\|plan" ; python scripts/show_bench.py gpurun_out/st_C5b.log | head -2
