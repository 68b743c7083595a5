#!/bin/bash
# the paper's video completion workload at full size (C6, ranks [80,80,3,20]); timeline of one block
mkdir -p gpurun_out/c6
O=gpurun_out/c6
timeout 900 python bench.py --config C6 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $O/bench_c6.log 2>&1
echo "c6 rc=$?"; tail -3 $O/bench_c6.log | cut -c1-1500
TRD_TIMELINE=1 timeout 900 python bench.py --config C6 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/tl_c6.log 2>&1
echo "tl rc=$?"; grep -A40 "trd timeline" $O/tl_c6.log | head -50
