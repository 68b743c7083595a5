#!/bin/bash
mkdir -p gpurun_out/r3d
O=gpurun_out/r3d
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_exchange.py -q --timeout 900 -p no:cacheprovider -rf -k "paper_ranks or large_ranks" > $O/large.log 2>&1
echo "large rc=$?"; tail -5 $O/large.log
timeout 900 python bench.py --config C6 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $O/bench_c6.log 2>&1
echo "c6 rc=$?"; tail -1 $O/bench_c6.log | cut -c1-300
TRD_TIMELINE=1 timeout 900 python bench.py --config C6 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/tl_c6.log 2>&1
echo "tl rc=$?"; grep -A25 "trd timeline" $O/tl_c6.log
