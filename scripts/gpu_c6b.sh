#!/bin/bash
mkdir -p gpurun_out/c6
O=gpurun_out/c6
timeout 900 python -m pytest tests/test_gpu_edges.py -q --timeout 800 -p no:cacheprovider -rf -k large_ranks > $O/large.log 2>&1
echo "large rc=$?"; tail -3 $O/large.log
timeout 900 python bench.py --config C6 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $O/bench_c6b.log 2>&1
echo "c6 rc=$?"; tail -1 $O/bench_c6b.log | cut -c1-400
TRD_TIMELINE=1 timeout 900 python bench.py --config C6 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/tl_c6b.log 2>&1
echo "tl rc=$?"; grep -A40 "trd timeline" $O/tl_c6b.log | head -50
