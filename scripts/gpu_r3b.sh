#!/bin/bash
# large-rank path: the paper's [80,80,3,20] parity test, then the whole GPU suite
mkdir -p gpurun_out/r3b
O=gpurun_out/r3b
timeout 900 python -m pytest tests/test_gpu_edges.py -q --timeout 800 -p no:cacheprovider -rf -k large_ranks > $O/large.log 2>&1
echo "large rc=$?"; tail -15 $O/large.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf > $O/gpu_tests.log 2>&1
echo "all rc=$?"; tail -8 $O/gpu_tests.log
