#!/bin/bash
mkdir -p gpurun_out/r3c
O=gpurun_out/r3c
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_exchange.py -q --timeout 900 -p no:cacheprovider -rf -k "paper_ranks or large_ranks" > $O/large.log 2>&1
echo "large rc=$?"; tail -15 $O/large.log
