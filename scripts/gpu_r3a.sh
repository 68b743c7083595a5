#!/bin/bash
# health check of HEAD: all -m gpu tests, smoke, default bench line
mkdir -p gpurun_out/r3a
O=gpurun_out/r3a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu_info.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf -x > $O/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -5 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"; tail -1 $O/bench.log | cut -c1-600
