#!/bin/bash
# round-2 session-4 verification of the restored tree: GPU suite, smoke, default bench + reference arm
mkdir -p gpurun_out/fin5
O=gpurun_out/fin5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu_info.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf > $O/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c5b.log 2>&1; echo "bench rc=$?"; tail -1 $O/bench_c5b.log | cut -c1-400
timeout 900 python bench.py --impl reference > $O/ref_c5b.log 2>&1; echo "ref rc=$?"; tail -1 $O/ref_c5b.log | cut -c1-300
