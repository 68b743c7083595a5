#!/bin/bash
# the driver's runs: default bench line (C5b, e2e, cpu_baseline) and the reference arm
mkdir -p gpurun_out
T=${1:-d}
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"
python scripts/show_bench.py gpurun_out/${T}_bench.log 2>/dev/null | head -3
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.log 2>&1; echo "ref rc=$?"
tail -c 1500 gpurun_out/${T}_ref.log
