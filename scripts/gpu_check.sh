#!/bin/bash
# usage: scripts/gpu_check.sh <tag>  -- GPU parity suite + C4/C5b bench lines (run on the GPU box)
mkdir -p gpurun_out
T=${1:-chk}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_gpu.log 2>&1; echo gpu_tests=$?
tail -15 gpurun_out/${T}_gpu.log
timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c4.log 2>&1; echo c4=$?
tail -1 gpurun_out/${T}_c4.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${T}_c5b.log 2>&1; echo c5b=$?
tail -1 gpurun_out/${T}_c5b.log
