#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "block_quantities" > gpurun_out/tc10_block.log 2>&1; echo block=$?
tail -30 gpurun_out/tc10_block.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/tc10_all.log 2>&1; echo all=$?
tail -15 gpurun_out/tc10_all.log
timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tc10_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tc10_c5b.log 2>&1; echo c5b=$?
