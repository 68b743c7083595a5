#!/bin/bash
# all -m gpu tests (per-test timeout), junit summary under gpurun_out/
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout ${1:-2400} python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf ${2:+-k "$2"} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/gpu_tests.log
