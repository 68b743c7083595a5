#!/bin/bash
mkdir -p gpurun_out
./scripts/microbench/fma_peak > gpurun_out/fp32_peak.json 2> gpurun_out/fp32_peak.err; echo "fma rc=$?"; cat gpurun_out/fp32_peak.json
bash scripts/gpu_tests.sh 1500
bash scripts/gpu_bench_all.sh r2c
