#!/bin/bash
mkdir -p gpurun_out
CFGS="C4 C5a" bash scripts/gpu_timeline.sh
bash scripts/gpu_bench_all.sh r2f
VARIANTS="full" UNITS="1" bash scripts/gpu_variants.sh
