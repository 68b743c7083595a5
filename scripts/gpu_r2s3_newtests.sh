#!/bin/bash
mkdir -p gpurun_out/s3
timeout 1200 python -m pytest tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider --timeout 600 -rf -k "solve_variants or upload_with_changed" > gpurun_out/s3/newtests.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/s3/newtests.log
