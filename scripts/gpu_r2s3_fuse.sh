#!/bin/bash
# session 3: fused block tail (world 1) -- bitwise test, parity subset, latency configs fused / separate
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_resume.py -m gpu -q -x -p no:cacheprovider --timeout 300 \
  -k "fused or pipelined or cores_after or final_error or zero_core or graph or resume or stop_metric" > $O/fuse_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/fuse_tests.log
for C in C1 C3 C4 C5a; do
  for F in 0 1; do
    TRD_NO_FUSE=$F timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/fuse_${C}_$F.log 2>&1
    echo "$C nofuse=$F rc=$? $(python scripts/show_bench.py $O/fuse_${C}_$F.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
