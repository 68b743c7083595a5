#!/bin/bash
# session 3: Q refresh on the side stream -- parity subset incl. world-2 exchange and large ranks, latency configs
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_resume.py tests/test_gpu_exchange.py -m gpu -q -x -p no:cacheprovider --timeout 600 \
  -k "fused or pipelined or cores_after or final_error or graph or resume or stop_metric or ablation or large_ranks or replica or world" > $O/qside_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/qside_tests.log
for C in C1 C3 C4 C5a; do
  for F in 1 0; do
    TRD_Q_MAIN=$F timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/qside_${C}_$F.log 2>&1
    echo "$C qmain=$F rc=$? $(python scripts/show_bench.py $O/qside_${C}_$F.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
