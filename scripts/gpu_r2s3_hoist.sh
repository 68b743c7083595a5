#!/bin/bash
# session 3: pass-1 entry ids / values loaded ahead of the S dump -- parity subset, bench, trace
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -x -p no:cacheprovider --timeout 300 \
  -k "block_quantities or cores_after or persistent or robust or pipelined" > $O/hoist_tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/hoist_tests.log
for C in C5b C5a C4; do
  timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/hoist_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py $O/hoist_$C.log 2>/dev/null | head -1 | cut -c1-220)"
done
TRD_LIB_PATH=$PWD/abtest/libtrd_exp.so TRD_GRAPH=0 TRD_TC_EXP=8 timeout 300 python bench.py --config C5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/tr5.log 2>&1; echo "trace rc=$?"
grep -A24 "tc trace\]" $O/tr5.log | head -26
