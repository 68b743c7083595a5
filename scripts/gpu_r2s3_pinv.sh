#!/bin/bash
# session 3: restaging of invalidated sweep-invariant blocks (after an upload) on the staging stream
# (TRD_PIPE_INV=1) -- upload / staging tests, C5b e2e A/B
mkdir -p gpurun_out/s3
O=gpurun_out/s3
TRD_PIPE_INV=1 timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider --timeout 900 \
  -k "upload or pipelined or packed or graph or c5b or C5b" > $O/pinv_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pinv_tests.log
for V in "0 8" "1 1" "1 2" "1 8"; do
  set -- $V
  TRD_PIPE_INV=$1 TRD_GATHER_CTAS=$2 timeout 900 python bench.py --config C5b --steps 8 --warmup 3 --no-cpu-baseline > $O/pinv_$1_$2.log 2>&1
  echo "pinv=$1 gather_ctas=$2 rc=$? $(python scripts/show_bench.py $O/pinv_$1_$2.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*') $(python scripts/show_bench.py $O/pinv_$1_$2.log 2>/dev/null | sed -n 2p | grep -o "'value': [0-9.e+]*")"
done
