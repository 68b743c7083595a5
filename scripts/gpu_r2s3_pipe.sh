#!/bin/bash
# session 3: pipelined staging of sampled blocks -- full GPU suite (default TRD_PIPE), then the
# latency configs per pipeline mode
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > $O/pipe_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pipe_tests.log
for C in C3 C4 C5a; do
  for P in 0 1 2 3; do
    TRD_PIPE=$P timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/pipe_${C}_$P.log 2>&1
    echo "$C pipe=$P rc=$? $(python scripts/show_bench.py $O/pipe_${C}_$P.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
