#!/bin/bash
# session 3: programmatic dependent launch of the per-block small kernels -- GPU suite, latency configs PDL on / off
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 2000 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > $O/pdl_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pdl_tests.log
for C in C1 C2 C3 C4 C5a C5b; do
  for P in 0 1; do
    TRD_PDL=$P timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/pdl_${C}_$P.log 2>&1
    echo "$C pdl=$P rc=$? $(python scripts/show_bench.py $O/pdl_${C}_$P.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
