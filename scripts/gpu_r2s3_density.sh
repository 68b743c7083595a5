#!/bin/bash
# session 3: dense tcgen05 tiles vs the per-entry SIMT pass (TRD_PASS=rows: warp per row, observed
# entries only) on the C5b shape at several densities; parity of the forced SIMT path first
mkdir -p gpurun_out/s3
O=gpurun_out/s3
TRD_PASS=rows timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 300 \
  -k "block_quantities_match or cores_after" > $O/rows_tests.log 2>&1
echo "rows parity rc=$?"; tail -2 $O/rows_tests.log
for R in 0.01 0.02 0.05 0.1 0.2; do
  for P in tc rows; do
    if [ $P = rows ]; then export TRD_PASS=rows; else unset TRD_PASS; fi
    timeout 600 python bench.py --config C5b --observed $R --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $O/dens_${P}_$R.log 2>&1
    echo "rho=$R $P rc=$? $(python scripts/show_bench.py $O/dens_${P}_$R.log 2>/dev/null | head -1 | grep -o 'value=[0-9.e+]* ms/step=[0-9.]*.*p2/sweep=[0-9.]*ms')"
  done
done
unset TRD_PASS
