#!/bin/bash
# session 3: 32-warp Gauss-Jordan for R^2 > 48 -- solve-dependent tests, kernel time, sweeps (50 timed)
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider --timeout 900 \
  -k "block_quantities or cores_after or final_error or zero_core or lambda or large_ranks or ablation or C4 or C3" > $O/gj32_tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/gj32_tests.log
for V in 0 1; do
  for C in C3 C4 C5a; do
    TRD_GJ3_8=$V timeout 300 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/gj32_${C}_$V.log 2>&1
    echo "gj3_8warps=$V $C $(python scripts/show_bench.py $O/gj32_${C}_$V.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
A="bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:gj --csv --log-file $O/gj32_C4.csv python $A > $O/gj32_ncu.log 2>&1
python scripts/launch_share.py $O/gj32_C4.csv | head -4
