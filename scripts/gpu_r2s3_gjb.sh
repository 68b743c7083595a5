#!/bin/bash
# session 3: blocked Gauss-Jordan solve (R^2 in (48, 128]) -- solve-dependent tests, kernel time, sweeps
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider --timeout 900 \
  -k "block_quantities or cores_after or final_error or zero_core or lambda or large_ranks or ablation or C4 or C3 or C5a" > $O/gjb_tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/gjb_tests.log
for V in 3 0; do
  for C in C3 C4 C5a; do
    TRD_SOLVE=$V timeout 300 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/gjb_${C}_$V.log 2>&1
    echo "solve=$V $C $(python scripts/show_bench.py $O/gjb_${C}_$V.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
A="bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:gj --csv --log-file $O/gjb_C4.csv python $A > $O/gjb_ncu.log 2>&1
python scripts/launch_share.py $O/gjb_C4.csv | head -4
