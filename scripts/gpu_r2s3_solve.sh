#!/bin/bash
# session 3: 2-D register Gauss-Jordan solve (gj3) -- parity of the solve-dependent tests, then the
# latency configs with the new and the previous (TRD_SOLVE=2) kernel
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -x -p no:cacheprovider \
  -k "block_quantities or cores_after or final_error or zero_core or lambda or large_ranks or ablation" > $O/solve_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/solve_tests.log
for C in C3 C4 C5a; do
  for S in 0 2; do
    TRD_SOLVE=$S timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/solve_${C}_$S.log 2>&1
    echo "$C solve=$S rc=$? $(python scripts/show_bench.py $O/solve_${C}_$S.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
A="bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gj --log-file $O/launches_gj_C4.csv python $A > $O/ncu_gj.log 2>&1
python scripts/launch_share.py $O/launches_gj_C4.csv | head -5
