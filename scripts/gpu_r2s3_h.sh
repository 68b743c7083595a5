#!/bin/bash
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 2000 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > $O/h_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/h_tests.log
for C in C3 C4 C5a; do
  timeout 300 python bench.py --config $C --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > $O/h_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py $O/h_$C.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
done
A="bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/h_C4.csv python $A > $O/h_ncu.log 2>&1
python scripts/launch_share.py $O/h_C4.csv | grep "trd::\|TOTAL" | head -30
