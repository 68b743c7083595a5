#!/bin/bash
# session 3: warp-per-index chain products (Rgt / Mid) -- GPU suite, latency configs new / thread-per-row
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 2000 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > $O/chain_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/chain_tests.log
for C in C1 C3 C4 C5a C5b; do
  for P in 1 0; do
    TRD_CHAIN_THREAD=$P timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/chain_${C}_$P.log 2>&1
    echo "$C thread_chains=$P rc=$? $(python scripts/show_bench.py $O/chain_${C}_$P.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
A="bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"rgt|mid" --csv --log-file $O/chain_C4.csv python $A > $O/chain_ncu.log 2>&1
python scripts/launch_share.py $O/chain_C4.csv | head -6
