#!/bin/bash
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > $O/qrule_tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/qrule_tests.log
for C in C1 C2 C3 C4 C5a; do
  timeout 300 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/qrule_$C.log 2>&1
  echo "$C $(python scripts/show_bench.py $O/qrule_$C.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
done
