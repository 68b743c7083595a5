#!/bin/bash
mkdir -p gpurun_out/s3v
O=gpurun_out/s3v
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"; python scripts/show_bench.py $O/bench.log | head -3 | cut -c1-250
for C in C3 C4 C5a; do
  timeout 300 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/cfg_$C.log 2>&1
  echo "$C $(python scripts/show_bench.py $O/cfg_$C.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
done
