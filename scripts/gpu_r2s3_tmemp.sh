#!/bin/bash
# session 3: pass-1 GEMM2 operand in TMEM (TRD_P1_TMEMP) -- smoke, parity subset, C5b / C5a / C4 bench
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/tp_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/tp_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 300 \
  -k "block_quantities or cores_after or persistent" > $O/tp_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/tp_tests.log
for C in C5b C5a C4; do
  timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/tp_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py $O/tp_$C.log 2>/dev/null | head -1 | cut -c1-220)"
done
