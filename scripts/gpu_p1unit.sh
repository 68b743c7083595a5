#!/bin/bash
mkdir -p gpurun_out
for U in 1 2; do
  TRD_P1_UNIT=$U timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/p1u$U.log 2>&1
  echo "p1unit=$U rc=$? $(python scripts/show_bench.py gpurun_out/p1u$U.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p2/sweep=[0-9.]*ms')"
done
