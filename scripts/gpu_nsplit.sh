#!/bin/bash
mkdir -p gpurun_out
for SP in 0 1 2 3 4; do
  if [ $SP = 0 ]; then unset TRD_NSPLIT; else export TRD_NSPLIT=$SP; fi
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/nsp.log 2>&1
  echo "nsplit=$SP rc=$? $(python scripts/show_bench.py gpurun_out/nsp.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p2/sweep=[0-9.]*ms')"
done
