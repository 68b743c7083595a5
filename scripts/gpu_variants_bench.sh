#!/bin/bash
# per-sweep time of the method variants (robust sigma, ablation arms) on C5a and C5b
mkdir -p gpurun_out
for C in C5a C5b; do
  for V in "" "--sigma-mode mad" "--scaling none" "--scaling local"; do
    timeout 300 python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $V > gpurun_out/vb.log 2>&1
    echo "$C [$V] rc=$? $(python scripts/show_bench.py gpurun_out/vb.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]* .*p2/sweep=[0-9.]*ms')"
  done
done
for C in C4 C5a; do
  for V in "" "--sampling rows"; do
    timeout 300 python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $V > gpurun_out/vb.log 2>&1
    echo "$C [$V] rc=$? $(python scripts/show_bench.py gpurun_out/vb.log 2>/dev/null | head -1 | grep -o 'value=[0-9.e+]* ms/step=[0-9.]* .*p2/sweep=[0-9.]*ms')"
  done
done
