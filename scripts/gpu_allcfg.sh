#!/bin/bash
# one short bench line per config (device-timed sweeps only)
mkdir -p gpurun_out
T=${1:-all}
for C in C1 C2 C3 C4 C5a C5b; do
  timeout 300 python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/${T}_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py gpurun_out/${T}_$C.log 2>/dev/null | head -1 | cut -c1-260)"
done
