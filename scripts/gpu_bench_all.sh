#!/bin/bash
# one device-timed bench line per config (tag $1) + the C5b default line with e2e
mkdir -p gpurun_out
T=${1:-b}
for C in C1 C2 C3 C4 C5a C5b; do
  timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py gpurun_out/${T}_$C.log 2>/dev/null | head -1 | cut -c1-260)"
done
timeout 300 python bench.py --config C5b --steps 5 --warmup 3 --sigma-mode mad --no-e2e --no-cpu-baseline > gpurun_out/${T}_C5b_mad.log 2>&1
echo "C5b mad rc=$? $(python scripts/show_bench.py gpurun_out/${T}_C5b_mad.log 2>/dev/null | head -1 | cut -c1-260)"
