#!/bin/bash
# per-stage timeline of one config's sweeps (TRD_TIMELINE=1, eager)
mkdir -p gpurun_out
for C in ${CFGS:-C4 C5a}; do
  TRD_TIMELINE=1 timeout 300 python bench.py --config $C --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/tl_$C.log 2>&1
  echo "== $C rc=$?"; grep -A40 "trd timeline" gpurun_out/tl_$C.log | head -40
done
