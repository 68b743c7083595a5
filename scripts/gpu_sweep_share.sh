#!/bin/bash
# per-kernel device time inside the NVTX "trd sweep" ranges (eager sweeps; ncu serialises and
# runs each kernel cold, so compare shares) for the latency-bound configs
mkdir -p gpurun_out
for C in ${CFGS:-C5a C4}; do
  TRD_GRAPH=0 timeout 900 ncu --nvtx --nvtx-include "trd sweep/" --cache-control none --clock-control none --metrics gpu__time_duration.sum -c 3000 --csv \
    python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/share_$C.csv 2>&1
  echo "$C rc=$?"
  python scripts/launch_share.py gpurun_out/share_$C.csv > gpurun_out/share_$C.txt; head -30 gpurun_out/share_$C.txt
done
