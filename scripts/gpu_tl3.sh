#!/bin/bash
mkdir -p gpurun_out
for V in "base:" "noamax:TRD_DIAG_NOAMAX=1"; do
  N=${V%%:*}; E=${V#*:}
  env $E TRD_TIMELINE=1 timeout 300 python bench.py --config C4 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/tl3_$N.log 2>&1
  echo "== $N rc=$?"; grep -A20 "trd timeline" gpurun_out/tl3_$N.log | grep "lft\|plan"
done
A="bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 ncu --set full --clock-control none -k regex:tc_lft_pack_hw -c 4 -o gpurun_out/lft_hw python $A > gpurun_out/lft_ncu.log 2>&1; echo "ncu rc=$?"
