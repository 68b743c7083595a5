#!/bin/bash
# session 4: gj4 on 16 warps (TRD_SOLVE=6) for every R^2 vs the default (16 warps only above 96)
mkdir -p gpurun_out/s4d
O=gpurun_out/s4d
for C in C5a C3 C2 C1; do
  for S in def 6; do
    if [ $S = def ]; then unset TRD_SOLVE; else export TRD_SOLVE=$S; fi
    timeout 600 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/ab_${C}_$S.log 2>&1
    echo "$C sel=$S rc=$? $(python scripts/show_bench.py $O/ab_${C}_$S.log 2>/dev/null | grep value= | head -1 | cut -c1-110)"
  done
done
unset TRD_SOLVE
TRD_TIMELINE=1 TRD_GRAPH=0 timeout 600 python bench.py --config C4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/timeline_C4.log 2>&1
echo "timeline rc=$?"; grep -v "^{" $O/timeline_C4.log | tail -40
