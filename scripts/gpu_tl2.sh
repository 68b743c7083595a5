#!/bin/bash
mkdir -p gpurun_out
for V in "base:" "tile:TRD_LFT_TILE=1" "noside:TRD_NO_SIDE=1" "tile_noside:TRD_LFT_TILE=1 TRD_NO_SIDE=1"; do
  N=${V%%:*}; E=${V#*:}
  env $E TRD_TIMELINE=1 timeout 300 python bench.py --config C4 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/tl2_$N.log 2>&1
  echo "== $N rc=$?"; grep -A20 "trd timeline" gpurun_out/tl2_$N.log | grep "lft\|plan\|solve\|gram\|stage\|reduce d\|sampler"
  env $E timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/tl2b_$N.log 2>&1
  echo "   bench: $(python scripts/show_bench.py gpurun_out/tl2b_$N.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
done
