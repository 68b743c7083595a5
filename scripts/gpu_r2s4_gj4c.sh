#!/bin/bash
# session 4: gj4 on 8 warps (TRD_SOLVE=4, default) vs 16 warps (6)
mkdir -p gpurun_out/s4c
O=gpurun_out/s4c
timeout 300 python -m pytest tests/test_gpu_edges.py -m gpu -q -k solve_variants -p no:cacheprovider > $O/solve_variants.log 2>&1
echo "solve_variants rc=$?"; tail -2 $O/solve_variants.log
for S in 4 6; do
  TRD_SOLVE=$S TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gj --csv \
    --log-file $O/gj_launch_$S.csv python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_gj_$S.log 2>&1
  echo "ncu sel=$S rc=$?"
  python - $O/gj_launch_$S.csv <<'PY'
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == 'gpu__time_duration.sum']
d = defaultdict(list)
for r in rows: d[r[4].split('(')[0]].append(float(r[-1].replace(",", "")))
for k, v in d.items(): print(f"  {k}: n={len(v)} mean={sum(v)/len(v):.0f} {rows[0][-2]}")
PY
done
for C in C4 C3; do
  for S in 4 6; do
    TRD_SOLVE=$S timeout 600 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/ab_${C}_$S.log 2>&1
    echo "$C sel=$S rc=$? $(python scripts/show_bench.py $O/ab_${C}_$S.log 2>/dev/null | grep value= | head -1 | cut -c1-120)"
  done
done
