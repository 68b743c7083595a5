#!/bin/bash
# session 4: chunked owner-resolved Gauss-Jordan (TRD_SOLVE=4) vs the default -- parity, per-launch
# time (ncu, cold), 50-sweep lines of the configs whose blocks go through the register solve
mkdir -p gpurun_out/s4
O=gpurun_out/s4
timeout 300 python -m pytest tests/test_gpu_edges.py -m gpu -q -k solve_variants -p no:cacheprovider > $O/solve_variants.log 2>&1
echo "solve_variants rc=$?"; tail -2 $O/solve_variants.log
for S in 0 4; do
  TRD_SOLVE=$S TRD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gj --csv \
    --log-file $O/gj_launch_$S.csv python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_gj_$S.log 2>&1
  echo "ncu sel=$S rc=$? $(grep -c gpu__time_duration $O/gj_launch_$S.csv)"
  python - $O/gj_launch_$S.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == 'gpu__time_duration.sum']
from collections import defaultdict
d = defaultdict(list)
for r in rows: d[r[4].split('(')[0]].append(float(r[-1].replace(",", "")))
for k, v in d.items(): print(f"  {k}: n={len(v)} mean={sum(v)/len(v):.0f} {rows[0][-2]}")
PY
done
for C in C4 C3 C5a; do
  for S in def 4; do
    if [ $S = def ]; then unset TRD_SOLVE; else export TRD_SOLVE=$S; fi
    timeout 600 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/ab_${C}_$S.log 2>&1
    echo "$C sel=$S rc=$? $(python scripts/show_bench.py $O/ab_${C}_$S.log 2>/dev/null | grep value= | head -1 | cut -c1-200)"
  done
done
unset TRD_SOLVE
TRD_SOLVE=4 timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -x > $O/gpu_tests_sel4.log 2>&1
echo "all gpu tests with TRD_SOLVE=4 rc=$?"; tail -2 $O/gpu_tests_sel4.log
