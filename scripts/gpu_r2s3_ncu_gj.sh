#!/bin/bash
mkdir -p gpurun_out/s3
O=gpurun_out/s3
A="bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
TRD_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gj3_solve -s 2 -c 1 -o $O/gj3 python $A > $O/ncu_gj3.log 2>&1
ncu -i $O/gj3.ncu-rep --page raw --csv > $O/gj3_raw.csv 2>/dev/null
ncu -i $O/gj3.ncu-rep --page details --csv > $O/gj3_details.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/s3/gj3_raw.csv')))
h=rows[0]; u=rows[1]; v=rows[2]
for i,n in enumerate(h):
    if any(k in n for k in ['gpu__time_duration.sum','pipe_fp64','inst_executed_pipe_fp64','smsp__average_warp','issue_active','warp_issue_stalled']) and ('pct' in n or 'sum' in n or 'ratio' in n):
        print(n, u[i], v[i])
PY
