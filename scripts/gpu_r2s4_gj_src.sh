#!/bin/bash
# session 4: source-level stall attribution of the R^2 = 100 Gauss-Jordan solve (C4's critical path)
mkdir -p gpurun_out/s4
O=gpurun_out/s4
A="bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
TRD_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gj3_solve -s 2 -c 1 -o $O/gj3 python $A > $O/ncu_gj3.log 2>&1
echo "ncu rc=$?"
ncu -i $O/gj3.ncu-rep --page source --csv --print-source sass > $O/gj3_sass.csv 2>/dev/null
ncu -i $O/gj3.ncu-rep --page details --csv > $O/gj3_details.csv 2>/dev/null
ls -la $O
