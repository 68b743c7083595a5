#!/bin/bash
mkdir -p gpurun_out
TRD_BENCH_VERBOSE=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_c.log 2>&1; grep "e2e step" gpurun_out/e2e_c.log; python scripts/show_bench.py gpurun_out/e2e_c.log | head -2
ncu --kernel-name regex:"stage|popc|Scan" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/stage_launches.csv python scripts/e2e_probe.py C5b > gpurun_out/stage_ncu.log 2>&1; echo ncu=$?
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/stage_launches.csv")))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"][:60]].append(float(d["Metric Value"].replace(",", "")))
for k, v in agg.items():
    print("%-60s n=%3d mean=%.1f us" % (k, len(v), sum(v) / len(v)))
PY
