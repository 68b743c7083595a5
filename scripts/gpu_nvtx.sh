#!/bin/bash
# NVTX ranges of the API: ncu filtered to the kernels enqueued inside "trd block 1" of a tiny
# sweep (profiles/r02_nvtx_block1.txt)
mkdir -p gpurun_out
timeout 600 ncu --nvtx --nvtx-include "trd block 1/" --metrics gpu__time_duration.sum -c 40 --csv \
  python scripts/tiny_sweep.py C4 > gpurun_out/nvtx_block1.csv 2>&1; echo "ncu nvtx rc=$?"
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/nvtx_block1.csv")) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
print(f"{len(rows)} kernel launches inside NVTX range 'trd block 1'")
names = {}
for r in rows:
    names[r[6].split("(")[0]] = names.get(r[6].split("(")[0], 0) + 1
for n, c in sorted(names.items(), key=lambda x: -x[1]):
    print(f"  {c:3d}  {n}")
PY
