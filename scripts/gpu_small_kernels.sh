#!/bin/bash
# C5b launch times of the per-block helper kernels (Lft pack, d contraction) and the bench line
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/sk_plain.log 2>&1 || exit 1
python scripts/show_bench.py gpurun_out/sk_plain.log | head -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lft_pack|reduce_d" --csv --log-file gpurun_out/sk_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_share.py gpurun_out/sk_launches.csv 2>&1 | head -6
