#!/bin/bash
# round-2 profiles: C5b launch list + ncu --set full of both pass kernels; clocks during a bench
mkdir -p gpurun_out
A="bench.py --config C5b --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 python $A > gpurun_out/p2_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5b.csv python $A > gpurun_out/p2_ncu_launch.log 2>&1
python scripts/launch_share.py gpurun_out/r02_launches_c5b.csv > gpurun_out/r02_launch_share_c5b.txt 2>&1
bash scripts/gpu_ncu1.sh r02_p1 tc_pass1
bash scripts/gpu_ncu1.sh r02_p2 tc_pass2
