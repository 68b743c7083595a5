#!/bin/bash
# one ncu --set full capture of stage_vals and stage_bits (C5b, block 1 of the first upload sweep)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name regex:"stage_(vals|bits)" --launch-skip 6 --launch-count 4 \
    -o gpurun_out/stage_full -f python scripts/e2e_probe.py C5b > gpurun_out/stage_full.log 2>&1; echo ncu=$?
