#!/bin/bash
# usage: scripts/gpu_prof.sh <tag> [config]
#   1) plain bench run (must exit 0)  2) ncu launch list of the same command
#   3) one ncu --set full capture of each pass kernel
mkdir -p gpurun_out
T=${1:-prof}; CFG=${2:-C5b}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/${T}_plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/${T}_plain.log; exit 1; }
tail -1 gpurun_out/${T}_plain.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_list.log 2>&1; echo list=$?
[ -n "$FULL" ] && { timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$FULL" -s 12 -c 2 -o gpurun_out/${T}_full $CMD > gpurun_out/${T}_ncu_full.log 2>&1; echo full=$?; }
python scripts/launch_share.py gpurun_out/${T}_launches.csv 2>&1 | head -40
