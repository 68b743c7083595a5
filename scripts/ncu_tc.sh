#!/bin/bash
# usage: ncu_tc.sh <tag> <config> <kernel-regex> <count>
mkdir -p gpurun_out
TAG=$1; CFG=$2; KRE=$3; CNT=${4:-2}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:$KRE" -c $CNT -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo ncu=$?
