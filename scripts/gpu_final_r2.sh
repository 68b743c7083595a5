#!/bin/bash
# round-2 final evidence: default bench line, reference arm, all configs, C5b launch list,
# ncu --set full of both pass kernels, latency timelines
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu_info.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> $O/gpu_info.txt
timeout 900 python bench.py > $O/bench_c5b.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/ref_c5b.log 2>&1; echo "ref rc=$?"
for C in C1 C2 C3 C4 C5a C5b; do
  timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py $O/cfg_$C.log 2>/dev/null | head -1 | cut -c1-240)"
done > $O/all_configs.txt
timeout 300 python bench.py --config C5b --steps 5 --warmup 3 --sigma-mode mad --no-e2e --no-cpu-baseline > $O/cfg_C5b_mad.log 2>&1
for C in C4 C5a; do TRD_TIMELINE=1 timeout 300 python bench.py --config $C --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > $O/tl_$C.log 2>&1; done
A="bench.py --config C5b --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 python $A > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5b.csv python $A > $O/ncu_launch.log 2>&1
python scripts/launch_share.py $O/launches_c5b.csv > $O/launch_share_c5b.txt 2>&1
for K in tc_pass1 tc_pass2; do
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s 2 -c 1 -o $O/$K python $A > $O/ncu_$K.log 2>&1
  ncu -i $O/$K.ncu-rep --page source --csv --print-source sass > $O/${K}_src.csv 2>/dev/null
  ncu -i $O/$K.ncu-rep --page details --csv > $O/${K}_details.csv 2>/dev/null
  ncu -i $O/$K.ncu-rep --page raw --csv > $O/${K}_raw.csv 2>/dev/null
done
ls -la $O
