#!/bin/bash
# round-2 closing evidence (third session): GPU suite, smoke, default bench + reference arm, every
# config, C5b launch list, ncu --set full of the pass-1 kernel
mkdir -p gpurun_out/fin4
O=gpurun_out/fin4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu_info.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> $O/gpu_info.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf > $O/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c5b.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/ref_c5b.log 2>&1; echo "ref rc=$?"
for C in C1 C2 C3 C4 C5a C5b; do
  S=50; W=20; [ $C = C5b ] && S=10 && W=3
  timeout 600 python bench.py --config $C --steps $S --warmup $W --no-e2e --no-cpu-baseline > $O/cfg_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py $O/cfg_$C.log 2>/dev/null | head -1 | cut -c1-240)"
done > $O/all_configs.txt
timeout 600 python bench.py --config C6 --steps 5 --warmup 2 --no-cpu-baseline > $O/cfg_C6.log 2>&1
echo "C6 rc=$? $(python scripts/show_bench.py $O/cfg_C6.log 2>/dev/null | head -1 | cut -c1-240)" >> $O/all_configs.txt
cat $O/all_configs.txt
A="bench.py --config C5b --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5b.csv python $A > $O/ncu_launch.log 2>&1
python scripts/launch_share.py $O/launches_c5b.csv > $O/launch_share_c5b.txt 2>&1
head -12 $O/launch_share_c5b.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_pass1_kernel -s 2 -c 1 -o $O/pass1 python $A > $O/ncu_pass1.log 2>&1
ncu -i $O/pass1.ncu-rep --page details --csv > $O/pass1_details.csv 2>/dev/null
ncu -i $O/pass1.ncu-rep --page raw --csv > $O/pass1_raw.csv 2>/dev/null
ls -la $O | head -40
