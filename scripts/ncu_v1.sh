#!/bin/bash
# v1 profile: plain bench run, then the launch list and one full capture of the pass kernel
mkdir -p gpurun_out
python bench.py --config C4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_c4.log 2>&1 || exit 1
K='regex:pass_kernel|sampler_kernel|offsets_kernel|mid_kernel|rgt_kernel|lft_kernel|reduce_d_kernel|reduce_den_kernel|q_kernel|matmul_f64_kernel|phi_kernel|solve_kernel|h_kernel|update2_kernel|block_scalars_kernel|sweep_begin_kernel|sweep_end_kernel|dt_T_kernel|dt_D_kernel'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_c4_v1.csv python bench.py --config C4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 8 -c 2 -o gpurun_out/prof_c4_v1 python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
