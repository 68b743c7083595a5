#!/bin/bash
# sweep time of the latency-bound configs: CUDA graphs on/off x profiling events on/off
mkdir -p gpurun_out
for C in ${CFGS:-C1 C4 C5a}; do
  for G in 0 1; do
    for P in 0 1; do
      if [ $P = 0 ]; then export TRD_BENCH_NOPROF=1; else unset TRD_BENCH_NOPROF; fi
      TRD_GRAPH=$G timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat_${C}_g${G}_p${P}.log 2>&1
      echo "$C graph=$G prof=$P rc=$? $(python scripts/show_bench.py gpurun_out/lat_${C}_g${G}_p${P}.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
    done
  done
done
unset TRD_BENCH_NOPROF
