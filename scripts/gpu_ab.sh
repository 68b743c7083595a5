#!/bin/bash
# A/B of whole libraries on the latency configs: in-tree vs abtest/libtrd_$V.so, alternating
mkdir -p gpurun_out
for R in 1 2; do
for C in ${CFGS:-C3 C4 C5a}; do
  for L in cur ${VARIANTS:-prev}; do
    if [ $L = cur ]; then unset TRD_LIB_PATH; else export TRD_LIB_PATH=$PWD/abtest/libtrd_$L.so; fi
    timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${C}_$L.log 2>&1
    echo "$C lib=$L rc=$? $(python scripts/show_bench.py gpurun_out/ab_${C}_$L.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
done
done
unset TRD_LIB_PATH
