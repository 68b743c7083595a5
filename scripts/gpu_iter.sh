#!/bin/bash
# one build -> measure iteration: GPU suite, C5b / C4 / C5a bench lines, optional pass-1 trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for CFG in ${CFGS:-C5b C4 C5a}; do
  timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/it_$CFG.log 2>&1
  echo "$CFG rc=$? $(python scripts/show_bench.py gpurun_out/it_$CFG.log 2>/dev/null | head -1)"
done
if [ -n "$TRACE" ]; then
  TRD_LIB_PATH=$PWD/abtest/libtrd_exp.so TRD_GRAPH=0 TRD_TC_EXP=8 timeout 300 python bench.py --config C5b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/tr_C5b.log 2>&1
  grep -A24 "tc trace\]" gpurun_out/tr_C5b.log | tail -14
fi
