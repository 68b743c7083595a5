#!/bin/bash
# session 3: A/B of the latency-path switches with long runs (50 timed sweeps after 20 warm-up
# sweeps: 10-sweep runs of the sub-ms configs were biased by the clock ramp)
mkdir -p gpurun_out/s3ab
O=gpurun_out/s3ab
run() {  # name, env...
  local name=$1; shift
  for C in C3 C4 C5a; do
    env "$@" timeout 300 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/${name}_$C.log 2>&1
    echo "$name $C $(python scripts/show_bench.py $O/${name}_$C.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
}
run default TRD_X=0
run default2 TRD_X=1
run pipe0 TRD_PIPE=0
run pipe3all TRD_PIPE=3
run pipe1all TRD_PIPE=1
run qside TRD_Q_SIDE=1
run nopdl TRD_PDL=0
run threadchain TRD_CHAIN_THREAD=1
run nofuse TRD_NO_FUSE=1
run solve2 TRD_SOLVE=2
