#!/bin/bash
# session 3: GPU suite with the new defaults (every sampled block pipelined, Q refresh on the side
# stream, PDL off), then single-switch A/B from them (50 timed sweeps after 20 warm-up sweeps)
mkdir -p gpurun_out/s3ab
O=gpurun_out/s3ab
timeout 2000 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/tests.log
run() {
  local name=$1; shift
  for C in C1 C2 C3 C4 C5a; do
    env "$@" timeout 300 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/b_${name}_$C.log 2>&1
    echo "$name $C $(python scripts/show_bench.py $O/b_${name}_$C.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
  done
}
run new TRD_X=0
run pipe0 TRD_PIPE=0
run qmain TRD_Q_SIDE=0
run pdl TRD_PDL=1
run threadchain TRD_CHAIN_THREAD=1
timeout 600 python bench.py --config C5b --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/b_new_C5b.log 2>&1
echo "new C5b $(python scripts/show_bench.py $O/b_new_C5b.log 2>/dev/null | head -1 | grep -o 'ms/step=[0-9.]*')"
