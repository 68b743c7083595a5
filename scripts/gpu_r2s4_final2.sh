#!/bin/bash
# session 4 closing run on the final code: GPU suite, smoke, default bench, C3 / C4 / C5a 50-sweep lines
mkdir -p gpurun_out/fin7
O=gpurun_out/fin7
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf > $O/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c5b.log 2>&1; echo "bench rc=$?"
python scripts/show_bench.py $O/bench_c5b.log | grep -v "^  |"
for C in C4 C5a; do
  timeout 600 python bench.py --config $C --steps 50 --warmup 20 --no-e2e --no-cpu-baseline > $O/cfg_$C.log 2>&1
  echo "$C rc=$? $(python scripts/show_bench.py $O/cfg_$C.log 2>/dev/null | grep value= | head -1 | cut -c1-120)"
done
