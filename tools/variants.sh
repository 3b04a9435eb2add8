#!/bin/bash
# A/B of prebuilt library variants (build_var/*.so, made with build.py -D... --out=...):
# the TC parity tests on each, then a short bench line with per-kernel times.
# Usage: BENCH_ARGS="--work-mb 256" bash tools/variants.sh TAG lib1.so lib2.so ...
TAG=$1; shift
mkdir -p gpurun_out
for L in "$@"; do
  n=$(basename $L .so)
  if [ -z "$NO_PARITY" ]; then
  RSVD_LIB=$L timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/${TAG}_${n}_parity.log 2>&1; echo "parity exit $?" >> gpurun_out/${TAG}_${n}_parity.log
  fi
  RSVD_LIB=$L timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/${TAG}_${n}_bench.log 2>&1
  echo "== $n: $(tail -2 gpurun_out/${TAG}_${n}_parity.log 2>/dev/null| tr '\n' ' ')"
  tail -1 gpurun_out/${TAG}_${n}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms_last_step'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
