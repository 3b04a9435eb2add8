#!/bin/bash
# A/B of library variants on the Large bench (5 steps): prints step, align, per-kernel ms, clock.
# Usage: bash tools/gpu_ab.sh TAG lib1.so [lib2.so ...]   (librsvd.so = the product build)
TAG=$1; shift
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off $BENCH_ARGS"
for rep in 1 2; do
for L in "$@"; do
  n=$(basename $L .so)
  RSVD_LIB=$L timeout 300 $B > gpurun_out/${TAG}_${n}_$rep.log 2>&1
  tail -1 gpurun_out/${TAG}_${n}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['step_roofline']['kernel_ms_per_step']; print('$n', d['ms_per_step'], d['phases_ms_last_step']['align'], k['contract'], k['fft_reduce'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
