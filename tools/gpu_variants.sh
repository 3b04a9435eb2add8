#!/bin/bash
# A/B of library variants on the Large bench: tools/gpu_variants.sh name=lib.so ... ("default" = in-tree)
out=gpurun_out/variants.txt; : > $out
for kv in "$@"; do
  name=${kv%%=*}; lib=${kv#*=}; extra=""
  [ "$lib" != default ] && extra="RSVD_LIB=$lib"
  env $extra $VARIANT_ENV timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off $BENCH_ARGS > gpurun_out/v.log 2>&1
  tail -1 gpurun_out/v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['step_roofline']['kernel_ms_per_step']; print('$name', d['ms_per_step'], d['phases_ms_last_step']['align'], r['contract'], r['fft_reduce'], d['clocks']['sm_mhz'])" >> $out 2>&1 || tail -3 gpurun_out/v.log >> $out
done
cat $out
