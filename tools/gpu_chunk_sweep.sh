#!/bin/bash
# chunk-size x spectrum-store L2 policy sweep of the Large bench (round 2)
out=gpurun_out/chunk_sweep.txt; : > $out
for pol in 2 0 1; do
  lib=""; [ $pol != 2 ] && lib="RSVD_LIB=build_var/librsvd_ws$pol.so"
  for mb in 48 64 96 128; do
    env $lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off --work-mb $mb > gpurun_out/cs.log 2>&1
    tail -1 gpurun_out/cs.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['step_roofline']['kernel_ms_per_step']; print('pol=$pol mb=$mb', d['ms_per_step'], d['phases_ms_last_step']['align'], r['contract'], r['fft_reduce'], d['clocks']['sm_mhz'])" >> $out 2>&1 || tail -3 gpurun_out/cs.log >> $out
  done
done
cat $out
