#!/bin/bash
# spectrum-store L2 policy per config: default build (evict_first) vs ws0 (normal) vs ws1 (evict_last)
mkdir -p gpurun_out
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for cfg in "medium --H 8" "medium --H 64" "translations" "large"; do
  n=$(echo $cfg | tr -d ' -')
  for l in default ws0 ws1; do
    if [ $l = default ]; then L=""; else L="RSVD_LIB=build_var/$l.so"; fi
    env $L timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/r2f_${n}_$l.log 2>&1
    summ gpurun_out/r2f_${n}_$l.log "$n $l"
  done
done
