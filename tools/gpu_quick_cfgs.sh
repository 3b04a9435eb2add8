#!/bin/bash
# quick per-config step / align / kernel times (no cpu baseline, no e2e, no traffic)
TAG=${1:-q}
mkdir -p gpurun_out
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for cfg in "medium --H 8" "medium --H 64" "translations" "small" "large"; do
  n=$(echo $cfg | tr -d ' -')
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/${TAG}_${n}.log 2>&1
  summ gpurun_out/${TAG}_${n}.log "$n"
done
