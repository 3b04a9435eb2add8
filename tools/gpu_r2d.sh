#!/bin/bash
# transform micro-opts: parity, then bench (two-kernel path)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2d_parity.log 2>&1; rc=$?
echo "pytest exit $rc" >> gpurun_out/r2d_parity.log; tail -2 gpurun_out/r2d_parity.log
[ $rc -ne 0 ] && exit 1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
timeout 300 $B > gpurun_out/r2d_b.log 2>&1; summ gpurun_out/r2d_b.log new
