#!/bin/bash
# fused persistent align: parity first (stop on failure), then timing vs the two-kernel path, KC sweep
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2c_parity.log 2>&1; rc=$?
echo "pytest exit $rc" >> gpurun_out/r2c_parity.log; tail -3 gpurun_out/r2c_parity.log
[ $rc -ne 0 ] && exit 1
timeout 600 python -m pytest tests/test_gpu_configs.py -x -q -m gpu -k "not simt" > gpurun_out/r2c_configs.log 2>&1; echo "configs exit $?" >> gpurun_out/r2c_configs.log; tail -2 gpurun_out/r2c_configs.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
RSVD_FUSED=0 timeout 300 $B > gpurun_out/r2c_off.log 2>&1; summ gpurun_out/r2c_off.log off
for kc in 14 18 22 10; do RSVD_FUSED_KC=$kc timeout 300 $B > gpurun_out/r2c_kc$kc.log 2>&1; summ gpurun_out/r2c_kc$kc.log kc$kc; done
RSVD_FUSED_NBUF=3 timeout 300 $B > gpurun_out/r2c_nb3.log 2>&1; summ gpurun_out/r2c_nb3.log nbuf3
