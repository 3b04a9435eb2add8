#!/bin/bash
# fft3 parity + A/B against fft2; L2 policy / chunk-size variants of the contraction
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/r2b_parity.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2b_parity.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for v in 3 2; do RSVD_FFT=$v timeout 600 $B > gpurun_out/r2b_fft$v.log 2>&1; summ gpurun_out/r2b_fft$v.log fft$v; done
for l in ws0 ws1; do RSVD_LIB=build_var/$l.so timeout 600 $B > gpurun_out/r2b_$l.log 2>&1; summ gpurun_out/r2b_$l.log $l; done
for mb in 64 96 192; do timeout 600 $B --work-mb $mb > gpurun_out/r2b_mb$mb.log 2>&1; summ gpurun_out/r2b_mb$mb.log mb$mb; done
