#!/bin/bash
# fused persistent align: KC (contraction clusters) sweep beyond round 2's 10..22, vs the two-kernel path
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r3kc_gpu.txt
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off"
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
RSVD_FUSED=0 timeout 300 $B > gpurun_out/r3kc_off.log 2>&1; summ gpurun_out/r3kc_off.log off
for kc in 22 28 32 36 40 46; do RSVD_FUSED=1 RSVD_FUSED_KC=$kc timeout 300 $B > gpurun_out/r3kc_kc$kc.log 2>&1; summ gpurun_out/r3kc_kc$kc.log kc$kc; done
