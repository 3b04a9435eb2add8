#!/bin/bash
# TMA L2-promotion A/B: transform spectrum loads (RSVD_FFT2_L2PROMO) and contraction operand loads (RSVD_TC_L2PROMO)
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for rep in 1 2; do for v in p33 p23 p03 p32; do
  RSVD_LIB=build_var/$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/r2i_l2p_$v.log 2>&1
  summ gpurun_out/r2i_l2p_$v.log $v
done; done
