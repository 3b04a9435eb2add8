#!/bin/bash
# chunk shape A/B: template tiles per chunk (RSVD_TCT) x workspace size; trace of the TCT=2 timeline
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off"
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], d['step_roofline']['kernel_ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
timeout 300 $B > gpurun_out/r3t_base.log 2>&1; summ gpurun_out/r3t_base.log base
RSVD_TCT=2 timeout 300 $B > gpurun_out/r3t_tct2.log 2>&1; summ gpurun_out/r3t_tct2.log tct2_128
RSVD_TCT=2 timeout 300 $B --work-mb 256 > gpurun_out/r3t_tct2_256.log 2>&1; summ gpurun_out/r3t_tct2_256.log tct2_256
RSVD_TCT=4 timeout 300 $B --work-mb 256 > gpurun_out/r3t_tct4_256.log 2>&1; summ gpurun_out/r3t_tct4_256.log tct4_256
RSVD_TCT=2 RSVD_LIB=paper_2202_07235_b200/build_var/trace.so timeout 300 python tools/trace_align.py > gpurun_out/r3t_trace_tct2.txt 2>&1
grep -v Warn gpurun_out/r3t_trace_tct2.txt | grep -v '"' 
