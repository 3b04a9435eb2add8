#!/bin/bash
# double-buffered workspace: parity (TC parity + large configs), A/B vs the single-buffer PDL chain, trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r3d_parity.log 2>&1; echo "parity exit $?" >> gpurun_out/r3d_parity.log; tail -2 gpurun_out/r3d_parity.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off"
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['step_roofline']['kernel_ms_per_step']; print('$2', d['ms_per_step'], d['phases_ms_last_step']['align'], k['contract'], k['fft_reduce'], d['clocks']['sm_mhz'], d['config'].get('workspace_mb'))" 2>&1 | tail -1; }
for rep in 1 2; do
RSVD_DBUF=0 timeout 300 $B --work-mb 128 > gpurun_out/r3d_single_$rep.log 2>&1; summ gpurun_out/r3d_single_$rep.log single128
timeout 300 $B > gpurun_out/r3d_dbuf_$rep.log 2>&1; summ gpurun_out/r3d_dbuf_$rep.log dbuf
done
timeout 300 $B --precision fast > gpurun_out/r3d_fast.log 2>&1; summ gpurun_out/r3d_fast.log dbuf_fast
RSVD_LIB=paper_2202_07235_b200/build_var/trace.so timeout 300 python tools/trace_align.py > gpurun_out/r3d_trace.txt 2>&1; cat gpurun_out/r3d_trace.txt | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -m gpu -k "large" > gpurun_out/r3d_configs.log 2>&1; echo "configs exit $?" >> gpurun_out/r3d_configs.log; tail -2 gpurun_out/r3d_configs.log
