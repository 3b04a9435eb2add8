#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "basis or ctf or transl" tests/test_gpu_dist.py tests/test_gpu_nccl.py > gpurun_out/r2g_kp_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2g_kp_tests.log
tail -3 gpurun_out/r2g_kp_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step'], d['step_roofline'].get('kernel_ms_per_step'), d['step_roofline'].get('kernel_partials_fp64'), d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for v in mma mma; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/r2g_kp2_$v.log 2>&1
  summ gpurun_out/r2g_kp2_$v.log $v
done
