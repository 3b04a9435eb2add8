#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/kp_ref.pt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "basis or ctf or transl" tests/test_gpu_dist.py tests/test_gpu_nccl.py 2>&1 | tail -2
bash tools/gpu_kp_ab.sh paper_2202_07235_b200/librsvd.so paper_2202_07235_b200/librsvd.so 2>&1 | tee gpurun_out/r2g_kp_variants3.txt
rm -f gpurun_out/kp_ref.pt
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['ms_per_step'], d['phases_ms_last_step'], d['step_roofline'].get('kernel_ms_per_step'), d['step_roofline'].get('kernel_partials_fp64'), d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/r2g_kp3_bench.log 2>&1
summ gpurun_out/r2g_kp3_bench.log mma
