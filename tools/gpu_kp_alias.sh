#!/bin/bash
# diagonal partials tiles staged once (xj aliased to xi): A/B against the previous library + parity
mkdir -p gpurun_out; rm -f gpurun_out/kp_ref.pt
bash tools/gpu_kp_ab.sh build_var/kp_head.so build_var/kp_alias.so build_var/kp_head.so build_var/kp_alias.so 2>&1 | tee gpurun_out/r2h_kp_alias.txt
rm -f gpurun_out/kp_ref.pt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "basis or ctf or transl or eigen" tests/test_gpu_dist.py tests/test_gpu_nccl.py 2>&1 | tail -2
