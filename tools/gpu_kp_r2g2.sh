#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/kp_ref.pt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "basis or ctf or transl" tests/test_gpu_dist.py tests/test_gpu_nccl.py 2>&1 | tail -2
bash tools/gpu_kp_ab.sh paper_2202_07235_b200/librsvd.so paper_2202_07235_b200/librsvd.so 2>&1 | tee gpurun_out/r2g_kp_variants2.txt
rm -f gpurun_out/kp_ref.pt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kernel_partials -c 1 -o gpurun_out/r2g_kp_mma2 -f python tools/prof_partials.py 1024 > gpurun_out/r2g_kp_ncu2.log 2>&1; echo "ncu exit $?"
