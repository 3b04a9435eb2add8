#!/bin/bash
# DMMA partials variants (Large shape, T = 8192) + ncu --set full of the default at T = 1024
mkdir -p gpurun_out; rm -f gpurun_out/kp_ref.pt
bash tools/gpu_kp_ab.sh build_var/kp_base.so build_var/kp_jb32.so build_var/kp_jb8.so build_var/kp_minb3.so build_var/kp_base.so 2>&1 | tee gpurun_out/r2g_kp_variants.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kernel_partials -c 1 -o gpurun_out/r2g_kp_mma -f python tools/prof_partials.py 1024 > gpurun_out/r2g_kp_ncu.log 2>&1; echo "ncu exit $?"
