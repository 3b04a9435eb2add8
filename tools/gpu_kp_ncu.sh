#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kernel_partials -c 1 -o gpurun_out/r2g_kp_mma -f python tools/prof_partials.py 1024 > gpurun_out/r2g_kp_ncu.log 2>&1; echo "ncu exit $?"
