#!/bin/bash
# compress kernels: timing A/B and one ncu --set full capture of compress_mma_kernel (round 2)
mkdir -p gpurun_out
python tools/compress_probe.py > gpurun_out/cp_mma.txt 2>&1
RSVD_COMPRESS_MMA=0 python tools/compress_probe.py > gpurun_out/cp_old.txt 2>&1
cat gpurun_out/cp_mma.txt gpurun_out/cp_old.txt
ncu --set full --import-source on --clock-control none -k regex:compress_mma -c 1 -o gpurun_out/cp_mma -f python tools/compress_probe.py --reps 1 > gpurun_out/cp_ncu.log 2>&1
tail -3 gpurun_out/cp_ncu.log
