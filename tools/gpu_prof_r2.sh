#!/bin/bash
# ncu --set full (with source) of the align kernels at the Large shape: one contraction + one fft3
# launch, and one fft2 launch for comparison.  Usage: bash tools/gpu_prof_r2.sh TAG
TAG=${1:-r2prof}
mkdir -p gpurun_out
ARGS="--M 4096 --T 2048 --work-mb 128"
timeout 300 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
RSVD_FFT=2 timeout 300 python tools/prof_align.py $ARGS >> gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"contract|fft" -s 4 -c 2 \
  -o gpurun_out/${TAG}_v3 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1 && \
RSVD_FFT=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fft" -s 2 -c 1 \
  -o gpurun_out/${TAG}_v2 python tools/prof_align.py $ARGS >> gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; tail -3 gpurun_out/${TAG}_ncu.log
