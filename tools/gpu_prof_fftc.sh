#!/bin/bash
TAG=${1:-r2pc}
mkdir -p gpurun_out
ARGS="--M 4096 --T 2048 --work-mb 128"
RSVD_FFTC=1 timeout 300 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
RSVD_FFTC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fftc|contract" -s 2 -c 2 \
  -o gpurun_out/${TAG} python tools/prof_align.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; tail -2 gpurun_out/${TAG}_ncu.log
