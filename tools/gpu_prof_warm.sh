#!/bin/bash
# ncu --set full of steady-state (warm L2, no cache flush) contraction + FFT launches at the Large shape.
TAG=${1:-warm}; shift
mkdir -p gpurun_out
ARGS="--M 16384 --T 512 --work-mb 128 --reps 1 $*"
timeout 300 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"contract|fft" -s 40 -c 2 \
  -o gpurun_out/${TAG} python tools/prof_align.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; tail -2 gpurun_out/${TAG}_ncu.log
