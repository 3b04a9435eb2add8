#!/bin/bash
# ncu --set full capture of the align kernels at the Large shape on a reduced M x T.
# Usage: bash tools/gpu_prof.sh TAG [extra prof_align args]
TAG=${1:-prof}; shift
mkdir -p gpurun_out
ARGS="--M 4096 --T 2048 --work-mb 128 $*"
timeout 300 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"contract|fft" -s 4 -c 2 \
  -o gpurun_out/${TAG} python tools/prof_align.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; tail -3 gpurun_out/${TAG}_ncu.log
