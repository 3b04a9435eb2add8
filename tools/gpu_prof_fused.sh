#!/bin/bash
# ncu --set full of the fused align kernel at the Large shape on a reduced M x T
TAG=${1:-fusedprof}
mkdir -p gpurun_out
ARGS="--M 2048 --T 1024 --work-mb 128"
timeout 300 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"align_fused" -s 1 -c 1 \
  -o gpurun_out/${TAG} python tools/prof_align.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; tail -3 gpurun_out/${TAG}_ncu.log
