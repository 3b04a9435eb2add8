#!/bin/bash
# round-2 closing ncu --set full captures of the default align kernels (steady-state launches of a
# Large-shape chunk; cache control none so L2 carries over from the previous kernel like in the bench)
TAG=${1:-r02final}
mkdir -p gpurun_out
ARGS="--M 4096 --T 2048 --work-mb 128"
timeout 300 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"contract|fft2" -s 6 -c 2 \
  -o gpurun_out/${TAG} python tools/prof_align.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; tail -2 gpurun_out/${TAG}_ncu.log
