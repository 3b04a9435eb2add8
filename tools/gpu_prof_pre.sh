#!/bin/bash
# ncu --set full capture of the precompute kernels (kernel partials, TC compress) at the Large shape.
TAG=${1:-prep}
mkdir -p gpurun_out
ARGS="--M 4096 --T 4096 --reps 1"
timeout 300 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"kernel_partials|compress" -c 3 \
  -o gpurun_out/${TAG} python tools/prof_align.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; tail -2 gpurun_out/${TAG}_ncu.log
