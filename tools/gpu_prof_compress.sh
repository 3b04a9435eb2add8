#!/bin/bash
# Time the compress kernel at the Large image shape, then one ncu --set full capture of it.
TAG=${1:-cpt}; shift
mkdir -p gpurun_out
timeout 300 python tools/prof_compress.py "$@" > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"compress_tc" -s 1 -c 1 \
  -o gpurun_out/${TAG} python tools/prof_compress.py --reps 1 "$@" > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; cat gpurun_out/${TAG}_plain.log; tail -3 gpurun_out/${TAG}_ncu.log
