#!/bin/bash
# ncu of the fast-path (fp16 spectrum) transform vs the fp32 one, same shape/chunk
TAG=${1:-r2pf}
mkdir -p gpurun_out
ARGS="--M 4096 --T 2048 --work-mb 128"
RSVD_PRECISION=fast timeout 300 python tools/prof_align.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
RSVD_PRECISION=fast timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fft2" -s 2 -c 1 \
  -o gpurun_out/${TAG}_h python tools/prof_align.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"; tail -2 gpurun_out/${TAG}_ncu.log
