#!/bin/bash
# compress_mma_kernel vs compress_tc_kernel over config shapes (round 2)
for s in "512 128 24 16384" "512 128 16 16384" "512 128 8 16384" "256 64 32 4096" "256 64 16 4096" "256 64 8 4096" "128 32 8 1024" "256 64 16 36864"; do
  set -- $s
  a=$(python tools/compress_probe.py --Q $1 --R $2 --H $3 --n $4 | grep -o "median [0-9.]* ms")
  b=$(RSVD_COMPRESS_MMA=0 python tools/compress_probe.py --Q $1 --R $2 --H $3 --n $4 | grep -o "median [0-9.]* ms")
  echo "Q=$1 R=$2 H=$3 n=$4  mma: $a   simt: $b"
done
