#!/bin/bash
# compress timing: default library and group-size variants
for v in default hg4 hg12 hg16; do
  if [ $v = default ]; then L=""; else L=$PWD/paper_2202_07235_b200/build/variants/$v.so; fi
  echo "== $v"; RSVD_LIB=$L timeout 120 python tools/prof_compress.py 2>&1 | tail -1
  RSVD_LIB=$L timeout 120 python tools/prof_compress.py --Q 1024 --n 8192 2>&1 | tail -1
  RSVD_LIB=$L timeout 120 python tools/prof_compress.py --Q 256 --n 16384 --H 16 2>&1 | tail -1
done
