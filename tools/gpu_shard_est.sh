#!/bin/bash
# per-rank step estimate on one GPU (collectives excluded) for G = 1, 2, 4, 8 on the template-only grid
# (the bench default) and on the dist.grid_shape image x template grid
mkdir -p gpurun_out
for a in "1 1" "2 1" "4 1" "8 1" "2" "4" "8"; do timeout 300 python tools/shard_estimate.py $a 2>&1 | tail -1; done | tee gpurun_out/r2h_shard_estimate.txt
