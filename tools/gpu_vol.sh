#!/bin/bash
# f4 measurement lines (paper-size N_A = 96, and 1024 volumes; argmax and landscape modes)
mkdir -p gpurun_out
for args in "--n 96" "--n 96 --landscape --no-cpu-baseline" "--n 1024 --no-cpu-baseline" "--n 1024 --landscape --no-cpu-baseline"; do
  timeout 600 python tools/vol_bench.py $args 2>&1 | tail -1
done
