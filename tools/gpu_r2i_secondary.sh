#!/bin/bash
# every secondary config's bench line with the final library (tag r02i) + the fast-path line
TAG=${1:-r02i}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${TAG}_bench_${name}.log 2>&1; echo "$name exit $?"; tail -1 gpurun_out/${TAG}_bench_${name}.log > gpurun_out/${TAG}_bench_${name}.json; }
run large_fast --config large --precision fast --steps 10 --warmup 3 --no-cpu-baseline --no-e2e
bash tools/bench_all_secondary.sh ${TAG}
