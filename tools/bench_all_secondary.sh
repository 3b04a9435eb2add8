#!/bin/bash
# (secondary configs only: the Large default and fast lines come from gpu_r2_final3.sh) One clocked bench.py line per BASELINE config / mode; writes gpurun_out/${TAG}_bench_*.json
TAG=${1:-r02}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${TAG}_bench_${name}.log 2>&1; echo "$name exit $?"; tail -1 gpurun_out/${TAG}_bench_${name}.log > gpurun_out/${TAG}_bench_${name}.json; }

run tiny --config tiny --steps 10 --warmup 3 --no-cpu-baseline --traffic off
run small --config small --steps 10 --warmup 3 --no-cpu-baseline
for h in 64 32 16 8; do run medium_h$h --config medium --H $h --steps 10 --warmup 3 --no-cpu-baseline; done
run translations --config translations --steps 10 --warmup 3 --no-cpu-baseline
run translations_landscape --config translations --mode landscape --steps 5 --warmup 3 --no-cpu-baseline --traffic off
run large_per_pair --config large --mode per_pair --steps 5 --warmup 3 --no-cpu-baseline --traffic off

run large_ctf4 --config large --ctf-groups 4 --steps 10 --warmup 3 --no-cpu-baseline --traffic off
