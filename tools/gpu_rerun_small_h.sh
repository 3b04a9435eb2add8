TAG=r02c
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${TAG}_bench_${name}.log 2>&1; echo "$name exit $?"; tail -1 gpurun_out/${TAG}_bench_${name}.log > gpurun_out/${TAG}_bench_${name}.json; }
run small --config small --steps 10 --warmup 3 --no-cpu-baseline
run medium_h8 --config medium --H 8 --steps 10 --warmup 3 --no-cpu-baseline
run medium_h16 --config medium --H 16 --steps 10 --warmup 3 --no-cpu-baseline
