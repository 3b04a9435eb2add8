#!/bin/bash
# round-2 closing evidence with the final library (device eigen-solver as the bench default):
# GPU tests, smoke, the driver's default bench command, the ncu launch list of a short bench run
TAG=${1:-r02i}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_pytest.log
tail -3 gpurun_out/${TAG}_gpu_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
tail -2 gpurun_out/${TAG}_smoke.log
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${TAG}_bench_${name}.log 2>&1; echo "$name exit $?"; tail -1 gpurun_out/${TAG}_bench_${name}.log > gpurun_out/${TAG}_bench_${name}.json; }
run large
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --traffic off > gpurun_out/${TAG}_ncu_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"contract|fft|compress|kernel_partials|kernel_reduce|winners|eigen" -c 6000 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --traffic off > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu exit $?"
