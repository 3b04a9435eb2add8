#!/bin/bash
# round-2 evidence: GPU tests, smoke, every config's bench line, the default bench's ncu launch list
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_pytest.log
tail -3 gpurun_out/${TAG}_gpu_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
tail -2 gpurun_out/${TAG}_smoke.log
bash tools/bench_all.sh ${TAG}
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --traffic off > gpurun_out/${TAG}_ncu_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"contract|fft|compress|kernel_partials|kernel_reduce|winners" -c 6000 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --traffic off > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu exit $?"
