#!/bin/bash
# One GPU session: parity tests, a default bench line, and the ncu launch list of the same command.
# Usage (from the repo root on the GPU box): bash tools/gpu_round.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"contract|fft|compress|kernel_partials|kernel_reduce|winners" -c 3000 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/${TAG}_ncu.log
tail -3 gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_bench.log
