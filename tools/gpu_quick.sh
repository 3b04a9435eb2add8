#!/bin/bash
# Quick GPU check: parity tests (bounded), then a short bench line with per-kernel timing.
TAG=${1:-quick}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_parity.log 2>&1; echo "parity exit $?" >> gpurun_out/${TAG}_parity.log
tail -15 gpurun_out/${TAG}_parity.log
if grep -q "parity exit 0" gpurun_out/${TAG}_parity.log; then
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
  tail -2 gpurun_out/${TAG}_bench.log | cut -c1-3000
fi
