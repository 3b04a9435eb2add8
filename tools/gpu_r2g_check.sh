#!/bin/bash
# Round-2 session g: re-check the restored checkpoint on a fresh box (GPU tests, smoke, default bench).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_gpu_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2g_gpu_pytest.log
tail -3 gpurun_out/r2g_gpu_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2g_smoke.log 2>&1; tail -1 gpurun_out/r2g_smoke.log
timeout 600 python bench.py > gpurun_out/r2g_bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/r2g_bench.log | cut -c1-600
