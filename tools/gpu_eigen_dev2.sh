#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "eigen or basis" 2>&1 | tail -15 | tee gpurun_out/r2g_eigen_tests.log
