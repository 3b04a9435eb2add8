#!/bin/bash
# round-2 session start on the box: GPU tests, FP32 probe, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gpu_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2a_gpu_pytest.log
python - > gpurun_out/r2a_probe.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2202_07235_b200 import api
for k in ["ffma", "ffma2", "fadd2", "ffma2", "ffma"]:
    print(k, round(api.probe_fp32(k), 2), "TFLOP/s")
PY
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r2a_bench.log
