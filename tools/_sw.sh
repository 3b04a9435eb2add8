bash tools/gpu_ws_sweep.sh 64 96 128 192
RSVD_NO_DISCARD=1 bash tools/gpu_ws_sweep.sh 64 128
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
