#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 120 python tools/prof_compress.py 2>&1 | tail -1
timeout 120 python tools/prof_compress.py --Q 1024 --n 8192 2>&1 | tail -1
timeout 120 python tools/prof_compress.py --Q 256 --n 16384 --H 16 2>&1 | tail -1
