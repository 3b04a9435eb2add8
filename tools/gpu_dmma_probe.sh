#!/bin/bash
# fp64 peaks on this B200: DFMA (SIMT) vs DMMA (mma.sync m8n8k4 / m16n8k4 tensor core)
mkdir -p gpurun_out
timeout 300 python -c "
import torch
from paper_2202_07235_b200 import api
torch.cuda.init()
for k, it in (('dfma', 100000), ('dmma8', 20000), ('dmma16', 20000), ('dmma8', 40000), ('dmma16', 40000), ('dfma', 100000), ('ffma2', 200000)):
    print(k, it, round(api.probe_fp32(k, it), 2), 'TF/s')
" > gpurun_out/r2g_dmma_probe.txt 2>&1
cat gpurun_out/r2g_dmma_probe.txt
