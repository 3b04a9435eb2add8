#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "eigen or basis" 2>&1 | tail -3
timeout 120 python - <<'PY' 2>&1 | tee gpurun_out/r2h_eigen_time.txt
import torch, numpy as np, sys, time
sys.path.insert(0, ".")
from paper_2202_07235_b200 import api
for R, H in ((128, 24), (64, 16), (64, 64), (32, 8)):
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.standard_normal((R, R))); lam = np.exp(-np.arange(R) / 6.0)
    C = torch.tensor((Q * lam) @ Q.T, device="cuda")
    for _ in range(3): api.eigen_basis_device(C, H)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record(); U, l, info = api.eigen_basis_device(C, H); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    Cn = C.cpu().numpy(); th = []
    for _ in range(10):
        t = time.perf_counter(); api.eigen_basis(Cn, H); th.append((time.perf_counter() - t) * 1e3)
    print(f"R={R} H={H}: device {sorted(ts)[5]:.3f} ms (info {int(info.item())}), host {sorted(th)[5]:.3f} ms")
PY
