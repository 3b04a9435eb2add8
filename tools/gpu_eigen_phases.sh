#!/bin/bash
# device eigen-solver phase times: diagnostic builds returning after phase 1 / 2 / 3 (RSVD_EV_STOP)
for k in 1 2 3 0; do
RSVD_LIB=build_var/ev$k.so timeout 120 python - <<PY
import torch, numpy as np, sys
sys.path.insert(0, ".")
from paper_2202_07235_b200 import api
R, H = 128, 24
rng = np.random.default_rng(0)
Q, _ = np.linalg.qr(rng.standard_normal((R, R))); lam = np.exp(-np.arange(R) / 6.0)
C = torch.tensor((Q * lam) @ Q.T, device="cuda")
for _ in range(3): api.eigen_basis_device(C, H)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); api.eigen_basis_device(C, H); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("stop after phase $k (0 = full):", round(sorted(ts)[5], 3), "ms")
PY
done
