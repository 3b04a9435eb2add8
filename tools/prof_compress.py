"""Time rsvd_compress (image side) at the Large shape: n rows x R=128 rings x Q=512, H=24 (profiling aid)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_07235_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--R", type=int, default=128)
ap.add_argument("--Q", type=int, default=512)
ap.add_argument("--H", type=int, default=24)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
rings = torch.randn(a.n, a.R, a.Q, dtype=torch.complex64, device="cuda", generator=g)
w = torch.rand(a.R, dtype=torch.float64, device="cuda", generator=g) + 0.5
U, _ = torch.linalg.qr(torch.randn(a.R, a.H, dtype=torch.float64, device="cuda", generator=g))
U = U.contiguous()
out = api.compress(rings, w, U, api.SIDE_IMAGE)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
for i in range(a.reps):
    ev[2 * i].record()
    api.compress(rings, w, U, api.SIDE_IMAGE, out=out)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
ms = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(a.reps)]
gb = a.n * a.R * a.Q * 8 / 1e9
print(f"compress n={a.n} R={a.R} Q={a.Q} H={a.H}: ms {min(ms):.3f} (median {sorted(ms)[len(ms)//2]:.3f}); "
      f"ring read {gb:.2f} GB -> {gb / min(ms):.2f} TB/s")
