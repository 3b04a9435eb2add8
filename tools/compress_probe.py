"""Compress-only timing probe (Large images: n x R=128 x Q=512, H=24), for ncu / A-B of the compress
kernels.  Synthetic random rings and an orthonormal random basis; not a parity check."""
import argparse
import sys, os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_07235_b200 import api  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=16384)
p.add_argument("--R", type=int, default=128)
p.add_argument("--Q", type=int, default=512)
p.add_argument("--H", type=int, default=24)
p.add_argument("--reps", type=int, default=5)
a = p.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
rings = torch.randn(a.n, a.R, a.Q, dtype=torch.complex64, device="cuda", generator=g)
w = torch.rand(a.R, dtype=torch.float64, device="cuda", generator=g) + 0.5
U = torch.linalg.qr(torch.randn(a.R, a.H, dtype=torch.float64, device="cuda", generator=g))[0].contiguous()
out = api.compress(rings, w, U, api.SIDE_IMAGE)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(a.reps):
    ev[0].record()
    api.compress(rings, w, U, api.SIDE_IMAGE, out=out)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
gb = (a.n * a.R * a.Q * 8 + out.numel() * 4) / 1e9
print(f"compress n={a.n} R={a.R} Q={a.Q} H={a.H}: median {sorted(ts)[len(ts)//2]:.3f} ms, {gb:.2f} GB -> "
      f"{gb / (sorted(ts)[len(ts)//2] * 1e-3) / 1e3:.2f} TB/s")
