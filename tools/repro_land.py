"""Diagnostic: landscape mode at the Translations shape (R=64, Q=256, H=16) on random rings."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_07235_b200 import api  # noqa: E402
from synth import radial_grid  # noqa: E402

M, T, R, Q, H = [int(x) for x in sys.argv[1:6]]
mode = sys.argv[6] if len(sys.argv) > 6 else "land"
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((M, R, Q), dtype=torch.complex64, device="cuda", generator=g)
B = torch.randn((T, R, Q), dtype=torch.complex64, device="cuda", generator=g)
k, w = radial_grid(R)
U, _ = api.build_basis(B, w, H)
wd = torch.tensor(w, device="cuda"); Ud = torch.tensor(U, device="cuda")
ib = api.compress(A, wd, Ud, api.SIDE_IMAGE); tb = api.compress(B, wd, Ud, api.SIDE_TEMPLATE)
torch.cuda.synchronize(); print("compress ok", flush=True)
work = torch.empty((128 << 20) // 4, dtype=torch.float32, device="cuda")
if mode == "land":
    X = torch.empty((M, T, Q), dtype=torch.float32, device="cuda")
    api.align_landscape(ib, M, tb, T, Q, H, work, X=X, ld_m=T * Q, ld_t=Q)
    torch.cuda.synchronize(); print("landscape ok", float(X[0, 0, 0]), flush=True)
else:
    v, kk = api.align_argmax(ib, M, tb, T, Q, H, api.PER_PAIR if mode == "pair" else api.PER_IMAGE, work) if mode == "pair" else (None, None)
    if mode == "image":
        keys = api.align_argmax(ib, M, tb, T, Q, H, api.PER_IMAGE, work)
    torch.cuda.synchronize(); print(mode, "ok", flush=True)
