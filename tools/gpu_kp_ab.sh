#!/bin/bash
# A/B of kernel-partials variants: Large-shape partials kernel time (T = 8192, CUDA events) per library
for L in "$@"; do
  n=$(basename $L .so)
  RSVD_LIB=$L timeout 120 python - <<PY
import torch, sys
sys.path.insert(0, ".")
from paper_2202_07235_b200 import api
g = torch.Generator(device="cuda").manual_seed(0)
B = torch.randn((8192, 128, 512), dtype=torch.complex64, device="cuda", generator=g)
P = api.kernel_partials(B); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record(); api.kernel_partials(B, out=P); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
L = torch.tril(P).cpu()                      # only r >= r' entries are written
S = L.sum(0)
import os
if not os.path.exists("gpurun_out/kp_ref.pt"): torch.save((L, S), "gpurun_out/kp_ref.pt"); same = "ref"
else:
    Lr, Sr = torch.load("gpurun_out/kp_ref.pt")
    same = "bitwise" if (Lr.shape == L.shape and torch.equal(Lr, L)) else "sum rel diff %.2e" % ((Sr - S).abs().max() / Sr.abs().max()).item()
print("$n", "partials ms", sorted(ts)[len(ts)//2], same)
PY
done
