"""ncu driver for the kernel-partials kernel (row a0) at the Large ring shape on a reduced T."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_07235_b200 import api  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device="cuda").manual_seed(0)
B = torch.randn((T, 128, 512), dtype=torch.complex64, device="cuda", generator=g)
for _ in range(2):
    P = api.kernel_partials(B)
torch.cuda.synchronize()
print("ok", T, tuple(P.shape))
