"""Small driver for ncu captures of the align kernels at a config's shape (R, Q, H) on a reduced
M x T (random rings; kernel timing does not depend on values).  Not a benchmark."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2202_07235_b200 import api  # noqa: E402
from synth import CONFIGS, radial_grid  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="large")
    p.add_argument("--M", type=int, default=1024)
    p.add_argument("--T", type=int, default=512)
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--mode", default="image", choices=["image", "pair", "landscape"])
    p.add_argument("--work-mb", type=int, default=None)
    a = p.parse_args()
    c = CONFIGS[a.config]
    R, Q, H = c["R"], c["Q"], c["H"][0]
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((a.M, R, Q), dtype=torch.complex64, device="cuda", generator=g)
    B = torch.randn((a.T, R, Q), dtype=torch.complex64, device="cuda", generator=g)
    k, w = radial_grid(R)
    U, _ = api.build_basis(B, w, H)
    wd = torch.tensor(w, device="cuda")
    Ud = torch.tensor(U, device="cuda")
    ib = api.compress(A, wd, Ud, api.SIDE_IMAGE)
    tb = api.compress(B, wd, Ud, api.SIDE_TEMPLATE)
    wb = a.work_mb * (1 << 20) if a.work_mb else api.align_workspace_bytes(a.M, a.T, Q, H)
    work = torch.empty(wb // 4, dtype=torch.float32, device="cuda")
    for _ in range(a.reps):
        if a.mode == "image":
            api.align_argmax(ib, a.M, tb, a.T, Q, H, api.PER_IMAGE, work)
        elif a.mode == "pair":
            api.align_argmax(ib, a.M, tb, a.T, Q, H, api.PER_PAIR, work)
        else:
            api.align_landscape(ib, a.M, tb, a.T, Q, H, work)
    torch.cuda.synchronize()
    print("ok", a.config, a.M, a.T, R, Q, H)


if __name__ == "__main__":
    main()
