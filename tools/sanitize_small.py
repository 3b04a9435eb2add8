"""Small workload for compute-sanitizer runs (racecheck / synccheck): Tiny smoke + a Small-shaped
align (Q = 128, H = 8, 256 x 256 pairs) in every mode on the TC path, and the SIMT path once."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402
from paper_2202_07235_b200 import api  # noqa: E402
from synth import make_dataset  # noqa: E402

g.smoke()
d = make_dataset("small", M=256, T=256, device="cuda")
w = d.w.contiguous()
for path in (api.PATH_TC, api.PATH_SIMT):
    api.set_path(path)
    U, _ = api.build_basis(d.templates, w.cpu().numpy(), 8)
    Ud = torch.tensor(U, device="cuda")
    ib = api.compress(d.images, w, Ud, api.SIDE_IMAGE)
    tb = api.compress(d.templates, w, Ud, api.SIDE_TEMPLATE)
    work = torch.empty(api.align_workspace_bytes(256, 256, d.Q, 8) // 4, dtype=torch.float32, device="cuda")
    api.align_argmax(ib, 256, tb, 256, d.Q, 8, api.PER_PAIR, work)
    api.align_argmax(ib, 256, tb, 256, d.Q, 8, api.PER_IMAGE, work)
    api.align_landscape(ib, 256, tb, 256, d.Q, 8, work)
torch.cuda.synchronize()
print("sanitize workload ok")
