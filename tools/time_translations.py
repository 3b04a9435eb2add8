"""Times row f2 at the Translations configuration (R=64, Q=256, H=16, 4096 base images x 9 shifts):
compressing the 36864 materialised translated rows vs rsvd_compress_translated on the base rows.
Prints one JSON line.  Diagnostic (not the bench)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_07235_b200 import api  # noqa: E402
from synth import make_dataset  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


d = make_dataset("translations", device="cuda")
H = 16
U, _ = api.build_basis(d.templates, d.w.cpu().numpy(), H)
Ud = torch.tensor(U, device="cuda")
w, k = d.w.contiguous(), d.k.contiguous()
base = d.images[4::9].contiguous()
sh = d.shift[:9].contiguous()
M = d.images.shape[0]
out = torch.empty(api.block_bytes(M, d.Q, H, api.SIDE_IMAGE) // 4, dtype=torch.float32, device="cuda")
t_mat = timed(lambda: api.compress(d.images, w, Ud, api.SIDE_IMAGE, out=out))
t_fus = timed(lambda: api.compress_translated(base, w, k, Ud, sh, api.SIDE_IMAGE, out=out))
print(json.dumps({"config": "translations", "rows": M, "base_rows": base.shape[0],
                  "compress_materialised_ms": round(t_mat, 3), "compress_translated_ms": round(t_fus, 3),
                  "ring_bytes_materialised": d.images.numel() * 8, "ring_bytes_base": base.numel() * 8}))
