"""Row f4 measurement: many volumes aligned to one target (N_A = 96 volumes, one
target, H_C = H_D = H).  Prints one JSON line in bench.py's shape.

Workload: L = 48 (M = 97, P = 128), R = 49 radial nodes, nb = M = 97
beta values, H = 16, phantoms of 60 atoms, volumes = jittered rotated copies of the target.
Timed step (device, CUDA events, inputs resident): items 7-11 of the operation count (PAPER.md:
1036-1040): principal shells of the volumes -> Steps 1/1b -> Steps 2/3 with the per-volume argmax.
The per-target precomputations (items 1-6: kernels, eigen-solves, target shells, Wigner table) are
timed once, separately.  `--landscape` also writes the full landscape X [n][nb][P][P].

    python tools/vol_bench.py [--n 96] [--L 48] [--H 16] [--steps 10] [--warmup 3] [--landscape]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2202_07235_b200 import api  # noqa: E402
from synth import volumes as sv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=96)
ap.add_argument("--L", type=int, default=48)
ap.add_argument("--R", type=int, default=None)
ap.add_argument("--H", type=int, default=16)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--landscape", action="store_true")
ap.add_argument("--no-cpu-baseline", action="store_true", help="(accepted for compatibility; no CPU leg)")
a = ap.parse_args()
L, R, H = a.L, a.R or a.L + 1, a.H
t0 = time.time()
vs = sv.make_volumes(L, R, min(a.n, 96), atoms=60, seed=7, jitter=0.01)
reps = (a.n + len(vs.volumes) - 1) // len(vs.volumes)
vols = torch.as_tensor(np.concatenate([vs.volumes] * reps)[:a.n]).cuda()
gen_s = time.time() - t0
w = torch.as_tensor(vs.w).cuda()
betas = torch.as_tensor(vs.betas).cuda()
P, nb, M = vs.P, len(vs.betas), 2 * L + 1
s = torch.cuda.current_stream()

# per-target precomputations (items 1-6)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t_pre = time.time()
al = api.VolumeAligner(torch.as_tensor(vs.target).cuda(), w, L, H, H, betas, P=P)
torch.cuda.synchronize()
pre_ms = (time.time() - t_pre) * 1e3

shells = torch.empty(a.n, H, (L + 1) ** 2, dtype=torch.complex64, device="cuda")
Y = torch.empty(a.n, H, M, M, dtype=torch.complex64, device="cuda")
keys = torch.zeros(a.n, dtype=torch.int64, device="cuda")
X = torch.empty(a.n, nb, P, P, dtype=torch.float32, device="cuda") if a.landscape else None
ev = ("compress", "degrees", "align")


def step(timed=False):
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timed else None
    if timed:
        marks[0].record()
    api.vol_compress(vols, w, al.U, L, out=shells)
    if timed:
        marks[1].record()
    api.vol_degrees(shells, al.shell_b, L, al.V, out=Y)
    if timed:
        marks[2].record()
    keys.zero_()
    api.vol_align(Y, al.T, L, P, landscape=a.landscape, keys=keys, X=X)
    if timed:
        marks[3].record()
        return marks


for _ in range(a.warmup):
    step()
torch.cuda.synchronize()
e0.record()
for _ in range(a.steps):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
allm = [step(True) for _ in range(a.steps)]
torch.cuda.synchronize()
kern = {k: float(np.mean([m[i].elapsed_time(m[i + 1]) for m in allm])) for i, k in enumerate(ev)}
val, b, aa, g = api.vol_best(keys, P)

# algorithmic work per volume (DESIGN.md §6 f4): Step 2 HD M^2 nb complex*real MACs (4 flops), Step 3
# nb (M + P) length-P complex FFTs at 5 P log2 P flops, Steps 1/1b sum_{m1,m2} (L+1-max) (HC+HD) complex
# MACs (8 flops), shells R NC HC complex*real MACs (4 flops)
NC = (L + 1) ** 2
s1 = sum((L + 1 - max(abs(m1), abs(m2))) for m1 in range(-L, L + 1) for m2 in range(-L, L + 1))
fl = {"compress": 4.0 * R * NC * H, "degrees": 8.0 * s1 * 2 * H, "align": 4.0 * H * M * M * nb + nb * (M + P) * 5 * P * np.log2(P)}
fl_tot = sum(fl.values())
line = {
    "metric": "volume-target pairs/s (landscape over nb x P x P rotations, radial+degree SVD)",
    "value": a.n / (ms * 1e-3), "unit": "volumes/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
    "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None,
    "dtype": "f32", "data": "synthetic (Gaussian-atom phantoms; PAPER.md's TRPV1 volumes are not available)",
    "config": {"workload": "f4 volumes", "n_volumes": a.n, "L": L, "M": M, "R": R, "P": P, "nb": nb, "HC": H,
               "HD": H, "landscape_out": a.landscape},
    "kernel_ms": {k: round(v, 4) for k, v in kern.items()},
    "achieved_tflops": {k: round(fl[k] * a.n / (kern[k] * 1e-3) / 1e12, 3) for k in kern},
    "step_tflops": round(fl_tot * a.n / (ms * 1e-3) / 1e12, 3),
    "precompute_ms": round(pre_ms, 2),
    "gen_seconds": round(gen_s, 1),
}
# winner check against the applied rotations (exact copies modulo jitter; degenerate beta compared as matrices)
ok = 0
for i in range(min(a.n, 96)):
    tb, ta, tg = vs.tau_index[i]
    Rt = sv.rotation(2 * np.pi * ta / P, vs.betas[tb], 2 * np.pi * tg / P)
    Rf = sv.rotation(2 * np.pi * int(aa[i]) / P, vs.betas[int(b[i])], 2 * np.pi * int(g[i]) / P)
    ok += int(np.abs(Rt - Rf).max() < 1e-6)
line["winners_recovered"] = f"{ok}/{min(a.n, 96)}"
line["cpu_baseline"] = None      # tools never execute oracle/ (only tests/, smoke() and bench.py may)
print(json.dumps(line))
