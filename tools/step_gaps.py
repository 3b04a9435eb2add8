"""Kernel timeline of one Large bench-like step (torch.profiler / CUPTI): kernel start/end per launch
and the idle gaps between consecutive kernels, grouped by phase -- finds host/launch overhead inside a
step (diagnostic; not the bench)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_07235_b200 import api  # noqa: E402
from paper_2202_07235_b200 import dist as pdist  # noqa: E402
from synth import make_dataset  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
ds = make_dataset(cfg, device="cuda")
imgs, tm, w = ds.images, ds.templates, ds.w.contiguous()
M, R, Q = imgs.shape
T = tm.shape[0]
H = {"large": 24, "medium": 16, "small": 8}[cfg]
ib = torch.empty(api.block_bytes(M, Q, H, api.SIDE_IMAGE) // 4, dtype=torch.float32, device="cuda")
tb = torch.empty(api.block_bytes(T, Q, H, api.SIDE_TEMPLATE) // 4, dtype=torch.float32, device="cuda")
work = torch.empty(api.align_workspace_bytes(M, T, Q, H) // 4, dtype=torch.float32, device="cuda")
keys = torch.zeros(M, dtype=torch.int64, device="cuda")
U_dev = torch.zeros((R, H), dtype=torch.float64, device="cuda")


def step():
    U, _, info = pdist.basis_from_shards_device(tm, T, w, H)
    U_dev.copy_(U)
    api.compress(imgs, w, U_dev, api.SIDE_IMAGE, out=ib)
    api.compress(tm, w, U_dev, api.SIDE_TEMPLATE, out=tb)
    api.winners_reset(keys)
    api.align_argmax(ib, M, tb, T, Q, H, api.PER_IMAGE, work, best_key=keys)
    return pdist.combine_keys(keys, Q)


for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev])
t0 = ks[0][0]
gaps = {}
prev_end, prev_name = None, None
for s, e, n in ks:
    if prev_end is not None and s > prev_end:
        key = (prev_name[:40], n[:40])
        g = gaps.setdefault(key, [0, 0.0])
        g[0] += 1
        g[1] += s - prev_end
    prev_end, prev_name = max(prev_end or 0, e), n
total = ks[-1][1] - t0
busy = sum(e - s for s, e, _ in ks)
print(f"{cfg}: {len(ks)} kernels/copies, span {total/1e3:.3f} ms, summed durations {busy/1e3:.3f} ms")
for (a, b), (c, g) in sorted(gaps.items(), key=lambda x: -x[1][1])[:15]:
    print(f"  gap {g/1e3:8.3f} ms over {c:5d}  after {a:40s} before {b}")
print("first kernels:")
for s, e, n in ks[:12]:
    print(f"  {(s-t0)/1e3:9.3f} {(e-s)/1e3:8.3f} ms  {n[:80]}")
