"""Per-rank phase times of the Large step for rank 0 of a G-GPU run on the dist.grid_shape grid
(GI image shards x GT template shards; `python tools/shard_estimate.py G [GI]`), without the
collectives -- an estimate of the multi-GPU step on one GPU (diagnostic, not the bench)."""
import json, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_07235_b200 import api  # noqa: E402
from paper_2202_07235_b200 import dist as pdist  # noqa: E402
from synth import CONFIGS, make_dataset  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = CONFIGS["large"]
T = cfg["T"]
GI, GT = (int(sys.argv[2]), G // int(sys.argv[2])) if len(sys.argv) > 2 else pdist.grid_shape(G, cfg["M"], T)
t1 = pdist.shard_range(T, GT, 0, api.kernel_chunk())[1]
b1 = pdist.basis_range(T, G, 0, api.kernel_chunk(), GI)[1]
ds = make_dataset("large", device="cuda", t_range=(0, t1))
m1 = pdist.image_range(ds.images.shape[0], GI, 0)[1]
imgs, tm = ds.images[:m1].contiguous(), ds.templates
M, R, Q = imgs.shape
H = cfg["H"][0]
w = ds.w.contiguous()
ib = torch.empty(api.block_bytes(M, Q, H, api.SIDE_IMAGE) // 4, dtype=torch.float32, device="cuda")
tb = torch.empty(api.block_bytes(t1, Q, H, api.SIDE_TEMPLATE) // 4, dtype=torch.float32, device="cuda")
work = torch.empty(api.align_workspace_bytes(M, t1, Q, H) // 4, dtype=torch.float32, device="cuda")
keys = torch.zeros(M, dtype=torch.int64, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
res = {}
for rep in range(4):
    e = [ev() for _ in range(6)]
    e[0].record()
    part = api.kernel_partials(tm[:b1])
    e[1].record()
    C = api.kernel_reduce(part, T, Q, w)
    th = time.perf_counter()
    Ud, lam, _ = api.eigen_basis_device(C, H)            # the bench's default a0 path (no host round trip)
    host_ms = (time.perf_counter() - th) * 1e3
    e[2].record()
    api.compress(imgs, w, Ud, api.SIDE_IMAGE, out=ib)
    e[3].record()
    api.compress(tm, w, Ud, api.SIDE_TEMPLATE, out=tb)
    e[4].record()
    api.winners_reset(keys)
    api.align_argmax(ib, M, tb, t1, Q, H, api.PER_IMAGE, work, best_key=keys)
    e[5].record()
    torch.cuda.synchronize()
    res = {"G": G, "GI": GI, "GT": GT, "M_shard": M, "T_shard": t1, "T_basis": b1, "partials_ms": e[0].elapsed_time(e[1]), "reduce_eigen_ms": e[1].elapsed_time(e[2]),
           "host_enqueue_ms": host_ms, "compress_images_ms": e[2].elapsed_time(e[3]),
           "compress_templates_ms": e[3].elapsed_time(e[4]), "align_ms": e[4].elapsed_time(e[5]),
           "total_ms": e[0].elapsed_time(e[5])}
print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.items()}))
