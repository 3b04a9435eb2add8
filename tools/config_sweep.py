"""Throughput of the align path at every BASELINE.json config on one B200 (the bench times only
Large): Small (per-pair argmax, H=8), Medium per-pair argmax at H in {64, 32, 16, 8}, Large per-image
(H=24), Translations per-pair argmax and the full M x T x Q landscape streamed to HBM in image
blocks (H=16).  Device-resident compressed blocks, CUDA events, median of 5 after 2 warm-ups; the
step roofline of SURVEY.md 8(d): t_roof = pairs (8HQ / Pi_contr + 5Q log2 Q / Pi_fp32), plus the
landscape's HBM write time where it is written.  Accuracy against the oracle is checked (and the
Medium rank-sweep report printed) by tests/test_gpu_configs.py.  One JSON line per case."""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_07235_b200 import api  # noqa: E402
from synth import make_dataset  # noqa: E402

PK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
SM = torch.cuda.get_device_properties(0).multi_processor_count
PI_FP32 = SM * 128 * 2 * PK.get("sm_max_mhz", 1965.0) * 1e6
PI_F16 = PK.get("bf16_tflops", 1683.2) * 1e12
HBM = PK.get("hbm_gbs", 6539.9) * 1e9


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def t_roof(pairs, H, Q, path, land_bytes=0.0):
    pi_c = PI_F16 / 3.0 if path == api.PATH_TC else PI_FP32
    t = pairs * (8 * H * Q / pi_c + 5 * Q * math.log2(Q) / PI_FP32)
    return max(t, land_bytes / HBM)


def emit(**kw):
    print(json.dumps(kw), flush=True)


def run(name, Hs, modes):
    d = make_dataset(name, device="cuda")
    M, T, Q = d.images.shape[0], d.templates.shape[0], d.Q
    wd = d.w.contiguous()
    for H in Hs:
        U, _ = api.build_basis(d.templates, wd.cpu().numpy(), H)
        Ud = torch.tensor(U, device="cuda")
        ib = api.compress(d.images, wd, Ud, api.SIDE_IMAGE)
        tb = api.compress(d.templates, wd, Ud, api.SIDE_TEMPLATE)
        work = torch.empty(api.align_workspace_bytes(M, T, Q, H) // 4, dtype=torch.float32, device="cuda")
        path = api.path_for(Q, H)
        c_ms = timed(lambda: api.compress(d.images, wd, Ud, api.SIDE_IMAGE, out=ib))
        for mode in modes:
            if mode == "per_pair":
                val = torch.empty((M, T), dtype=torch.float32, device="cuda")
                k = torch.empty((M, T), dtype=torch.int32, device="cuda")
                ms = timed(lambda: api.align_argmax(ib, M, tb, T, Q, H, api.PER_PAIR, work, best_val=val, best_k=k))
                land = 0.0
                del val, k
            elif mode == "per_image":
                keys = torch.zeros(M, dtype=torch.int64, device="cuda")
                ms = timed(lambda: (api.winners_reset(keys),
                                    api.align_argmax(ib, M, tb, T, Q, H, api.PER_IMAGE, work, best_key=keys)))
                land = 0.0
            else:                                   # full landscape, streamed in image blocks
                blk = 4608
                X = torch.empty((blk, T, Q), dtype=torch.float32, device="cuda")
                bibs = [api.compress(d.images[b0:b0 + blk].contiguous(), wd, Ud, api.SIDE_IMAGE) for b0 in range(0, M, blk)]

                def land_all():
                    for i, b0 in enumerate(range(0, M, blk)):
                        nb = min(blk, M - b0)
                        api.align_landscape(bibs[i], nb, tb, T, Q, H, work, X=X, ld_m=T * Q, ld_t=Q)
                ms = timed(land_all, reps=3)
                land = float(M) * T * Q * 4
                del X, bibs
            pairs = M * T
            tr = t_roof(pairs, H, Q, path, land)
            emit(config=name, M=M, T=T, R=d.R, Q=Q, H=H, mode=mode, path="tc" if path == api.PATH_TC else "simt",
                 align_ms=round(ms, 3), pairs_per_s=pairs / (ms / 1e3), t_roof_ms=round(tr * 1e3, 3),
                 roofline_frac=round(tr * 1e3 / ms, 4), compress_images_ms=round(c_ms, 3),
                 landscape_gb=round(land / 1e9, 1) if land else None,
                 landscape_write_gbs=round(land / (ms / 1e3) / 1e9, 1) if land else None)
        del ib, tb, work
        torch.cuda.empty_cache()
    del d
    torch.cuda.empty_cache()


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "medium", "large", "translations"]
    if "small" in which:
        run("small", [8], ["per_pair"])
    if "medium" in which:
        run("medium", [64, 32, 16, 8], ["per_pair"])
    if "large" in which:
        run("large", [24], ["per_image"])
    if "translations" in which:
        run("translations", [16], ["per_pair", "landscape"])
