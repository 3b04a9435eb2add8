"""CTA timeline of the two-kernel align path (diagnostic; needs the -DRSVD_TRACE library variant):

    python paper_2202_07235_b200/build.py -DRSVD_TRACE --out=$PWD/paper_2202_07235_b200/build_var/trace.so
    RSVD_LIB=paper_2202_07235_b200/build_var/trace.so python tools/trace_align.py [--M 16384 --T 8192]

Every CTA of contract_tc_kernel and fft2_reduce_kernel records %globaltimer stamps (entry, dependency
wait passed, first accumulator / first item ready, exit).  Per chunk this prints where the time between
two chunk starts goes: contraction span and tail, the gap to the transform's wait, the transform's
first-item latency, span and tail.  Random rings of the config's shape (timing does not depend on values)."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2202_07235_b200 import api, _lib  # noqa: E402
from synth import CONFIGS, radial_grid  # noqa: E402

REC = np.dtype([("t0", "<u8"), ("t1", "<u8"), ("t2", "<u8"), ("t3", "<u8"), ("kb", "<u4"), ("key", "<u4")])


def dump(lib, name, reset=True):
    fn = getattr(lib, "rsvd_trace_dump_" + name)
    fn.restype = ctypes.c_int
    buf = np.zeros(1 << 20, dtype=REC)
    n = fn(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(len(buf)), ctypes.c_int(1 if reset else 0))
    assert n >= 0, "trace dump failed"
    return buf[:n]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="large")
    p.add_argument("--M", type=int, default=16384)
    p.add_argument("--T", type=int, default=8192)
    p.add_argument("--mode", default="image", choices=["image", "pair"])
    p.add_argument("--work-mb", type=int, default=None)
    a = p.parse_args()
    c = CONFIGS[a.config]
    R, Q, H = c["R"], c["Q"], c["H"][0]
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((a.M, R, Q), dtype=torch.complex64, device="cuda", generator=g)
    B = torch.randn((a.T, R, Q), dtype=torch.complex64, device="cuda", generator=g)
    k, w = radial_grid(R)
    U, _ = api.build_basis(B[:1024], w, H)
    wd = torch.tensor(w, device="cuda")
    Ud = torch.tensor(U, device="cuda")
    ib = api.compress(A, wd, Ud, api.SIDE_IMAGE)
    tb = api.compress(B, wd, Ud, api.SIDE_TEMPLATE)
    del A, B
    wb = a.work_mb * (1 << 20) if a.work_mb else api.align_workspace_bytes(a.M, a.T, Q, H)
    work = torch.empty(wb // 4, dtype=torch.float32, device="cuda")
    mode = api.PER_IMAGE if a.mode == "image" else api.PER_PAIR
    lib = _lib.lib()

    def run():
        return api.align_argmax(ib, a.M, tb, a.T, Q, H, mode, work)

    run()
    torch.cuda.synchronize()
    dump(lib, "contract"), dump(lib, "fft")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    C, F = dump(lib, "contract"), dump(lib, "fft")
    assert len(C) and len(F), "no trace records: is RSVD_LIB the -DRSVD_TRACE variant?"
    C = C.astype([(n, "<i8") if n.startswith("t") else (n, "<u4") for n in REC.names])   # signed differences
    F = F.astype([(n, "<i8") if n.startswith("t") else (n, "<u4") for n in REC.names])
    t_origin = min(C["t0"].min(), F["t0"].min())
    keys = np.unique(C["key"])
    rows = []
    for kk in keys:
        c_ = C[C["key"] == kk]
        f_ = F[F["key"] == kk]
        rows.append(dict(
            c0=c_["t0"].min(), c0med=np.median(c_["t0"]), cwait=np.median(c_["t1"]), cacc=np.median(c_["t2"]),
            c3med=np.median(c_["t3"]), c3=c_["t3"].max(), nc=len(c_),
            f0=f_["t0"].min(), f0med=np.median(f_["t0"]), fw=np.median(f_["t1"]), fwmin=f_["t1"].min(),
            ff=np.median(f_["t2"]), f3med=np.median(f_["t3"]), f3=f_["t3"].max(), nf=len(f_)))
    rows.sort(key=lambda r: r["c0"])
    rows = rows[2:] if len(rows) > 8 else rows            # drop the first chunks (pipeline start)
    us = lambda x: np.mean(x) / 1e3  # noqa: E731
    per = np.diff([r["c0"] for r in rows])
    out = {
        "align_ms_events": ms,
        "chunks": len(keys),
        "ctas_per_chunk_contract": int(np.median([r["nc"] for r in rows])),
        "ctas_per_chunk_fft": int(np.median([r["nf"] for r in rows])),
        "chunk_period_us": us(per),
        "contract: first CTA start -> median CTA start": us([r["c0med"] - r["c0"] for r in rows]),
        "contract: first CTA start -> median epilogue wait passed": us([r["cwait"] - r["c0"] for r in rows]),
        "contract: first CTA start -> median first accumulator": us([r["cacc"] - r["c0"] for r in rows]),
        "contract: first CTA start -> median CTA end": us([r["c3med"] - r["c0"] for r in rows]),
        "contract: first CTA start -> last CTA end (span)": us([r["c3"] - r["c0"] for r in rows]),
        "contract tail: median end -> last end": us([r["c3"] - r["c3med"] for r in rows]),
        "fft: first CTA start (rel. contract last end)": us([r["f0"] - r["c3"] for r in rows]),
        "fft: wait passed (median, rel. contract last end)": us([r["fw"] - r["c3"] for r in rows]),
        "fft: first item landed (median, rel. wait passed)": us([r["ff"] - r["fw"] for r in rows]),
        "fft: wait passed -> median CTA end": us([r["f3med"] - r["fw"] for r in rows]),
        "fft: wait passed -> last CTA end (span)": us([r["f3"] - r["fw"] for r in rows]),
        "fft tail: median end -> last end": us([r["f3"] - r["f3med"] for r in rows]),
        "next contract first start (rel. fft last end)": us([rows[i + 1]["c0"] - rows[i]["f3"] for i in range(len(rows) - 1)]),
        "next contract epilogue wait passed (rel. fft last end)": us([rows[i + 1]["cwait"] - rows[i]["f3"] for i in range(len(rows) - 1)]),
    }
    busy_c = float((C["t3"] - C["t0"]).sum()) / 1e6
    busy_f = float((F["t3"] - F["t0"]).sum()) / 1e6
    span = float(max(C["t3"].max(), F["t3"].max()) - t_origin) / 1e6
    out["timeline_ms"] = span
    out["cta_ms_contract_sum"] = busy_c
    out["cta_ms_fft_sum"] = busy_f
    for k_, v in out.items():
        print(f"{k_:60s} {v:12.3f}" if isinstance(v, float) else f"{k_:60s} {v}")


if __name__ == "__main__":
    main()
