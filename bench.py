#!/usr/bin/env python
"""bench.py -- many-to-many radial-SVD rotational alignment on B200 (arXiv 2202.07235 hot path).

One "step" = one pass of the whole hot path over one batch of
synthetic input resident in HBM:
  a0 kernel-matrix partials on the rank's template shard -> all-gather (G > 1) -> reduce -> host
     eigen-solver -> U;
  a1 compress all images and the rank's template shard;
  a2-a4 contraction + length-Q FFT + per-image argmax (packed keys, t_offset = shard start);
  G > 1: all-gather of the per-image keys (NCCL over NVLink) + combine kernel.
value = M * T pairs / step time (whole job, max over ranks, CUDA events).  Templates are sharded
over the ranks (total work fixed: "strong" scaling).  Default workload: the Large config
(BASELINE.json configs[3]: R=128, Q=512, H=24, M=16384, T=8192), the configuration the north star's
scaling target is stated on; DESIGN.md explains the choice.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config large] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from synth import CONFIGS, make_dataset, sample_pairs  # noqa: E402

METRIC = "image–template pairs/s (full landscape over Q angles) at rank H; % roofline"
UNIT = "pairs/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="large", choices=list(CONFIGS))
    p.add_argument("--H", type=int, default=None)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--mode", default=None, choices=["per_image", "per_pair", "landscape"],
                   help="Step-4 output (default: the config's BASELINE mode -- per_image for Large, per_pair otherwise)")
    p.add_argument("--traffic", default="auto", choices=["auto", "off"],
                   help="measure the dominant kernel's DRAM bytes per launch with an ncu child run of the same "
                        "workload (rank 0, N = 1)")
    p.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--landscape-gb", type=float, default=8.0, help="landscape tile buffer (GB) for --mode landscape")
    p.add_argument("--ctf-groups", type=int, default=0,
                   help="row f3: split the images into G CTF groups (toy radial CTFs), one basis per group from "
                        "one kernel pass, templates compressed per group, one grouped align call (per-image mode)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-kernel-timing", action="store_true", help="(diagnostic) no per-kernel CUDA events in the timed region")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--e2e-img-block", type=int, default=512, help="image rows per streamed block (e2e)")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--work-mb", type=int, default=None, help="align workspace (default: library recommendation)")
    p.add_argument("--path", default=None, choices=["auto", "simt", "tc"], help="contraction path override")
    p.add_argument("--precision", default="fp32", choices=["fp32", "fast"],
                   help="fp32: the 1e-5 path (default); fast: single fp16 MMA + fp16 spectrum, the 2e-3 tensor-core path")
    p.add_argument("--eigen", default="device", choices=["device", "host"],
                   help="row a0 eigen-solve: on the device (rsvd_eigen_basis_device, no host round trip; R <= 128) or on the host")
    p.add_argument("--shard", default="templates", choices=["2d", "templates"],
                   help="rank grid: templates only (north_star: templates sharded over the GPUs, default) or "
                        "image x template shards (dist.grid_shape)")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            ident = str(self.dev)
            try:
                uuid = str(torch.cuda.get_device_properties(self.dev).uuid)
                ident = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            except Exception:
                pass
            self.proc = subprocess.Popen(["nvidia-smi", "-i", ident, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ helpers
def flops_per_pair(H: int, Q: int):
    """SURVEY.md §8(d) algorithmic FLOPs per pair: contraction 8HQ + FFT 5 Q log2 Q."""
    return 8 * H * Q, 5 * Q * math.log2(Q)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("BENCH_SHARED_GPU") == "1":
            # functional check of the multi-rank path on a one-GPU box: every rank on cuda:0, gloo
            # collectives staged through host memory.  Not a scaling measurement.
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        dist.barrier()


def _red_device():
    return "cpu" if dist.get_backend() == "gloo" else "cuda"


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_red_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_red_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------------ oracle (cpu baseline / reference arm)
def oracle_pairs_per_s(A, B, w, U, m, t, seconds: float, threads: int | None = None):
    """Time the fp64 oracle (O2 direct sum, as it stands) on sampled pairs; grow the sample until
    it takes ~`seconds`.  Returns (pairs/s, pairs timed, threads, seconds)."""
    from oracle import ref
    threads = threads or os.cpu_count() or 1
    n = 4
    while True:
        n = min(n, len(m))
        t0 = time.perf_counter()
        X = ref.landscape_rank(A, B, w, U, m[:n], t[:n], nthreads=threads)
        _ = ref.argmax_first(X.real)
        dt = time.perf_counter() - t0
        if dt >= seconds * 0.5 or n >= len(m):
            return n / dt, n, threads, dt
        n = int(min(len(m), max(2 * n, n * seconds / max(dt, 1e-3))))


# ------------------------------------------------------------------ our arm
DEFAULT_MODE = {"tiny": "per_pair", "small": "per_pair", "medium": "per_pair", "large": "per_image",
                "translations": "per_pair"}
TRAFFIC_KERNELS = {"fft_reduce": "fft2_reduce_kernel|fft_reduce_kernel", "contract": "contract_tc_kernel|contract_kernel"}


def measure_traffic(args, kernel_key: str, timeout_s: int = 600):
    """DRAM bytes per launch of one kernel family, from an ncu child run of this workload
    (`bench.py --traffic-probe`: one warm-up step + one step, no timing).  ncu runs with
    --cache-control none so the counts are the steady-state ones (a flushed L2 would charge every
    spectrum read to DRAM).  Returns a dict or {"error": ...}."""
    import csv
    import shutil
    import tempfile
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    log = tempfile.NamedTemporaryFile(suffix=".csv", delete=False).name
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--cache-control", "none", "-k", f"regex:{TRAFFIC_KERNELS[kernel_key]}",
           "-s", "8", "-c", "6", "--csv", "--log-file", log,
           sys.executable, os.path.abspath(__file__), "--traffic-probe", "--config", args.config,
           "--mode", args.mode]
    if args.H:
        cmd += ["--H", str(args.H)]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, env=env)
        if r.returncode != 0:
            return {"error": f"ncu exit {r.returncode}: {(r.stderr or r.stdout)[-200:]}"}
        rows = [row for row in csv.reader(open(log)) if len(row) > 10]
        hdr = rows[0]
        ci = {h: i for i, h in enumerate(hdr)}
        per = {}
        for row in rows[1:]:
            kid = row[ci["ID"]]
            per.setdefault(kid, {})[row[ci["Metric Name"]]] = (float(row[ci["Metric Value"]].replace(",", "")),
                                                                row[ci["Metric Unit"]])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                 "msecond": 1e-3, "nsecond": 1e-9}
        rd, wr, tm = [], [], []
        for m in per.values():
            v, u = m["dram__bytes_read.sum"]
            rd.append(v * scale.get(u, 1))
            v, u = m["dram__bytes_write.sum"]
            wr.append(v * scale.get(u, 1))
            v, u = m["gpu__time_duration.sum"]
            tm.append(v * scale.get(u, 1e-9))
        if not rd:
            return {"error": "no launches profiled"}
        return {"dram_read_per_launch": float(np.mean(rd)), "dram_write_per_launch": float(np.mean(wr)),
                "launches": len(rd), "ncu_launch_ms": float(np.mean(tm) * 1e3),
                "command": "ncu --metrics dram__bytes_{read,write}.sum --cache-control none (child run of this workload)"}
    except Exception as exc:  # noqa: BLE001
        return {"error": str(exc)[:200]}
    finally:
        try:
            os.unlink(log)
        except OSError:
            pass


def run_ours(args):
    from paper_2202_07235_b200 import api
    from paper_2202_07235_b200 import dist as pdist

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    cfg = CONFIGS[args.config]
    H = args.H or cfg["H"][0]
    Q, R = cfg["Q"], cfg["R"]
    args.mode = args.mode or DEFAULT_MODE[args.config]
    mode = args.mode
    chunk = api.kernel_chunk()
    T, M = cfg["T"], cfg["M"] * cfg.get("shifts", 1)
    # rank grid: GI image shards x GT template shards (dist.grid_shape); --shard templates = 1 x world
    GI, GT = pdist.grid_shape(world, M, T) if args.shard == "2d" else (1, world)
    ri, rt = pdist.grid_coords(rank, GI)
    t0, t1 = pdist.shard_range(T, GT, rt, chunk)
    b0, b1 = pdist.basis_range(T, world, rank, chunk, GI)
    tg0 = time.perf_counter()
    ds = make_dataset(args.config, device=dev, t_range=(t0, t1))
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - tg0
    assert ds.images.shape[0] == M, (ds.images.shape, M)
    m0, m1 = pdist.image_range(M, GI, ri)
    images = ds.images[m0:m1].contiguous() if GI > 1 else ds.images
    tmpl = ds.templates
    M_loc = images.shape[0]
    T_loc = tmpl.shape[0]
    w_dev = ds.w.contiguous()
    if args.path:
        api.set_path({"simt": api.PATH_SIMT, "tc": api.PATH_TC, "auto": api.PATH_AUTO}[args.path])
    api.set_precision(api.PREC_FAST if args.precision == "fast" else api.PREC_FP32)
    path = api.path_for(Q, H)
    fast = args.precision == "fast" and path == api.PATH_TC
    tb = torch.empty(max(api.block_bytes(T_loc, Q, H, api.SIDE_TEMPLATE), 16) // 4, dtype=torch.float32, device=dev)
    # landscape mode: the M x T x Q landscape is streamed to HBM in image blocks through one tile buffer
    # (each block's rows compressed on their own: the block layout is per call)
    if mode == "landscape":
        per_img = max(T_loc, 1) * Q * 4
        lblk = max(128, int(args.landscape_gb * 1e9 // per_img) // 128 * 128)
        lblk = min(lblk, M_loc)
        blocks = [(a, min(a + lblk, M_loc)) for a in range(0, M_loc, lblk)]
        Xbuf = torch.empty((lblk, T_loc, Q), dtype=torch.float32, device=dev)
    else:
        blocks = [(0, M_loc)]
        Xbuf = None
    ibs = [torch.empty(max(api.block_bytes(e - a, Q, H, api.SIDE_IMAGE), 16) // 4, dtype=torch.float32, device=dev)
           for a, e in blocks]
    wbytes = args.work_mb * (1 << 20) if args.work_mb else api.align_workspace_bytes(blocks[0][1] - blocks[0][0], T_loc, Q, H)
    work = torch.empty(wbytes // 4, dtype=torch.float32, device=dev)
    keys = torch.zeros(M, dtype=torch.int64, device=dev)
    if mode == "per_pair":
        best_val = torch.empty((M_loc, T_loc), dtype=torch.float32, device=dev)
        best_k = torch.empty((M_loc, T_loc), dtype=torch.int32, device=dev)
    U_dev = torch.zeros((R, H), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    G_ctf = args.ctf_groups if mode == "per_image" else 0
    if G_ctf:
        # row f3 input model: images of group g carry the toy CTF c_g (applied once, outside the timed
        # region -- it is the data, not the method); group g = images [gb[g], gb[g+1])
        from synth import toy_ctf
        kk = ds.k.cpu().numpy()
        ctfs = np.stack([toy_ctf(kk, 0.01 + 0.01 * g) for g in range(G_ctf)])
        gb = [(M_loc * g // G_ctf) // 128 * 128 for g in range(G_ctf)] + [M_loc]
        images = images.clone()
        for g in range(G_ctf):
            images[gb[g]:gb[g + 1]] *= torch.tensor(ctfs[g], dtype=images.dtype, device=dev)[None, :, None]
        ibs_g = [torch.empty(max(api.block_bytes(gb[g + 1] - gb[g], Q, H, api.SIDE_IMAGE), 16) // 4,
                             dtype=torch.float32, device=dev) for g in range(G_ctf)]
        tbs_g = [torch.empty(max(api.block_bytes(T_loc, Q, H, api.SIDE_TEMPLATE), 16) // 4, dtype=torch.float32,
                             device=dev) for g in range(G_ctf)]

    # NVTX ranges per SURVEY.md section 8 row (visible in nsys / ncu --nvtx timelines): one range per phase
    nvtx_next = {"start": "a0 basis", "basis": "a1 compress", "compress": "a2-a4 align", "align": "combine"}

    def nvtx_mark(name):
        if name != "start":
            torch.cuda.nvtx.range_pop()
        if name in nvtx_next:
            torch.cuda.nvtx.range_push(nvtx_next[name])

    def step_grouped(imgs, tmps, marks=None):
        def mark(name):
            nvtx_mark(name)
            if marks is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks.append((name, e))
        mark("start")
        C = pdist.kernel_from_shards(tmps[b0 - t0:b1 - t0], T, w_dev, GI=GI).cpu().numpy()      # one kernel pass
        bases = [api.eigen_basis_ctf(C, ctfs[g], H) for g in range(G_ctf)]
        mark("basis")
        groups = []
        for g, (Ug, Utg, _) in enumerate(bases):
            a, e = gb[g], gb[g + 1]
            api.compress(imgs[a:e], w_dev, torch.as_tensor(Ug, device=dev), api.SIDE_IMAGE, out=ibs_g[g])
            api.compress(tmps, w_dev, torch.as_tensor(Utg, device=dev), api.SIDE_TEMPLATE, out=tbs_g[g])
            groups.append(dict(img_blocks=ibs_g[g], M=e - a, tmpl_blocks=tbs_g[g], T=T_loc, t_offset=t0,
                               best_key=keys[m0 + a:m0 + e]))
        mark("compress")
        api.winners_reset(keys)
        api.align_argmax_grouped(groups, Q, H, api.PER_IMAGE, work)
        mark("align")
        out = pdist.combine_keys(keys, Q)
        mark("combine")
        return out, bases[0][0]

    dev_eigen = args.eigen == "device" and R <= 128 and R * H <= 8192
    eig_infos = []

    def step(imgs, tmps, marks=None):
        if G_ctf:
            return step_grouped(imgs, tmps, marks)

        def mark(name):
            nvtx_mark(name)
            if marks is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks.append((name, e))
        mark("start")
        if dev_eigen:                                                              # a0, no host round trip
            U, _, info = pdist.basis_from_shards_device(tmps[b0 - t0:b1 - t0], T, w_dev, H, GI=GI)
            U_dev.copy_(U)
            eig_infos.append(info)
        else:
            U, lam = pdist.basis_from_shards(tmps[b0 - t0:b1 - t0], T, w_dev, H, GI=GI)   # a0 (syncs for the host solve)
            U_dev.copy_(torch.from_numpy(U), non_blocking=False)
        mark("basis")
        for (a, e), ib in zip(blocks, ibs):                                        # a1
            if e > a:
                api.compress(imgs[a:e] if len(blocks) > 1 else imgs, w_dev, U_dev, api.SIDE_IMAGE, out=ib)
        if T_loc:
            api.compress(tmps, w_dev, U_dev, api.SIDE_TEMPLATE, out=tb)
        mark("compress")
        out = None
        if mode == "per_image":                                                    # a2-a4
            api.winners_reset(keys)
            if T_loc and M_loc:
                api.align_argmax(ibs[0], M_loc, tb, T_loc, Q, H, api.PER_IMAGE, work, best_key=keys[m0:m1], t_offset=t0)
            mark("align")
            out = pdist.combine_keys(keys, Q)                                      # all-gather + combine
        elif mode == "per_pair":
            if T_loc and M_loc:
                api.align_argmax(ibs[0], M_loc, tb, T_loc, Q, H, api.PER_PAIR, work, best_val=best_val, best_k=best_k)
            mark("align")
        else:
            for (a, e), ib in zip(blocks, ibs):
                if e > a and T_loc:
                    api.align_landscape(ib, e - a, tb, T_loc, Q, H, work, X=Xbuf, ld_m=T_loc * Q, ld_t=Q)
            mark("align")
        mark("combine")
        return out, U

    if args.traffic_probe:                      # child of measure_traffic: run under ncu, print nothing
        step(images, tmpl)
        step(images, tmpl)
        torch.cuda.synchronize()
        return

    for _ in range(args.warmup):
        step(images, tmpl)
    torch.cuda.synchronize()
    barrier(world)
    # measured FP32 peak of this GPU (Pi_fp32 of SURVEY.md 8(d)), outside the timed region
    fp32_meas = {k: api.probe_fp32(k) for k in ("ffma2", "ffma")}
    fp64_meas = {"dfma": api.probe_fp32("dfma", 100000),          # fp64 peaks for row a0 (kernel partials)
                 "dmma8": api.probe_fp32("dmma8", 20000)}

    clocks = Clocks(local)
    clocks.start()
    api.timing_read()
    api.timing_enable(False)
    n0 = api.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    # headline region: K steps, events only at step boundaries (the align path chains its contraction /
    # FFT launches with programmatic dependent launch; a per-launch event would serialise them)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    step_marks = []
    last_U, out = None, None
    for _ in range(args.steps):
        mk = []
        out, last_U = step(images, tmpl, marks=mk)
        step_marks.append(mk)
    end.record(stream)
    torch.cuda.synchronize()
    elapsed_ms = start.elapsed_time(end)
    barrier(world)
    launches = api.launch_count() - n0
    clk = clocks.stop()
    per_step = [mk[0][1].elapsed_time(nxt[0][1]) for mk, nxt in zip(step_marks[:-1], step_marks[1:])]
    per_step.append(step_marks[-1][0][1].elapsed_time(end))
    names = [n for n, _ in step_marks[-1]]
    phase = {b: step_marks[-1][i][1].elapsed_time(step_marks[-1][i + 1][1]) for i, b in enumerate(names[1:])}
    # kernel-duration region: the same K steps again with a CUDA event pair on the launching stream
    # around every library launch (rsvd_timing_*), for the per-kernel roofline
    timing_steps = 0
    if not args.no_kernel_timing:
        api.timing_enable(True)
        for _ in range(args.steps):
            step(images, tmpl)
        torch.cuda.synchronize()
        api.timing_enable(False)
        timing_steps = args.steps
    ktime = api.timing_read()
    if eig_infos:                                 # device eigen-solves all passed their residual test
        bad = int(torch.stack(eig_infos).sum().item())
        if bad:
            raise RuntimeError(f"device eigen-solver failed its residual test in {bad} steps (rerun with --eigen host)")
        eig_infos.clear()
    if torch.is_tensor(last_U):
        last_U = last_U.cpu().numpy()
    ms_step = max_over_ranks(elapsed_ms / args.steps, world)
    ms_median = max_over_ranks(float(np.median(per_step)), world)
    launches_all = int(sum_over_ranks(launches, world))
    pairs = M * T
    value = pairs / (ms_step / 1e3)

    # dominant-kernel roofline (the kernel with the larger measured share of the step)
    pk, pk_kind = peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_nom = sm_count * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12      # TFLOP/s at max clock
    fp32_peak = fp32_meas["ffma2"]                                                   # measured (FFMA2 probe)
    f16_peak = pk.get("bf16_tflops", 1656.1)                                        # fp16 dense = bf16 dense rate
    f_contr, f_fft = flops_per_pair(H, Q)
    f_fft_strict = f_fft / 2.0                                                       # G18: c2r costs 2.5 Q log2 Q
    c_ms, c_n = ktime["contract"]
    f_ms, f_n = ktime["fft_reduce"]
    n_pairs_timed = max(timing_steps, 1) * M_loc * T_loc
    if c_ms >= f_ms:
        achieved = n_pairs_timed * f_contr / (c_ms / 1e3) / 1e12 if c_ms > 0 else None
        if path == api.PATH_TC and fast:
            peak, bound = f16_peak, "tensor"
            kname = "contract_tc_kernel (Step 2, tcgen05 kind::f16 on CTA pairs, single fp16 MMA: the 2e-3 path)"
            note = f"fp16 dense = measured bf16 {f16_peak:.1f} TF/s ({pk_kind}, same rate), one MMA per MAC"
        elif path == api.PATH_TC:
            peak, bound = f16_peak / 3.0, "tensor"
            kname = "contract_tc_kernel (Step 2, tcgen05 kind::f16 on CTA pairs, fp16 hi/lo split x3)"
            note = (f"fp16 dense = measured bf16 {f16_peak:.1f} TF/s ({pk_kind}, same rate); the hi/lo split "
                    f"executes 3 MMAs per algorithmic MAC -> peak/3 for algorithmic 8HQ flops per pair")
        else:
            peak, bound = fp32_peak, "alu"
            kname = "contract_kernel (Step 2, FP32 SIMT)"
            note = f"measured FFMA2 peak {fp32_peak:.1f} TF/s (rsvd_probe_fp32); nominal {fp32_nom:.1f} at max clock"
        k_ms, k_n, fpp, tkey = c_ms, c_n, f_contr, "contract"
        strict = None
    else:
        achieved = n_pairs_timed * f_fft / (f_ms / 1e3) / 1e12 if f_ms > 0 else None
        peak, bound = fp32_peak, "alu"
        kname = "fft2_reduce_kernel (Steps 3-4, FP32 SIMT)"
        note = (f"peak = measured sustained FFMA2 rate {fp32_peak:.2f} TF/s of this GPU (rsvd_probe_fp32, scalar "
                f"FFMA {fp32_meas['ffma']:.1f}); nominal {fp32_nom:.1f} TF/s = {sm_count} SMs x 128 lanes x 2 x "
                f"{pk.get('sm_max_mhz', 1965.0):.0f} MHz; algorithmic 5 Q log2 Q flops per pair")
        k_ms, k_n, fpp, tkey = f_ms, f_n, f_fft, "fft_reduce"
        strict = round(n_pairs_timed * f_fft_strict / (f_ms / 1e3) / 1e12 / fp32_peak, 4) if f_ms > 0 else None
    traffic = None
    if rank == 0 and world == 1 and args.traffic == "auto" and k_n > 0:
        traffic = measure_traffic(args, tkey)
    roof = {"bound": bound, "kernel": kname,
            "achieved": round(achieved, 3) if achieved else None, "peak": round(peak, 2),
            "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if achieved else None,
            "frac_nominal_peak": round(achieved / fp32_nom, 4) if (achieved and bound == "alu") else None,
            "frac_strict_c2r": strict,
            "traffic": (traffic["dram_read_per_launch"] + traffic["dram_write_per_launch"])
            if traffic and "dram_read_per_launch" in traffic else None,
            "traffic_detail": traffic, "peak_note": note,
            "avg_launch_ms": round(k_ms / max(k_n, 1), 4), "launches": k_n,
            "timing": f"CUDA events around every launch on its stream over a second {timing_steps}-step region",
            "algorithmic_flops_per_pair": fpp, "contraction_path": "tc" if path == api.PATH_TC else "simt"}
    # The contraction against the L2 it saturates: per launch it writes the chunk's spectrum
    # (pairs x Q/2 slots x 8 B) and reads the fp16 hi/lo operand rows ((Q/2 + 1) x KB x 2 B per pair for
    # 128 x 256 pair tiles); bound t = writes / BW_w + reads / BW_r with the L2 write / read bandwidths
    # measured by tools/l2_bw_probe.cu on this pool's B200s (profiles/r01s3_l2_bw_probe.txt).
    contr_l2 = None
    if path == api.PATH_TC and c_n > 0 and c_ms > 0:
        L2_W, L2_R = 7300.0, 15500.0                       # GB/s
        pairs_launch = n_pairs_timed / c_n
        kb = (H + 7) // 8
        w_b = pairs_launch * (Q // 2) * 8
        r_b = pairs_launch * (Q // 2 + 1) * kb * 2
        t_launch = c_ms / c_n / 1e3
        t_min = w_b / (L2_W * 1e9) + r_b / (L2_R * 1e9)
        contr_l2 = {"bound": "l2", "kernel": "contract_tc_kernel", "achieved": round((w_b + r_b) / t_launch / 1e9, 1),
                    "peak": round((w_b + r_b) / t_min / 1e9, 1), "unit": "GB/s", "frac": round(t_min / t_launch, 4),
                    "bytes_per_launch": {"spectrum_write": int(w_b), "operand_read": int(r_b)},
                    "peak_note": f"time-weighted L2 ceiling: write {L2_W:.0f} / read {L2_R:.0f} GB/s measured by "
                                 "tools/l2_bw_probe.cu (profiles/r01s3_l2_bw_probe.txt)"}
    pi_c = (f16_peak if fast else f16_peak / 3.0) if path == api.PATH_TC else fp32_peak
    land_bytes = float(M) * T * Q * 4 if mode == "landscape" else 0.0
    hbm = pk.get("hbm_gbs", 6539.9) * 1e9
    t_flop = pairs * (f_contr / pi_c + f_fft / fp32_peak) / 1e12 / world
    t_roof = max(t_flop, land_bytes / hbm / world)
    ts = max(timing_steps, 1)
    step_roof = {"t_roof_ms": round(t_roof * 1e3, 3), "frac": round(t_roof * 1e3 / ms_step, 4),
                 "frac_align_only": round(t_roof * 1e3 / max(phase.get("align", 0.0), 1e-9), 4),
                 "definition": ("max(M*T*(8HQ/Pi_contr + 5Q log2 Q/Pi_fp32), landscape bytes/BW_HBM) / G vs the "
                                "measured step, Pi_contr = " + (("fp16 dense (1 MMA per MAC)" if fast else
                                                                  "fp16 dense/3 (3 MMAs per MAC)")
                                                                 if path == api.PATH_TC else "Pi_fp32")
                                + ", Pi_fp32 = measured FFMA2 peak (SURVEY.md 8(d))"),
                 "kernel_ms_per_step": {k: round(v[0] / ts, 3) for k, v in ktime.items()}}
    # row a0 against the measured fp64 tensor-core peak: the kernel partials run the Gram of each 64 x 64
    # tile of the lower triangle as mma.sync m8n8k4 .f64 (2 real K per sample, 4 flops per entry and
    # sample); diagonal tiles skip the warp block above the diagonal and the m8n8 blocks a < b of the two
    # diagonal warp blocks (36 of 64 blocks executed).  RSVD_KP_SIMT=1 selects the DFMA tile (20 of 32).
    kp_ms = ktime["kernel_partials"][0] / ts
    if kp_ms > 0 and R % 64 == 0:
        nt = R // 64
        simt = os.environ.get("RSVD_KP_SIMT", "0") == "1"
        entries = (nt * (nt - 1) // 2) * 4096 + nt * 4096 * (20 if simt else 36) // (32 if simt else 64)
        kp_tf = 2.0 * 2 * entries * (b1 - b0) * Q / (kp_ms / 1e3) / 1e12       # the rank's basis sub-shard
        kp_alg = 2.0 * 2 * (R * (R + 1) // 2) * (b1 - b0) * Q / (kp_ms / 1e3) / 1e12
        kp_peak = fp64_meas["dfma"] if simt else fp64_meas["dmma8"]
        step_roof["kernel_partials_fp64"] = {
            "bound": "fp64", "achieved": round(kp_tf, 2), "peak": round(kp_peak, 2), "unit": "TFLOP/s",
            "frac": round(kp_tf / kp_peak, 4), "achieved_algorithmic": round(kp_alg, 2),
            "frac_algorithmic": round(kp_alg / kp_peak, 4),
            "peak_note": ("measured sustained " + ("DFMA rate (rsvd_probe_fp32 kind 3)" if simt else
                          "fp64 tensor-core rate (rsvd_probe_fp32 kind 4, mma.sync m8n8k4 .f64)")
                          + "; achieved = executed flops of the tile schedule, achieved_algorithmic = the "
                          "lower triangle R(R+1)/2 only")}

    # e2e: host (pinned) rings -> device -> step -> winners back, through the public API (per-image mode)
    e2e = None
    if not args.no_e2e and mode == "per_image" and not G_ctf:
        try:
            h_img = torch.empty(images.shape, dtype=images.dtype, pin_memory=True)
            h_tmp = torch.empty(tmpl.shape, dtype=tmpl.dtype, pin_memory=True)
            h_img.copy_(images)
            h_tmp.copy_(tmpl)
            d_img = torch.empty_like(images)
            d_tmp = torch.empty_like(tmpl)
            h_out = [torch.empty(M, dtype=x, pin_memory=True) for x in (torch.float32, torch.int32, torch.int32)]
            # one untimed pass: allocator growth for the per-block buffers, first-touch of the pinned pages
            e2e_kw = dict(work=work, img_block=args.e2e_img_block, M_total=M, m_offset=m0,
                          basis_sub=(b0 - t0, b1 - t0), GI=GI)
            pdist.align_from_host(h_img, h_tmp, T, t0, w_dev, H, d_img, d_tmp, **e2e_kw)
            torch.cuda.synchronize()
            barrier(world)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.e2e_steps):
                # public streamed path: copies of template / image blocks overlap partials, compress, align
                (kk, val, tt, k), _ = pdist.align_from_host(h_img, h_tmp, T, t0, w_dev, H, d_img, d_tmp, **e2e_kw)
                for h, d in zip(h_out, (val, tt, k)):
                    h.copy_(d, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, world)
            # the streamed result must equal the device-resident step's winners
            same = bool(torch.equal(kk, out[0]))
            h2d = int(sum_over_ranks(h_img.numel() * 8 + h_tmp.numel() * 8, world))
            d2h = int(sum_over_ranks(M * 12, world))
            e2e = {"value": pairs / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": round(e2e_ms, 3),
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                   "matches_device_step": same,
                   "path": "pinned host rings -> paper_2202_07235_b200.dist.align_from_host (H2D of template / "
                           "image blocks on a copy stream overlapped with partials, compress and per-block "
                           "align) -> combine -> winners (val,t,k) to pinned host"}
            del h_img, h_tmp, d_img, d_tmp
        except Exception as exc:  # host memory etc.
            e2e = {"value": None, "unit": UNIT, "error": str(exc)[:200]}
    elif G_ctf:
        e2e = {"value": None, "unit": UNIT, "reason": "end-to-end line is measured for the plain per-image path"}
    elif mode != "per_image":
        e2e = {"value": None, "unit": UNIT, "reason": f"end-to-end line is measured for the per-image mode only "
                                                      f"({mode} outputs are M x T{' x Q' if mode == 'landscape' else ''})"}

    # cpu baseline: the oracle as it stands, rank 0 at N = 1 only, on all host cores and on one core
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not G_ctf:
        m, t = sample_pairs(args.config, M, T, 2048, 0)
        rows_m, inv_m = np.unique(m, return_inverse=True)
        rows_t, inv_t = np.unique(t, return_inverse=True)
        A = images[torch.as_tensor(rows_m, device=dev)].cpu().numpy()
        B = tmpl[torch.as_tensor(rows_t, device=dev)].cpu().numpy()
        wn = ds.w.cpu().numpy()
        rate, n, thr, secs = oracle_pairs_per_s(A, B, wn, last_U, inv_m, inv_t, args.cpu_seconds)
        rate1, n1, _, secs1 = oracle_pairs_per_s(A, B, wn, last_U, inv_m, inv_t, max(2.0, args.cpu_seconds / 4), threads=1)
        cpu = {"value": rate, "unit": UNIT, "cores": thr, "kind": "oracle",
               "sample": f"{n} seeded random (m,t) pairs of the {args.config} workload, O2 rank-{H} fp64 direct "
                         f"sum (oracle/direct.c, OpenMP) + argmax, library U; {secs:.1f} s",
               "one_core": {"value": rate1, "unit": UNIT, "cores": 1, "sample": f"{n1} pairs, {secs1:.1f} s"}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "ms_per_step_median": round(ms_median, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f16 MMA / f16 spectrum, f32 transform (2e-3 path)" if fast else "f32", "data": "synthetic",
            "config": {"workload": args.config + (f"+ctf{G_ctf}" if G_ctf else ""), "M": M, "T": T, "R": R, "Q": Q,
                       "H": H, "mode": mode, "ctf_groups": G_ctf or None,
                       "precision": "fast (<= 2e-3 gate)" if fast else "fp32 (<= 1e-5 gate)",
                       "workspace_mb": round(wbytes / 2**20, 1),
                       "parallelism": f"{GI} image x {GT} template shards on {world} GPU(s)"
                                      + (" (NCCL all-gather of winners)" if mode == "per_image" else ""),
                       "l2": "inputs larger than L2 (rings %.1f GB per step)" % ((images.numel() + T_loc * R * Q) * 8 / 1e9),
                       "seed": 220207235},
            "roofline": roof, "contraction_l2": contr_l2, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clk, "fp32_peak_measured_tflops": {k: round(v, 2) for k, v in fp32_meas.items()},
            "fp64_peak_measured_tflops": {k: round(v, 2) for k, v in fp64_meas.items()},
            "gpu_launches": launches_all, "phases_ms_last_step": {k: round(v, 3) for k, v in phase.items()},
            "gen_seconds": round(gen_s, 1),
            "a0_eigen": ("device (rsvd_eigen_basis_device)" if dev_eigen else "host (rsvd_eigen_basis)")
                        if not G_ctf else "host (rsvd_eigen_basis_ctf per group)",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    cfg = CONFIGS[args.config]
    H = args.H or cfg["H"][0]
    Q, R, T = cfg["Q"], cfg["R"], cfg["T"]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    # inputs: the same seeded workload (harness generator); oracle basis from a template sample
    ds = make_dataset(args.config, device=dev)
    M = ds.images.shape[0]
    w = ds.w.cpu().numpy()
    nb = min(T, 512)
    tb = ds.templates[:nb].cpu().numpy()
    U, lam = ref.basis(ref.kernel_C(tb, w), H)
    m, t = sample_pairs(args.config, M, T, 4096, 0)
    rows_m, inv_m = np.unique(m, return_inverse=True)
    rows_t, inv_t = np.unique(t, return_inverse=True)
    A = ds.images[torch.as_tensor(rows_m, device=dev)].cpu().numpy()
    B = ds.templates[torch.as_tensor(rows_t, device=dev)].cpu().numpy()
    del ds
    # size one step to ~cpu_seconds/2 of oracle work
    rate, n, thr, secs = oracle_pairs_per_s(A, B, w, U, inv_m, inv_t, max(2.0, args.cpu_seconds / 2))
    n_step = max(1, int(rate * max(2.0, args.cpu_seconds / 2)))
    n_step = min(n_step, len(inv_m))

    def one_step():
        X = ref.landscape_rank(A, B, w, U, inv_m[:n_step], inv_t[:n_step], nthreads=thr)
        return ref.argmax_first(X.real)

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    dt = (time.perf_counter() - t0) / args.steps
    value = n_step / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.config, "M": M, "T": T, "R": R, "Q": Q, "H": H,
                   "mode": args.mode or DEFAULT_MODE[args.config],
                   "parallelism": "host cores (OpenMP over pairs)", "seed": 220207235},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle",
                         "sample": f"{n_step} seeded random (m,t) pairs of the workload per step: O2 rank-{H} fp64 "
                                   f"direct-sum landscape over all {Q} angles + argmax per pair (the per-image "
                                   f"winner is the max of these), oracle basis (eigh of C from {nb} templates)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without a torchrun environment: re-launch this script as N ranks
    (one process per GPU) through torch.distributed.run on 127.0.0.1 and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ, BENCH_SPAWNED="1"))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
