"""Torch-facing wrappers of the C ABI (include/rsvd.h): the names mirror the library's entry
points and every function only marshals arguments.  Tensors are CUDA, contiguous; complex rings
are torch.complex64 [n, R, Q]; weights w are float64 [R]; packed per-image keys are int64 tensors
holding the uint64 bit patterns.

The `Aligner` class strings the entry points into the full hot path (rows a0-a4 of SURVEY.md §8):
basis from the templates -> compress images and templates -> align -> winners."""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import PER_IMAGE, PER_PAIR, SIDE_IMAGE, SIDE_TEMPLATE, RsvdError, check, ptr, require_cuda, stream_handle

__all__ = ["block_bytes", "path_for", "set_path", "set_precision", "precision", "PREC_FP32", "PREC_FAST", "PATH_AUTO", "PATH_SIMT", "PATH_TC", "kernel_chunk", "kernel_partials_bytes", "align_workspace_bytes",
           "align_min_workspace_bytes", "kernel_partials", "kernel_reduce", "eigen_basis", "eigen_basis_ctf", "ctf_group_bases", "align_argmax_grouped", "build_basis",
           "build_basis_translated", "compress", "compress_translated", "blocks_unpack", "align_argmax", "align_landscape", "align_argmax_fine",
           "align_landscape_fine", "winners_reset",
           "winners_unpack", "combine_winners", "launch_count", "timing_enable", "timing_read", "Aligner", "RsvdError", "PER_PAIR", "PER_IMAGE",
           "SIDE_IMAGE", "SIDE_TEMPLATE", "vol_ncoef", "vol_grid", "vol_kernels", "vol_bases", "vol_compress",
           "vol_wigner_table", "vol_degrees", "vol_align", "vol_best", "VolumeAligner"]


# ------------------------------------------------------------------ sizes
def block_bytes(rows: int, Q: int, H: int, side: int = SIDE_IMAGE) -> int:
    return int(_lib.lib().rsvd_block_bytes(rows, Q, H, side))


PATH_AUTO, PATH_SIMT, PATH_TC = 0, 1, 2


def path_for(Q: int, H: int) -> int:
    """1 = FP32 SIMT contraction, 2 = tcgen05 contraction, fp16 hi/lo split x3 MMAs (include/rsvd.h)."""
    return int(_lib.lib().rsvd_path_for(Q, H))


PREC_FP32, PREC_FAST = 0, 1


def set_precision(precision: int):
    """rsvd_set_precision: PREC_FP32 (default; 1e-5 gate) or PREC_FAST (single fp16 MMA + fp16 spectrum;
    2e-3 gate) for the tensor-core align path."""
    _lib.lib().rsvd_set_precision(int(precision))


def precision() -> int:
    return int(_lib.lib().rsvd_precision())


def set_compress_mma(mode: int):
    """rsvd_set_compress_mma: 1 auto (default), 2 force the tensor-core projection, 0 force the FFMA2 one."""
    _lib.lib().rsvd_set_compress_mma(int(mode))


def compress_mma_mode() -> int:
    return int(_lib.lib().rsvd_compress_mma_mode())


def set_path(path: int):
    _lib.lib().rsvd_set_path(int(path))


def kernel_chunk() -> int:
    return int(_lib.lib().rsvd_kernel_chunk())


def kernel_partials_bytes(T: int, R: int) -> int:
    return int(_lib.lib().rsvd_kernel_partials_bytes(T, R))


def align_workspace_bytes(M: int, T: int, Q: int, H: int) -> int:
    return int(_lib.lib().rsvd_align_workspace_bytes(M, T, Q, H))


def align_min_workspace_bytes(Q: int) -> int:
    return int(_lib.lib().rsvd_align_min_workspace_bytes(Q))


# ------------------------------------------------------------------ row a0
def kernel_partials(templates: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    require_cuda(templates)
    T, R, Q = templates.shape
    nch = (T + kernel_chunk() - 1) // kernel_chunk()
    if out is None:
        out = torch.empty((nch, R, R), dtype=torch.float64, device=templates.device)
    check(_lib.lib().rsvd_kernel_partials(ptr(templates), T, R, Q, ptr(out), stream_handle(stream)))
    return out


def kernel_reduce(partials: torch.Tensor, T_total: int, Q: int, w: torch.Tensor, out=None, stream=None):
    require_cuda(partials, w)
    nch, R, _ = partials.shape
    if out is None:
        out = torch.empty((R, R), dtype=torch.float64, device=partials.device)
    check(_lib.lib().rsvd_kernel_reduce(ptr(partials), nch, R, T_total, Q, ptr(w), ptr(out),
                                        stream_handle(stream)))
    return out


def eigen_basis(C: np.ndarray, H: int):
    """Host eigen-solver of the library.  Returns (U [R, H], lambda [R]) as float64 numpy."""
    C = np.ascontiguousarray(C, dtype=np.float64)
    R = C.shape[0]
    U = np.zeros((R, H), dtype=np.float64)
    lam = np.zeros(R, dtype=np.float64)
    check(_lib.lib().rsvd_eigen_basis(ptr(C), R, H, ptr(U), ptr(lam)))
    return U, lam


def eigen_basis_device(C: torch.Tensor, H: int, stream=None):
    """rsvd_eigen_basis_device: the eigenbasis on the device (no host round trip).  C: device fp64
    [R, R].  Returns (U [R, H], lambda [R], info [1] int32) as device tensors, enqueued on the stream;
    info != 0 (read it after synchronising) means U failed the residual test -- use eigen_basis(C)."""
    require_cuda(C)
    if C.dtype != torch.float64 or C.dim() != 2 or C.shape[0] != C.shape[1]:
        raise ValueError("eigen_basis_device: C must be a square float64 device tensor")
    C = C.contiguous()
    R = C.shape[0]
    U = torch.empty((R, H), dtype=torch.float64, device=C.device)
    lam = torch.empty(R, dtype=torch.float64, device=C.device)
    info = torch.zeros(1, dtype=torch.int32, device=C.device)
    check(_lib.lib().rsvd_eigen_basis_device(ptr(C), R, H, ptr(U), ptr(lam), ptr(info), stream_handle(stream)))
    return U, lam, info


def eigen_basis_ctf(C: np.ndarray, ctf, H: int):
    """rsvd_eigen_basis_ctf (row f3): (U, U_tmpl, lambda) of one CTF group from the raw kernel C."""
    C = np.ascontiguousarray(C, dtype=np.float64)
    R = C.shape[0]
    ctf = np.ascontiguousarray(np.asarray(ctf), dtype=np.float64)
    U = np.zeros((R, H), dtype=np.float64)
    Ut = np.zeros((R, H), dtype=np.float64)
    lam = np.zeros(R, dtype=np.float64)
    check(_lib.lib().rsvd_eigen_basis_ctf(ptr(C), R, ptr(ctf), H, ptr(U), ptr(Ut), ptr(lam)))
    return U, Ut, lam


def ctf_group_bases(templates: torch.Tensor, w: torch.Tensor, ctfs, H: int):
    """Row f3: one kernel-partials pass over the raw templates, then per CTF group g (ctfs[g] = c_g(k_r),
    [G, R]) the group basis U_g (for its images) and U_tmpl_g = diag(c_g) U_g (compresses the raw
    templates into the group's CTF-corrected targets).  Returns [(U_g, U_tmpl_g, lambda_g)]."""
    require_cuda(templates, w)
    T, R, Q = templates.shape
    C = kernel_reduce(kernel_partials(templates), T, Q, w).cpu().numpy()
    return [eigen_basis_ctf(C, c, H) for c in np.asarray(ctfs, dtype=np.float64).reshape(-1, R)]


def build_basis(templates: torch.Tensor, w, H: int, stream=None):
    """rsvd_build_basis: (U [R, H], lambda [R]) float64 numpy, computed from all templates."""
    require_cuda(templates)
    T, R, Q = templates.shape
    w = np.ascontiguousarray(np.asarray(w if not torch.is_tensor(w) else w.cpu().numpy()), dtype=np.float64)
    U = np.zeros((R, H), dtype=np.float64)
    lam = np.zeros(R, dtype=np.float64)
    check(_lib.lib().rsvd_build_basis(ptr(templates), T, R, Q, ptr(w), H, ptr(U), ptr(lam),
                                      stream_handle(stream)))
    return U, lam


def build_basis_translated(templates: torch.Tensor, w, k, shifts, H: int, stream=None):
    """rsvd_build_basis_translated: basis of the kernel averaged over the S translated copies of
    every template (row f2).  w, k: [R] radial weights / wavenumbers; shifts: [S, 2] (dx, dy)."""
    require_cuda(templates)
    T, R, Q = templates.shape
    as64 = lambda x: np.ascontiguousarray(np.asarray(x.cpu() if torch.is_tensor(x) else x), dtype=np.float64)
    w, k, sh = as64(w), as64(k), as64(shifts).reshape(-1, 2)
    U = np.zeros((R, H), dtype=np.float64)
    lam = np.zeros(R, dtype=np.float64)
    check(_lib.lib().rsvd_build_basis_translated(ptr(templates), T, R, Q, ptr(w), ptr(k), ptr(sh), sh.shape[0], H,
                                                 ptr(U), ptr(lam), stream_handle(stream)))
    return U, lam


def kernel_translated_sh(Bsh: torch.Tensor, k: torch.Tensor, w: torch.Tensor, sigma: float, stream=None) -> torch.Tensor:
    """rsvd_kernel_translated_sh: the closed-form translation- and view-averaged kernel (PAPER.md:1156-1166,
    row f2) from a volume's spherical-harmonic coefficients Bsh [R, (L+1)^2] complex128 (device);
    k, w: device fp64 [R].  Returns C [R, R] fp64 (device); U from eigen_basis(C)."""
    require_cuda(Bsh, k, w)
    R, nlm = Bsh.shape
    L = int(round(nlm ** 0.5)) - 1
    if (L + 1) ** 2 != nlm or Bsh.dtype != torch.complex128:
        raise RsvdError(1, "Bsh must be complex128 [R, (L+1)^2]")
    C = torch.empty((R, R), dtype=torch.float64, device=Bsh.device)
    check(_lib.lib().rsvd_kernel_translated_sh(ptr(Bsh.contiguous()), R, L, ptr(k.contiguous()), ptr(w.contiguous()),
                                               float(sigma), ptr(C), stream_handle(stream)))
    return C


# ------------------------------------------------------------------ row a1
def compress(rings: torch.Tensor, w: torch.Tensor, U: torch.Tensor, side: int, out=None, stream=None):
    """rsvd_compress -> opaque block buffer (float32 tensor of block_bytes/4 elements)."""
    require_cuda(rings, w, U)
    n, R, Q = rings.shape
    H = U.shape[1]
    nb = block_bytes(n, Q, H, side)
    if out is None:
        out = torch.empty(nb // 4, dtype=torch.float32, device=rings.device)
    elif out.numel() * out.element_size() < nb:
        raise RsvdError(1, "block buffer too small")
    check(_lib.lib().rsvd_compress(ptr(rings), n, R, Q, ptr(w), ptr(U), H, side, ptr(out), stream_handle(stream)))
    return out


def compress_translated(rings: torch.Tensor, w: torch.Tensor, k: torch.Tensor, U: torch.Tensor,
                        shifts: torch.Tensor, side: int, out=None, stream=None):
    """rsvd_compress_translated: blocks of the S translated copies (row b*S + s) of every base row."""
    require_cuda(rings, w, k, U, shifts)
    n, R, Q = rings.shape
    H = U.shape[1]
    S = shifts.shape[0]
    nb = block_bytes(n * S, Q, H, side)
    if out is None:
        out = torch.empty((nb + 3) // 4, dtype=torch.float32, device=rings.device)
    elif out.numel() * out.element_size() < nb:
        raise RsvdError(1, "block buffer too small")
    check(_lib.lib().rsvd_compress_translated(ptr(rings), n, R, Q, ptr(w), ptr(k), ptr(U), H, ptr(shifts), S,
                                              side, ptr(out), stream_handle(stream)))
    return out


def blocks_unpack(blocks: torch.Tensor, n: int, Q: int, H: int, side: int, stream=None) -> torch.Tensor:
    require_cuda(blocks)
    out = torch.empty((n, Q, H), dtype=torch.complex64, device=blocks.device)
    check(_lib.lib().rsvd_blocks_unpack(ptr(blocks), n, Q, H, side, ptr(out), stream_handle(stream)))
    return out


# ------------------------------------------------------------------ rows a2-a4
def align_argmax(img_blocks, M: int, tmpl_blocks, T: int, Q: int, H: int, mode: int, work,
                 best_val=None, best_k=None, best_key=None, t_offset: int = 0, stream=None):
    require_cuda(img_blocks, tmpl_blocks, work)
    dev = img_blocks.device
    if mode == PER_PAIR:
        if best_val is None:
            best_val = torch.empty((M, T), dtype=torch.float32, device=dev)
        if best_k is None:
            best_k = torch.empty((M, T), dtype=torch.int32, device=dev)
    else:
        if best_key is None:
            best_key = torch.zeros(M, dtype=torch.int64, device=dev)
    check(_lib.lib().rsvd_align_argmax(ptr(img_blocks), M, ptr(tmpl_blocks), T, t_offset, Q, H, mode,
                                       ptr(work), work.numel() * work.element_size(), ptr(best_val),
                                       ptr(best_k), ptr(best_key), stream_handle(stream)))
    return (best_val, best_k) if mode == PER_PAIR else best_key


def align_argmax_grouped(groups, Q: int, H: int, mode: int, work, stream=None):
    """Row f3, rsvd_align_argmax_grouped: G independent CTF groups in one call.  groups: list of dicts
    with img_blocks, M, tmpl_blocks, T and optionally t_offset / best_val / best_k (PER_PAIR) /
    best_key (PER_IMAGE; reset by the caller).  Missing outputs are allocated; returns the list of
    (best_val, best_k) or best_key per group."""
    require_cuda(work)
    arr = (_lib.AlignGroup * max(len(groups), 1))()
    outs = []
    for i, g in enumerate(groups):
        require_cuda(g["img_blocks"], g["tmpl_blocks"])
        dev = g["img_blocks"].device
        M, T = int(g["M"]), int(g["T"])
        if mode == PER_PAIR:
            bv = g.get("best_val")
            bk = g.get("best_k")
            bv = torch.empty((M, T), dtype=torch.float32, device=dev) if bv is None else bv
            bk = torch.empty((M, T), dtype=torch.int32, device=dev) if bk is None else bk
            require_cuda(bv, bk)
            outs.append((bv, bk))
            key = None
        else:
            key = g.get("best_key")
            key = torch.zeros(M, dtype=torch.int64, device=dev) if key is None else key
            require_cuda(key)
            outs.append(key)
            bv = bk = None
        arr[i] = _lib.AlignGroup(ptr(g["img_blocks"]), M, ptr(g["tmpl_blocks"]), T, int(g.get("t_offset", 0)),
                                 ptr(bv), ptr(bk), ptr(key))
    check(_lib.lib().rsvd_align_argmax_grouped(ctypes.addressof(arr), len(groups), Q, H, mode, ptr(work),
                                               work.numel() * work.element_size(), stream_handle(stream)))
    return outs


def align_landscape(img_blocks, M: int, tmpl_blocks, T: int, Q: int, H: int, work, X=None,
                    ld_m: int | None = None, ld_t: int | None = None, stream=None):
    require_cuda(img_blocks, tmpl_blocks, work)
    if X is None:
        X = torch.empty((M, T, Q), dtype=torch.float32, device=img_blocks.device)
        ld_m, ld_t = T * Q, Q
    check(_lib.lib().rsvd_align_landscape(ptr(img_blocks), M, ptr(tmpl_blocks), T, Q, H, ptr(work),
                                          work.numel() * work.element_size(), ptr(X), ld_m, ld_t,
                                          stream_handle(stream)))
    return X


def align_argmax_fine(img_blocks, M: int, tmpl_blocks, T: int, Q: int, H: int, Q_out: int, mode: int, work,
                      best_val=None, best_k=None, best_key=None, best_gamma=None, refine: bool = True,
                      t_offset: int = 0, stream=None):
    """rsvd_align_argmax_fine: argmax on the zero-padded grid gamma_k = 2 pi k / Q_out;
    PER_PAIR also returns the 3-point parabolic-refined angle when refine=True."""
    require_cuda(img_blocks, tmpl_blocks, work)
    dev = img_blocks.device
    if mode == PER_PAIR:
        if best_val is None:
            best_val = torch.empty((M, T), dtype=torch.float32, device=dev)
        if best_k is None:
            best_k = torch.empty((M, T), dtype=torch.int32, device=dev)
        if refine and best_gamma is None:
            best_gamma = torch.empty((M, T), dtype=torch.float32, device=dev)
    else:
        if best_key is None:
            best_key = torch.zeros(M, dtype=torch.int64, device=dev)
    check(_lib.lib().rsvd_align_argmax_fine(ptr(img_blocks), M, ptr(tmpl_blocks), T, t_offset, Q, H, Q_out, mode,
                                            ptr(work), work.numel() * work.element_size(), ptr(best_val),
                                            ptr(best_k), ptr(best_key), ptr(best_gamma), stream_handle(stream)))
    return (best_val, best_k, best_gamma) if mode == PER_PAIR else best_key


def align_landscape_fine(img_blocks, M: int, tmpl_blocks, T: int, Q: int, H: int, Q_out: int, work, X=None,
                         ld_m: int | None = None, ld_t: int | None = None, stream=None):
    """rsvd_align_landscape_fine: Re X on the zero-padded grid gamma_k = 2 pi k / Q_out."""
    require_cuda(img_blocks, tmpl_blocks, work)
    if X is None:
        X = torch.empty((M, T, Q_out), dtype=torch.float32, device=img_blocks.device)
        ld_m, ld_t = T * Q_out, Q_out
    check(_lib.lib().rsvd_align_landscape_fine(ptr(img_blocks), M, ptr(tmpl_blocks), T, Q, H, Q_out, ptr(work),
                                               work.numel() * work.element_size(), ptr(X), ld_m, ld_t,
                                               stream_handle(stream)))
    return X


def winners_reset(keys: torch.Tensor, stream=None):
    require_cuda(keys)
    check(_lib.lib().rsvd_winners_reset(ptr(keys), keys.numel(), stream_handle(stream)))
    return keys


def winners_unpack(keys: torch.Tensor, Q: int, stream=None):
    require_cuda(keys)
    M = keys.numel()
    val = torch.empty(M, dtype=torch.float32, device=keys.device)
    t = torch.empty(M, dtype=torch.int32, device=keys.device)
    k = torch.empty(M, dtype=torch.int32, device=keys.device)
    check(_lib.lib().rsvd_winners_unpack(ptr(keys), M, Q, ptr(val), ptr(t), ptr(k), stream_handle(stream)))
    return val, t, k


def combine_winners(keys_g: torch.Tensor, Q: int, stream=None):
    """keys_g [G, M] (all-gathered per-rank keys) -> (keys, val, t, k) of the global winners."""
    require_cuda(keys_g)
    G, M = keys_g.shape
    out = torch.empty(M, dtype=torch.int64, device=keys_g.device)
    val = torch.empty(M, dtype=torch.float32, device=keys_g.device)
    t = torch.empty(M, dtype=torch.int32, device=keys_g.device)
    k = torch.empty(M, dtype=torch.int32, device=keys_g.device)
    check(_lib.lib().rsvd_combine_winners(ptr(keys_g), G, M, Q, ptr(out), ptr(val), ptr(t), ptr(k),
                                          stream_handle(stream)))
    return out, val, t, k


# ------------------------------------------------------------------ instrumentation
TIMING_KINDS = ("contract", "fft_reduce", "compress", "kernel_partials", "align_fused")


def launch_count() -> int:
    return int(_lib.lib().rsvd_launch_count())


def timing_enable(on: bool = True):
    _lib.lib().rsvd_timing_enable(1 if on else 0)


def timing_read():
    """{kind: (total_ms, launches)} for the event-bracketed launches since the last read."""
    ms = np.zeros(len(TIMING_KINDS), dtype=np.float64)
    cnt = np.zeros(len(TIMING_KINDS), dtype=np.int64)
    check(_lib.lib().rsvd_timing_read(ptr(ms), ptr(cnt), len(TIMING_KINDS)))
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(TIMING_KINDS)}


PROBE_KINDS = {"ffma": 0, "ffma2": 1, "fadd2": 2, "dfma": 3, "dmma8": 4, "dmma16": 5}


def probe_fp32(kind: str = "ffma2", iters: int = 200000, stream=None) -> float:
    """Measured sustained FP32 TFLOP/s of the current device (rsvd_probe_fp32): the Pi_fp32 roofline
    denominator of SURVEY.md 8(d)."""
    out = np.zeros(1, dtype=np.float64)
    check(_lib.lib().rsvd_probe_fp32(PROBE_KINDS[kind], iters, ptr(out), stream_handle(stream)))
    return float(out[0])


# ------------------------------------------------------------------ the full path
class Aligner:
    """Many-to-many rotational alignment compressed by the radial-SVD (one GPU).

    >>> al = Aligner(w, H)                       # radial weights of the shared polar grid
    >>> al.fit(templates)                        # a0: basis from the templates' kernel C
    >>> res = al.align(images, templates)        # a1-a4: compress both, align, argmax
    """

    def __init__(self, w, H: int, device="cuda", workspace_bytes: int | None = None):
        self.H = int(H)
        self.device = torch.device(device)
        self.w_host = np.ascontiguousarray(np.asarray(w.cpu() if torch.is_tensor(w) else w), dtype=np.float64)
        self.w = torch.tensor(self.w_host, dtype=torch.float64, device=self.device)
        self.U = None
        self.U_dev = None
        self.lam = None
        self._work = None
        self._work_bytes = workspace_bytes

    def set_basis(self, U):
        self.U = np.ascontiguousarray(U, dtype=np.float64)
        self.U_dev = torch.tensor(self.U, device=self.device)
        return self

    def fit(self, templates: torch.Tensor):
        U, lam = build_basis(templates, self.w_host, self.H)
        self.lam = lam
        return self.set_basis(U)

    def workspace(self, M: int, T: int, Q: int) -> torch.Tensor:
        nb = self._work_bytes or align_workspace_bytes(M, T, Q, self.H)
        nb = max(nb, align_min_workspace_bytes(Q))
        if self._work is None or self._work.numel() * 4 < nb:
            self._work = torch.empty((nb + 3) // 4, dtype=torch.float32, device=self.device)
        return self._work

    def compress(self, rings: torch.Tensor, side: int, out=None):
        return compress(rings, self.w, self.U_dev, side, out=out)

    def align_blocks(self, img_blocks, M, tmpl_blocks, T, Q, mode=PER_IMAGE, t_offset=0, keys=None):
        work = self.workspace(M, T, Q)
        if mode == PER_PAIR:
            return align_argmax(img_blocks, M, tmpl_blocks, T, Q, self.H, PER_PAIR, work)
        if keys is None:
            keys = torch.zeros(M, dtype=torch.int64, device=self.device)
        return align_argmax(img_blocks, M, tmpl_blocks, T, Q, self.H, PER_IMAGE, work, best_key=keys,
                            t_offset=t_offset)

    def landscape_blocks(self, img_blocks, M, tmpl_blocks, T, Q, X=None, ld_m=None, ld_t=None):
        return align_landscape(img_blocks, M, tmpl_blocks, T, Q, self.H, self.workspace(M, T, Q), X, ld_m, ld_t)

    def align(self, images: torch.Tensor, templates: torch.Tensor, mode=PER_IMAGE):
        """Full pass from rings: returns per-pair (val [M,T], k [M,T]) or per-image (val, t, k) [M]."""
        M, R, Q = images.shape
        T = templates.shape[0]
        if self.U is None:
            self.fit(templates)
        ib = self.compress(images, SIDE_IMAGE)
        tb = self.compress(templates, SIDE_TEMPLATE)
        if mode == PER_PAIR:
            return self.align_blocks(ib, M, tb, T, Q, PER_PAIR)
        keys = self.align_blocks(ib, M, tb, T, Q, PER_IMAGE)
        return winners_unpack(keys, Q)


# ------------------------------------------------------------------ row f4: volumes (include/rsvd_vol.h)
def vol_ncoef(L: int) -> int:
    return int(_lib.lib().rsvd_vol_ncoef(L))


def vol_grid(L: int) -> int:
    """Default alpha/gamma grid size P: the smallest power of two >= max(32, 2L + 1) (V1)."""
    P = 32
    while P < 2 * L + 1:
        P *= 2
    return P


def vol_kernels(B: torch.Tensor, w: torch.Tensor, L: int, stream=None):
    """rsvd_vol_kernels: B complex64 [nB, R, (L+1)^2] -> (C [R, R], D [L+1, L+1]) float64 device tensors."""
    require_cuda(B, w)
    nB, R, _ = B.shape
    C = torch.empty(R, R, dtype=torch.float64, device=B.device)
    D = torch.empty(L + 1, L + 1, dtype=torch.float64, device=B.device)
    check(_lib.lib().rsvd_vol_kernels(ptr(B), nB, R, L, ptr(w), ptr(C), ptr(D), stream_handle(stream)))
    return C, D


def vol_bases(B: torch.Tensor, w: torch.Tensor, L: int, HC: int, HD: int, stream=None):
    """Kernels on the device, eigen-solves in the library's host solver -> (U [R, HC], V [L+1, HD]) fp64 numpy."""
    C, D = vol_kernels(B, w, L, stream)
    U, _ = eigen_basis(C.cpu().numpy(), HC)
    V, _ = eigen_basis(D.cpu().numpy(), HD)
    return U, V


def vol_compress(A: torch.Tensor, w: torch.Tensor, U: torch.Tensor, L: int, out=None, stream=None):
    """rsvd_vol_compress: A complex64 [n, R, (L+1)^2] -> principal shells complex64 [n, HC, (L+1)^2]."""
    require_cuda(A, w, U)
    n, R, _ = A.shape
    HC = U.shape[1]
    if out is None:
        out = torch.empty(n, HC, (L + 1) ** 2, dtype=torch.complex64, device=A.device)
    check(_lib.lib().rsvd_vol_compress(ptr(A), n, R, L, ptr(w), ptr(U), HC, ptr(out), stream_handle(stream)))
    return out


def vol_wigner_table(beta: torch.Tensor, L: int, V: torch.Tensor, out=None, stream=None):
    """rsvd_vol_wigner_table: beta float64 [nb], V float64 [L+1, HD] -> T float32 [nb, HD, M (m2), M (m1)]."""
    require_cuda(beta, V)
    nb, HD, M = beta.numel(), V.shape[1], 2 * L + 1
    if out is None:
        out = torch.empty(nb, HD, M, M, dtype=torch.float32, device=V.device)
    check(_lib.lib().rsvd_vol_wigner_table(ptr(beta), nb, L, ptr(V), HD, ptr(out), stream_handle(stream)))
    return out


def vol_degrees(shells_a: torch.Tensor, shell_b: torch.Tensor, L: int, V: torch.Tensor, out=None, stream=None):
    """rsvd_vol_degrees (Steps 1 + 1b): -> Y complex64 [n, HD, M (m2), M (m1)]."""
    require_cuda(shells_a, shell_b, V)
    n, HC, _ = shells_a.shape
    HD, M = V.shape[1], 2 * L + 1
    if out is None:
        out = torch.empty(n, HD, M, M, dtype=torch.complex64, device=shells_a.device)
    check(_lib.lib().rsvd_vol_degrees(ptr(shells_a), n, ptr(shell_b), L, HC, ptr(V), HD, ptr(out), stream_handle(stream)))
    return out


def vol_align(Y: torch.Tensor, T: torch.Tensor, L: int, P: int, landscape: bool = True, keys=None, X=None,
              stream=None):
    """rsvd_vol_align (Steps 2 + 3): -> (X float32 [n, nb, P, P] or None, keys int64 [n] or None)."""
    require_cuda(Y, T)
    n, HD = Y.shape[0], Y.shape[1]
    nb = T.shape[0]
    if landscape and X is None:
        X = torch.empty(n, nb, P, P, dtype=torch.float32, device=Y.device)
    check(_lib.lib().rsvd_vol_align(ptr(Y), n, ptr(T), nb, L, HD, P, ptr(X) if landscape else None,
                                    ptr(keys) if keys is not None else None, stream_handle(stream)))
    return (X if landscape else None), keys


def vol_best(keys: torch.Tensor, P: int, stream=None):
    """Decode packed per-volume keys -> (value, b, a, g) with rsvd_winners_unpack (Q := P*P)."""
    val, b, ag = winners_unpack(keys, P * P, stream)
    return val, b, ag // P, ag % P


class VolumeAligner:
    """Row f4 end to end: bases from the target -> principal shells -> Wigner table ->
    Steps 1/1b -> Steps 2/3 with the per-volume argmax.  All arithmetic runs in librsvd's kernels."""

    def __init__(self, target: torch.Tensor, w: torch.Tensor, L: int, HC: int, HD: int, betas: torch.Tensor,
                 P: int | None = None, stream=None):
        self.L, self.P = L, P or vol_grid(L)
        self.w = w
        self.stream = stream
        tgt = target if target.dim() == 3 else target[None]
        U, V = vol_bases(tgt, w, L, HC, HD, stream)
        self.U = torch.as_tensor(U, device=w.device)
        self.V = torch.as_tensor(V, device=w.device)
        self.shell_b = vol_compress(tgt[:1], w, self.U, L, stream=stream)[0]
        self.T = vol_wigner_table(betas, L, self.V, stream=stream)

    def align(self, volumes: torch.Tensor, landscape: bool = False):
        """-> (X or None, (value, b, a, g)) for every volume."""
        sa = vol_compress(volumes, self.w, self.U, self.L, stream=self.stream)
        Y = vol_degrees(sa, self.shell_b, self.L, self.V, stream=self.stream)
        keys = torch.zeros(volumes.shape[0], dtype=torch.int64, device=volumes.device)
        X, keys = vol_align(Y, self.T, self.L, self.P, landscape=landscape, keys=keys, stream=self.stream)
        return X, vol_best(keys, self.P, self.stream)
