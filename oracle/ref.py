"""fp64 CPU oracle for the radial-SVD alignment path (arXiv 2202.07235).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module.  It shares no code with the CUDA path
(paper_2202_07235_b200/) and never imports it.  Inputs are the exact complex64 samples the
GPU consumed, up-cast to complex128, plus w_r in fp64.

Functions (each follows the cited passage; numbers refer to /root/reference/PAPER.md lines):

O1 landscape_full      X[k] = sum_r w_r dpsi sum_j conj(a[r,j]) b[r,(j-k) mod Q]
                       (PAPER.md:127-135 §2.2, :236-240 §2.3) -- C direct sum, oracle/direct.c
O2 landscape_rank      same sum over the H principal rings at = U^T (sqrt(w) a) (PAPER.md:580-585
                       §3.2, eta_r = sqrt(w_r) per DESIGN.md reading G2) -- C direct sum
O3 kernel_C / basis    C_{rr'} = (1/T) sum_t sum_{q != 0} Re( conj(b'_t[r,q]) b'_t[r',q] ),
                       b'_t[r,q] = sqrt(w_r) bhat_t[r,q], bhat = (1/Q) DFT_psi  (Eq. Image_simple_kern
                       PAPER.md:661-665 with the eta rescaling of Eq. Image_single_kern :643-651,
                       averaged over targets per Eq. image_cost_and_kern :704-708; constants
                       (2pi)^3/(4 sigma_hat^2) dropped, real part taken: readings G1, G6).
                       Basis = eigenvectors of C by LAPACK eigh, descending (the paper's "SVD of C",
                       :667; reading G7).
O4 reductions          per-pair argmax of Re X with smallest-k tie-break; per-image argmax over
                       (t, k) lexicographic; top-2 gap and near-tie set (DESIGN.md tolerance rules).
O5 metrics             relative Frobenius error, Pearson correlation, backward-error fraction f
                       (§3.5).
P8 landscape_fb        2 pi sum_q e^{-2 pi i q k / Q} sum_r w_r conj(ahat[r,q]) bhat[r,q] with a
                       DIRECT (matrix) DFT -- Eq. image_innerproduct_0; used only
                       as a pin against O1.
F1 landscape_rank_fine Re X at gamma_k = 2 pi k / Q_out from the rank-H coefficients, evaluated
                       directly (no FFT): "zero-padded prior to the FFT" with the
                       Nyquist bin split between +-Q/2 (reading G4).
F1 argmax_refine       grid argmax + 3-point quadratic interpolation (SPEC.md argmax_refine).
F2 translate           a exp(-i k_r (dx cos psi_j + dy sin psi_j)), the Fourier shift theorem with the
                       transform convention of PAPER.md:80 (reading G15), fp64; the translation-averaged
                       kernel of Eq. eq_Image_single_cost_with_translations (:1146-1150) for a discrete
                       shift distribution is kernel_C of the translated templates.

T1 kernel_translated_sh  the closed-form target-averaged kernel with Gaussian translations (sigma_d)
                       and uniform views, Eq. template_cost_with_translations, from
                       the target volume's spherical-harmonic coefficients B_l^m(k_r), with E+ and E-
                       written exactly as printed (E- via the modified Bessel functions I_{-1/2}, I_{1/2});
                       times sqrt(w_r w_r'), real part (readings G6, T1 in DESIGN.md).

Parity pins for every function live in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "direct.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile oracle/direct.c into oracle/liboracle.so (gcc -O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build_oracle()
            lib = ctypes.CDLL(_LIB)
            d, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
            lib.oracle_landscape_full_pairs.argtypes = [i32, i32, d, d, d, i64, d, d, d, i32]
            lib.oracle_landscape_rank_pairs.argtypes = [i32, i32, i32, d, d, d, d, i64, d, d, d, i32]
            lib.oracle_principal_rings.argtypes = [i32, i32, i32, d, d, d, d]
            lib.oracle_correlate_pairs.argtypes = [i32, i32, d, d, i64, d, d, d, i32]
            lib.oracle_max_threads.restype = i32
            _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x), dtype=np.complex128)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _pairs(ia, ib):
    ia = np.ascontiguousarray(np.asarray(ia, dtype=np.int64).ravel())
    ib = np.ascontiguousarray(np.asarray(ib, dtype=np.int64).ravel())
    assert ia.shape == ib.shape
    return ia, ib


# ------------------------------------------------------------------------------------ O1 / O2
def landscape_full(A, B, w, ia, ib, nthreads: int = 0) -> np.ndarray:
    """O1 for pairs (A[ia[p]], B[ib[p]]); A: [NA,R,Q], B: [NB,R,Q] complex.  Returns [P,Q] c128."""
    A, B = _c128(A), _c128(B)
    w = np.ascontiguousarray(w, dtype=np.float64)
    ia, ib = _pairs(ia, ib)
    _, R, Q = A.shape
    X = np.zeros((ia.size, Q), dtype=np.complex128)
    _load().oracle_landscape_full_pairs(R, Q, _ptr(w), _ptr(A), _ptr(B), ia.size, _ptr(ia),
                                        _ptr(ib), _ptr(X), int(nthreads))
    return X


def principal_rings(A, w, U) -> np.ndarray:
    """at[n, h, j] = sum_r U[r, h] sqrt(w_r) A[n, r, j] (eta_r = sqrt(w_r))."""
    A = _c128(A)
    w = np.ascontiguousarray(w, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    n, R, Q = A.shape
    H = U.shape[1]
    out = np.zeros((n, H, Q), dtype=np.complex128)
    lib = _load()
    for i in range(n):
        lib.oracle_principal_rings(R, Q, H, _ptr(w), _ptr(U), _ptr(A[i]), _ptr(out[i]))
    return out


def landscape_rank(A, B, w, U, ia, ib, nthreads: int = 0) -> np.ndarray:
    """O2: rank-H landscape through U's principal rings, direct sum.  Returns [P,Q] c128.

    Principal rings are computed once per distinct row, then correlated per pair."""
    ia, ib = _pairs(ia, ib)
    ua, inv_a = np.unique(ia, return_inverse=True)
    ub, inv_b = np.unique(ib, return_inverse=True)
    AT = principal_rings(np.asarray(A)[ua], w, U)
    BT = principal_rings(np.asarray(B)[ub], w, U)
    H, Q = AT.shape[1], AT.shape[2]
    ja = np.ascontiguousarray(inv_a.astype(np.int64))
    jb = np.ascontiguousarray(inv_b.astype(np.int64))
    X = np.zeros((ia.size, Q), dtype=np.complex128)
    _load().oracle_correlate_pairs(H, Q, _ptr(AT), _ptr(BT), ia.size, _ptr(ja), _ptr(jb),
                                   _ptr(X), int(nthreads))
    return X


def landscape_fb(A, B, w, ia, ib) -> np.ndarray:
    """P8 form (pin only): 2 pi sum_q e^{-2 pi i q k/Q} sum_r w_r conj(ahat) bhat with a direct DFT,
    ahat[r,q] = (1/Q) sum_j a[r,j] e^{-2 pi i q j / Q} (reading G1).  Eq. image_innerproduct_0."""
    A, B = _c128(A), _c128(B)
    ia, ib = _pairs(ia, ib)
    Q = A.shape[2]
    j = np.arange(Q)
    F = np.exp(-2j * np.pi * np.outer(j, j) / Q)           # F[q, j] = e^{-2 pi i q j / Q}
    out = np.zeros((ia.size, Q), dtype=np.complex128)
    for p in range(ia.size):
        ah = A[ia[p]] @ F.T / Q                            # [R, Q] over q
        bh = B[ib[p]] @ F.T / Q
        S = (np.asarray(w)[:, None] * np.conj(ah) * bh).sum(axis=0)     # Step 1 (:358)
        out[p] = 2.0 * np.pi * (F @ S)                     # Step 2 (:359): sum_q e^{-i q gamma_k} S_q
    return out


# ------------------------------------------------------------------------------------ F1
def landscape_rank_fine(A, B, w, U, ia, ib, Q_out: int) -> np.ndarray:
    """F1: Re X(gamma_k), gamma_k = 2 pi k / Q_out, of the rank-H landscape (real, [P, Q_out]).

    Coefficients of the principal rings (eta_r = sqrt(w_r): G2) by a direct DFT,
    Ahat[h, q] = (1/Q) sum_j at[h, j] e^{-2 pi i q j/Q} (G1); S_q = sum_h conj(Ahat[h,q]) Bhat[h,q]
    (Step 1, :672); then the zero-padded transform (:363) evaluated term by term:
      X(gamma) = 2 pi [ sum_{q=-Q/2+1}^{Q/2-1} e^{-i q gamma} S_q + cos(Q gamma / 2) S_{Q/2} ],
    S_{-q} == S_{Q-q}; the unpaired bin Q/2 split symmetrically between +-Q/2 (reading G4)."""
    ia, ib = _pairs(ia, ib)
    AT = principal_rings(np.asarray(A)[ia], w, U)          # [P, H, Q]
    BT = principal_rings(np.asarray(B)[ib], w, U)
    Q = AT.shape[2]
    j = np.arange(Q)
    F = np.exp(-2j * np.pi * np.outer(j, j) / Q)           # F[q, j]
    Ah = AT @ F.T / Q                                      # [P, H, q]
    Bh = BT @ F.T / Q
    S = (np.conj(Ah) * Bh).sum(axis=1)                     # [P, q]
    N = Q // 2
    gam = 2.0 * np.pi * np.arange(Q_out) / Q_out
    qs = np.concatenate([np.arange(0, N), np.arange(-N + 1, 0)])       # signed frequencies, Nyquist apart
    cols = np.concatenate([np.arange(0, N), np.arange(N + 1, Q)])
    E = np.exp(-1j * np.outer(qs, gam))                    # [freq, gamma]
    X = S[:, cols] @ E + S[:, N][:, None] * np.cos(N * gam)[None, :]
    return (2.0 * np.pi * X).real


def translate(A, k, shifts) -> np.ndarray:
    """F2: rows b*S + s = A[b] exp(-i k_r (dx_s cos psi_j + dy_s sin psi_j)) in fp64 (reading G15)."""
    A = _c128(A)
    n, R, Q = A.shape
    k = np.asarray(k, dtype=np.float64)
    sh = np.asarray(shifts, dtype=np.float64).reshape(-1, 2)
    psi = 2.0 * np.pi * np.arange(Q) / Q
    out = np.empty((n * sh.shape[0], R, Q), dtype=np.complex128)
    for s, (dx, dy) in enumerate(sh):
        ramp = np.exp(-1j * k[:, None] * (dx * np.cos(psi) + dy * np.sin(psi))[None, :])
        out[s::sh.shape[0]] = A * ramp[None]
    return out


def argmax_refine(x: np.ndarray) -> np.ndarray:
    """SPEC.md argmax_refine along the last axis: gamma = 2 pi (k + d) / Q, k the first argmax,
    d = (y[k-1] - y[k+1]) / (2 (y[k-1] - 2 y[k] + y[k+1])) (vertex of the parabola through the three
    cyclic neighbours), d = 0 unless the curvature is negative, clamped to [-1/2, 1/2]; in [0, 2 pi)."""
    x = np.asarray(x, dtype=np.float64)
    Q = x.shape[-1]
    k = argmax_first(x)
    y0 = np.take_along_axis(x, k[..., None], -1)[..., 0]
    ym = np.take_along_axis(x, ((k - 1) % Q)[..., None], -1)[..., 0]
    yp = np.take_along_axis(x, ((k + 1) % Q)[..., None], -1)[..., 0]
    den = ym - 2.0 * y0 + yp
    with np.errstate(divide="ignore", invalid="ignore"):
        d = np.where(den < 0, 0.5 * (ym - yp) / np.where(den < 0, den, 1.0), 0.0)
    d = np.clip(d, -0.5, 0.5)
    return np.mod(2.0 * np.pi * (k + d) / Q, 2.0 * np.pi)


# ------------------------------------------------------------------------------------ O3
def fb_coefficients(A) -> np.ndarray:
    """bhat[n, r, q] = (1/Q) sum_j a[n, r, j] e^{-2 pi i q j/Q} (reading G1)."""
    A = _c128(A)
    return np.fft.fft(A, axis=-1) / A.shape[-1]


def kernel_C(templates, w) -> np.ndarray:
    """O3 kernel: C_{rr'} = (1/T) sum_t sum_{q=1}^{Q-1} Re(conj(b'[r,q]) b'[r',q]), b' = sqrt(w) bhat.

    Eq. Image_simple_kern averaged per Eq. image_cost_and_kern (:704-708),
    q = 0 excluded as the paper states (:665); constants dropped, Re taken (G6)."""
    B = fb_coefficients(templates)                         # [T, R, Q]
    T = B.shape[0]
    Bp = np.sqrt(np.asarray(w, dtype=np.float64))[None, :, None] * B[:, :, 1:]
    C = np.einsum("trq,tsq->rs", np.conj(Bp), Bp).real / T
    return 0.5 * (C + C.T)


def basis(C, H: int):
    """Top-H eigenvectors of C (descending eigenvalues) by LAPACK eigh.  Returns (U [R,H], lam [R])."""
    lam, V = np.linalg.eigh(np.asarray(C, dtype=np.float64))
    order = np.argsort(lam)[::-1]
    lam = lam[order]
    V = V[:, order]
    return V[:, :H].copy(), lam


def projector(U) -> np.ndarray:
    U = np.asarray(U, dtype=np.float64)
    return U @ U.T


# ------------------------------------------------------------------------------------ O4
def argmax_first(x: np.ndarray) -> np.ndarray:
    """Index of the maximum along the last axis, smallest index among equal maxima."""
    return np.argmax(x, axis=-1)          # numpy returns the first occurrence


def top2_gap(x: np.ndarray) -> np.ndarray:
    """Largest minus second-largest entry along the last axis (entries, not local peaks: G10)."""
    s = np.sort(x, axis=-1)
    return s[..., -1] - s[..., -2]


def near_tie_ok(x_ref: np.ndarray, k_gpu: np.ndarray, tol_abs: float) -> np.ndarray:
    """True where the GPU index lies in {k : x_ref[k] >= max - tol_abs} (DESIGN.md gating rule)."""
    mx = x_ref.max(axis=-1)
    val = np.take_along_axis(x_ref, np.asarray(k_gpu)[..., None].astype(np.int64), axis=-1)[..., 0]
    return val >= mx - tol_abs


def per_image_winner(X_re: np.ndarray):
    """X_re [T, Q] for one image: (value, t, k) of the max with lexicographic (t, k) tie-break."""
    flat = X_re.reshape(-1)
    i = int(np.argmax(flat))               # first occurrence = smallest t*Q + k
    return float(flat[i]), i // X_re.shape[1], i % X_re.shape[1]


# ------------------------------------------------------------------------------------ O5
def rel_frobenius(approx, full) -> float:
    """||approx - full||_F / ||full||_F."""
    return float(np.linalg.norm(np.asarray(approx) - np.asarray(full)) / np.linalg.norm(full))


def correlation(approx, full) -> float:
    """Pearson correlation over the whole array."""
    a = np.asarray(approx, dtype=np.float64).ravel()
    b = np.asarray(full, dtype=np.float64).ravel()
    a = a - a.mean()
    b = b - b.mean()
    return float((a @ b) / np.sqrt((a @ a) * (b @ b)))


def backward_fraction(approx, full) -> np.ndarray:
    """f per pair: fraction of full[k] <= full[argmax approx] (inclusive <=)."""
    approx = np.asarray(approx)
    full = np.asarray(full)
    ke = argmax_first(approx)
    xe = np.take_along_axis(full, ke[..., None], axis=-1)
    return (full <= xe).sum(axis=-1) / full.shape[-1]


# ------------------------------------------------------------------------------------ T1
def E_plus(k, kp, sigma: float) -> np.ndarray:
    """E+(k_r, k_r') = exp(-sigma^2/2 [k_r^2 + k_r'^2]) exp(k_r k_r' sigma^2), as
    printed: the outer product over the radial nodes."""
    k = np.asarray(k, np.float64)[:, None]
    kp = np.asarray(kp, np.float64)[None, :]
    return np.exp(-0.5 * sigma ** 2 * (k ** 2 + kp ** 2)) * np.exp(k * kp * sigma ** 2)


def E_minus(k, sigma: float) -> np.ndarray:
    """E-(k_r) = kt sqrt(pi/2) exp(-kt^2) (I_{-1/2}(kt^2) - I_{+1/2}(kt^2)), kt = k sigma / 2
    (PAPER.md:1164-1166), as printed; E-(k) -> 1 as sigma -> 0 (the limit is taken at kt = 0)."""
    import scipy.special
    k = np.asarray(k, np.float64)
    kt = k * sigma / 2.0
    out = np.ones_like(kt)
    nz = kt > 0
    x = kt[nz] ** 2
    out[nz] = kt[nz] * np.sqrt(np.pi / 2.0) * np.exp(-x) * (scipy.special.iv(-0.5, x) - scipy.special.iv(0.5, x))
    return out


def kernel_translated_sh(Bsh, k, w, sigma: float) -> np.ndarray:
    """T1: C_{rr'} = sqrt(w_r w_r') Re[ (sum_{l,m} conj(B_l^m(k_r)) B_l^m(k_r')) E+(k_r, k_r')
                                          - conj(B_0^0(k_r)) B_0^0(k_r') E-(k_r) E-(k_r') ]
    Eq. template_cost_with_translations, up to the paper's constant factor.
    Bsh [R, (L+1)^2] complex (index l*l + l + m), k [R] radial nodes, w [R] radial weights."""
    B = _c128(Bsh)
    S = np.einsum("rl,sl->rs", np.conj(B), B)
    b0 = B[:, 0]
    Em = E_minus(k, sigma)
    C = (S * E_plus(k, k, sigma) - np.outer(np.conj(b0), b0) * np.outer(Em, Em)).real
    sw = np.sqrt(np.asarray(w, np.float64))
    C = sw[:, None] * C * sw[None, :]
    return 0.5 * (C + C.T)
