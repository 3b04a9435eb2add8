"""fp64 CPU oracle for row f4: volume alignment with radial- and degree-SVD (arXiv 2202.07235 §5).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module.  It shares no code with the CUDA path
(paper_2202_07235_b200/) and never imports it.  Inputs are the exact complex64 coefficients the GPU
consumed, up-cast to complex128, plus w_r in fp64.

Volume data: spherical-harmonic coefficients A[r][lm] = A_l^m(k_r), packed lm = l*l + l + m
(0 <= l <= L, -l <= m <= l), PAPER.md:836-847 (§5.2).  Orders m in [-L, L] are stored on the
alpha/gamma grids at index m mod P ("treat the order indices periodically").

Functions (PAPER.md line numbers):

V1 wigner_d          d^l(beta) = exp(-i beta J_y) on the degree-l subspace, J_y = (J+ - J-)/(2i),
                     <l,m+1|J+|l,m> = sqrt(l(l+1) - m(m+1)): the matrix of the rotation about the
                     second axis in the spherical-harmonic basis, i.e. the
                     "degree-l wigner-d matrix associated with the interior euler-angle beta"
                     (:855-860).  scipy.linalg.expm is the library primitive.
V2 vol_kernel_C      C_{rr'} = sqrt(w_r w_r') sum_{l>=1} sum_m Re conj(B_l^m(k_r)) B_l^m(k_r')
                     (Eq. Volume_simple_radial_kern :951-954 with the sqrt(w) of :944-948; reading V2),
                     averaged over targets.
   vol_kernel_D      D_{ll'} = [l,l' >= 1] sum_r w_r sum_m Re conj(B_l^m(k_r)) B_{l'}^m(k_r)
                     (Eq. Volume_simple_degree_kern :1001-1007 as its text states: zero whenever l or
                     l' is 0; reading V3), averaged over targets.
   vol_basis         eigenvectors of C (or D), descending (the paper's "principal-vectors", :955, :1008).
V4 vol_landscape_full  X(beta_b; alpha_a, gamma_g) = Re sum_{m1,m2} e^{-i m1 alpha_a} e^{-i m2 gamma_g}
                     sum_l d^l_{m1 m2}(beta_b) sum_r w_r conj(A_l^{m1}(k_r)) B_l^{m2}(k_r),
                     alpha_a = 2 pi a / P, gamma_g = 2 pi g / P  (Eq. volume_innerproduct :894-904 with
                     the P-point grids of reading V1), the three steps written out as stated.
V5 vol_landscape_rank  the same with the radial- and degree-SVD: Steps 1, 1b, 2, 3 of
                     Eq. volume_innerproduct_pm (:1017-1023): principal shells
                     [u_h^T A]_l^m = sum_r u_h[r] sqrt(w_r) A_l^m(k_r) (:921-927, eta_r = sqrt(w_r)),
                     Xt(m1,m2;l) = sum_h conj([u_h^T A]_l^{m1}) [u_h^T B]_l^{m2},
                     Y_j(m1,m2) = sum_l v_j[l] Xt(m1,m2;l), F(m1,m2;beta) = sum_j [v_j^T d]_{m1m2}(beta) Y_j,
                     X = 2-D DFT of F.
V6 vol_best          per volume argmax over (b, a, g) of X, smallest flat index (b*P + a)*P + g on ties.

Pins for every function live in tests/test_oracle_vol_pins.py.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg


def lm_index(l: int, m: int) -> int:
    return l * l + l + m


def wigner_d(L: int, beta: float) -> list[np.ndarray]:
    """V1: [d^0(beta), ..., d^L(beta)], d^l indexed [m1 + l, m2 + l]."""
    out = []
    for l in range(L + 1):
        m = np.arange(-l, l)                                     # J+ |l,m> -> |l,m+1>
        jp = np.zeros((2 * l + 1, 2 * l + 1))
        jp[m + l + 1, m + l] = np.sqrt(l * (l + 1) - m * (m + 1))
        # -i beta J_y = -i beta (J+ - J-) / (2i) = -(beta / 2) (J+ - J-), a real generator
        out.append(scipy.linalg.expm(-0.5 * beta * (jp - jp.T)))
    return out


def _as_c128(x):
    return np.asarray(x, dtype=np.complex128)


def vol_kernel_C(B, w) -> np.ndarray:
    """V2: B [nB, R, (L+1)^2] (or [R, (L+1)^2]); w [R]."""
    B = _as_c128(B)
    if B.ndim == 2:
        B = B[None]
    sw = np.sqrt(np.asarray(w, np.float64))
    Bp = B[:, :, 1:] * sw[None, :, None]                         # drop l = 0 (lm = 0)
    C = np.einsum("nrj,nsj->rs", Bp.conj(), Bp).real / B.shape[0]
    return C


def vol_kernel_D(B, w, L: int) -> np.ndarray:
    B = _as_c128(B)
    if B.ndim == 2:
        B = B[None]
    w = np.asarray(w, np.float64)
    D = np.zeros((L + 1, L + 1))
    for l in range(1, L + 1):
        for lp in range(1, L + 1):
            s = 0.0
            for m in range(-min(l, lp), min(l, lp) + 1):
                s += np.sum(w[None, :] * (B[:, :, lm_index(l, m)].conj() * B[:, :, lm_index(lp, m)]).real)
            D[l, lp] = s / B.shape[0]
    return D


def vol_basis(K: np.ndarray, H: int):
    lam, V = np.linalg.eigh(K)
    order = np.argsort(lam)[::-1]
    return V[:, order[:H]], lam[order]


def _dft_orders(L: int, P: int) -> np.ndarray:
    """E[a, m + L] = exp(-i m 2 pi a / P) for m in [-L, L]."""
    m = np.arange(-L, L + 1)
    return np.exp(-2j * np.pi * np.outer(np.arange(P), m) / P)


def vol_landscape_full(A, B, w, L: int, betas, P: int) -> np.ndarray:
    """V4: A [R, (L+1)^2] one volume, B [R, (L+1)^2] the target -> X [nb, P, P] (Re)."""
    A, B = _as_c128(A), _as_c128(B)
    w = np.asarray(w, np.float64)
    M = 2 * L + 1
    E = _dft_orders(L, P)
    out = np.empty((len(betas), P, P))
    # Step 1: Xt(m1, m2; l) = sum_r w_r conj(A_l^{m1}(k_r)) B_l^{m2}(k_r)
    Xt = []
    for l in range(L + 1):
        a = A[:, l * l:(l + 1) * (l + 1)]                        # [R, 2l+1], m = -l..l
        b = B[:, l * l:(l + 1) * (l + 1)]
        Xt.append(np.einsum("r,ri,rj->ij", w, a.conj(), b))
    for ib, beta in enumerate(betas):
        d = wigner_d(L, beta)
        F = np.zeros((M, M), np.complex128)                      # Step 2, orders m1, m2 in [-L, L]
        for l in range(L + 1):
            F[L - l:L + l + 1, L - l:L + l + 1] += d[l] * Xt[l]
        out[ib] = (E @ F @ E.T).real                             # Step 3: sum_{m1,m2} e^{-i m1 a} e^{-i m2 g} F
    return out


def vol_shells(A, w, U) -> np.ndarray:
    """[u_h^T A]_l^m = sum_r U[r,h] sqrt(w_r) A_l^m(k_r) -> [H, (L+1)^2]."""
    A = _as_c128(A)
    return np.einsum("rh,r,rj->hj", np.asarray(U, np.float64), np.sqrt(np.asarray(w, np.float64)), A)


def vol_landscape_rank(A, B, w, U, V, L: int, betas, P: int) -> np.ndarray:
    """V5: Steps 1, 1b, 2, 3 of Eq. volume_innerproduct_pm with U [R, HC], V [L+1, HD]."""
    sA, sB = vol_shells(A, w, U), vol_shells(B, w, U)
    V = np.asarray(V, np.float64)
    M = 2 * L + 1
    HD = V.shape[1]
    E = _dft_orders(L, P)
    # Step 1: Xt(m1, m2; l) = sum_h conj([u_h^T A]_l^{m1}) [u_h^T B]_l^{m2}
    Xt = [np.einsum("hi,hj->ij", sA[:, l * l:(l + 1) ** 2].conj(), sB[:, l * l:(l + 1) ** 2]) for l in range(L + 1)]
    # Step 1b: Y_j(m1, m2) = sum_l v_j[l] Xt(m1, m2; l)
    Y = np.zeros((HD, M, M), np.complex128)
    for l in range(L + 1):
        Y[:, L - l:L + l + 1, L - l:L + l + 1] += V[l][:, None, None] * Xt[l][None]
    out = np.empty((len(betas), P, P))
    for ib, beta in enumerate(betas):
        d = wigner_d(L, beta)
        vd = np.zeros((HD, M, M))                                # [v_j^T d]_{m1 m2}(beta)
        for l in range(L + 1):
            vd[:, L - l:L + l + 1, L - l:L + l + 1] += V[l][:, None, None] * d[l][None]
        F = np.sum(vd * Y, axis=0)                               # Step 2
        out[ib] = (E @ F @ E.T).real                             # Step 3
    return out


def vol_best(X: np.ndarray):
    """V6: X [n, nb, P, P] -> (value, flat index (b*P + a)*P + g) per volume, first max on ties."""
    flat = X.reshape(X.shape[0], -1)
    idx = np.argmax(flat, axis=1)
    return flat[np.arange(flat.shape[0]), idx], idx
