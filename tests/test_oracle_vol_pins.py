"""Pins of the f4 volume oracle (oracle/vol.py) to things other than itself: textbook Wigner-d
values and identities, library Legendre functions, the closed-form overlap of Gaussian phantoms in
real space, rotation invariants, and the full-rank reduction of the compressed landscape."""
import math

import numpy as np
import pytest
import scipy.special

from oracle import vol as ov
from synth import volumes as sv


# ------------------------------------------------------------------ V1 wigner_d
def test_wigner_identity_orthogonality_group():
    L = 12
    for l, d in enumerate(ov.wigner_d(L, 0.0)):
        assert np.abs(d - np.eye(2 * l + 1)).max() < 1e-14
    b1, b2 = 0.83, -2.1
    d1, d2, d12 = ov.wigner_d(L, b1), ov.wigner_d(L, b2), ov.wigner_d(L, b1 + b2)
    for l in range(L + 1):
        assert np.abs(d1[l] @ d1[l].T - np.eye(2 * l + 1)).max() < 1e-12      # real orthogonal
        assert np.abs(d1[l] @ d2[l] - d12[l]).max() < 1e-12                    # one-parameter group
        m = np.arange(-l, l + 1)
        sign = (-1.0) ** (m[:, None] - m[None, :])
        assert np.abs(d1[l] - sign * d1[l].T).max() < 1e-12                    # d_{m'm} = (-1)^{m'-m} d_{mm'}


def test_wigner_textbook_l1():
    b = 0.7
    d = ov.wigner_d(1, b)[1]                                                   # rows/cols m = -1, 0, 1
    c, s = math.cos(b), math.sin(b)
    want = np.array([[(1 + c) / 2, s / math.sqrt(2), (1 - c) / 2],
                     [-s / math.sqrt(2), c, s / math.sqrt(2)],
                     [(1 - c) / 2, -s / math.sqrt(2), (1 + c) / 2]])
    assert np.abs(d - want).max() < 1e-14


def test_wigner_column_m2_zero_is_associated_legendre():
    """d^l_{m0}(beta) = sqrt((l-m)!/(l+m)!) P_l^m(cos beta) (Condon-Shortley P_l^m, scipy.lpmv)."""
    L = 20
    for b in (0.3, 1.9, 2.7):                          # beta in [0, pi]: sin beta >= 0 as in P_l^m
        d = ov.wigner_d(L, b)
        for l in range(L + 1):
            for m in range(0, l + 1):
                want = math.sqrt(math.factorial(l - m) / math.factorial(l + m)) * scipy.special.lpmv(m, l, math.cos(b))
                assert abs(d[l][m + l, l] - want) < 1e-11, (b, l, m)


# ------------------------------------------------------------------ generator conventions
def test_phantom_coefficients_rotate_by_wigner_D():
    """The rotated phantom's coefficients equal e^{-i m1 alpha} d^l(beta) e^{-i m2 gamma} applied to the
    original's: pins V1's sign/phase convention against the generator's Y_l^m."""
    vs = sv.make_volumes(10, 12, 1, nb=8, atoms=6, K=8.0, seed=1)
    B = sv.sh_coefficients(vs.target_centres, vs.k, 10)
    al, be, ga = 0.7, 1.1, -0.4
    Brot = sv.sh_coefficients(vs.target_centres @ sv.rotation(al, be, ga).T, vs.k, 10)
    d = ov.wigner_d(10, be)
    for l in range(11):
        m = np.arange(-l, l + 1)
        D = np.exp(-1j * m[:, None] * al) * d[l] * np.exp(-1j * m[None, :] * ga)
        assert np.abs(B[:, l * l:(l + 1) ** 2] @ D.T - Brot[:, l * l:(l + 1) ** 2]).max() < 1e-11


def test_phantom_parseval_closed_form():
    vs = sv.make_volumes(10, 12, 1, nb=8, atoms=6, K=8.0, seed=2)
    A = sv.sh_coefficients(vs.target_centres, vs.k, 10)
    lhs = np.sum(vs.w[:, None] * np.abs(A) ** 2)
    assert abs(lhs / sv.gaussian_overlap(vs.target_centres, vs.target_centres, vs.k, vs.w) - 1) < 1e-10


# ------------------------------------------------------------------ V2 / V3 kernels
def test_kernels_invariants():
    L, R = 9, 10
    vs = sv.make_volumes(L, R, 1, nb=4, atoms=8, K=7.0, seed=3)
    B = sv.sh_coefficients(vs.target_centres, vs.k, L)
    Brot = sv.sh_coefficients(vs.target_centres @ sv.rotation(0.4, 2.2, 1.3).T, vs.k, L)
    C, D = ov.vol_kernel_C(B, vs.w), ov.vol_kernel_D(B, vs.w, L)
    assert np.abs(C - C.T).max() < 1e-9 * np.abs(C).max() and np.linalg.eigvalsh(C).min() > -1e-9 * np.abs(C).max()
    assert np.abs(D - D.T).max() < 1e-9 * np.abs(D).max() and np.linalg.eigvalsh(D).min() > -1e-9 * np.abs(D).max()
    assert np.all(D[0] == 0) and np.all(D[:, 0] == 0)                           # l = 0 excluded
    # both traces are sum_r w_r sum_{l>=1} ||B_l(k_r)||^2: the sqrt(w) of C and the w of D agree
    assert abs(np.trace(C) / np.trace(D) - 1) < 1e-12
    # C and diag(D) are invariant under rotating the target (each degree rotates unitarily)
    assert np.abs(ov.vol_kernel_C(Brot, vs.w) - C).max() < 1e-9 * np.abs(C).max()
    assert np.abs(np.diag(ov.vol_kernel_D(Brot, vs.w, L)) - np.diag(D)).max() < 1e-9 * np.abs(D).max()
    # closed form: tr C = sum_r w_r int |B(k_r, .)|^2 minus the l = 0 part
    full = sv.gaussian_overlap(vs.target_centres, vs.target_centres, vs.k, vs.w)
    l0 = np.sum(vs.w * np.abs(B[:, 0]) ** 2)
    assert abs((np.trace(C) + l0) / full - 1) < 1e-8


# ------------------------------------------------------------------ V4 landscape
@pytest.fixture(scope="module")
def small_case():
    L, R = 10, 12
    vs = sv.make_volumes(L, R, 3, nb=6, atoms=7, K=8.0, seed=4)
    return vs


def test_landscape_matches_real_space_overlap(small_case):
    """X(tau) = <A, R_tau B> equals the closed-form overlap of the phantoms with the
    target's atoms rotated by tau -- at every grid point of two betas."""
    vs = small_case
    A = vs.volumes[0].astype(np.complex128)
    ca = vs.target_centres @ sv.rotation(2 * np.pi * vs.tau_index[0, 1] / vs.P, vs.betas[vs.tau_index[0, 0]],
                                         2 * np.pi * vs.tau_index[0, 2] / vs.P).T
    # volumes are stored complex64; compare with the phantom in fp64 instead for the closed form
    A64 = sv.sh_coefficients(ca, vs.k, vs.L)
    B64 = sv.sh_coefficients(vs.target_centres, vs.k, vs.L)
    for b in (1, 4):
        X = ov.vol_landscape_full(A64, B64, vs.w, vs.L, [vs.betas[b]], vs.P)[0]
        for a, g in [(0, 0), (3, 17), (31, 5), (12, 12)]:
            Rm = sv.rotation(2 * np.pi * a / vs.P, vs.betas[b], 2 * np.pi * g / vs.P)
            want = sv.gaussian_overlap(ca, vs.target_centres @ Rm.T, vs.k, vs.w)
            assert abs(X[a, g] - want) < 1e-8 * abs(sv.gaussian_overlap(ca, ca, vs.k, vs.w)), (b, a, g)
    assert A.shape == A64.shape


def test_landscape_recovers_grid_rotation(small_case):
    vs = small_case
    B = vs.target.astype(np.complex128)
    for i in range(3):
        X = ov.vol_landscape_full(vs.volumes[i], B, vs.w, vs.L, vs.betas, vs.P)
        val, idx = ov.vol_best(X[None])
        b, a, g = vs.tau_index[i]
        assert idx[0] == (b * vs.P + a) * vs.P + g
        norm = np.sum(vs.w[:, None] * np.abs(vs.volumes[i].astype(np.complex128)) ** 2)
        assert abs(val[0] / norm - 1) < 1e-5                                   # complex64 storage


# ------------------------------------------------------------------ V5 compressed landscape
def test_rank_full_equals_full(small_case):
    vs = small_case
    B = vs.target
    U, _ = ov.vol_basis(ov.vol_kernel_C(B, vs.w), vs.R)
    V = np.eye(vs.L + 1)                                                        # all degrees
    Xr = ov.vol_landscape_rank(vs.volumes[1], B, vs.w, U, V, vs.L, vs.betas[:3], vs.P)
    Xf = ov.vol_landscape_full(vs.volumes[1], B, vs.w, vs.L, vs.betas[:3], vs.P)
    assert np.abs(Xr - Xf).max() < 1e-10 * np.abs(Xf).max()
    Vd, _ = ov.vol_basis(ov.vol_kernel_D(B, vs.w, vs.L) + np.diag([1.0] + [0.0] * vs.L), vs.L + 1)
    Xr2 = ov.vol_landscape_rank(vs.volumes[1], B, vs.w, U, Vd, vs.L, vs.betas[:3], vs.P)
    assert np.abs(Xr2 - Xf).max() < 1e-9 * np.abs(Xf).max()                   # any orthonormal full V


def test_rank_truncated_projector_form(small_case):
    """Truncated ranks: equal to the uncompressed sums with w_r replaced by the radial projector
    sum_h U U^T (sqrt w sqrt w') and d^l X_l by sum_{l'} (V V^T)_{l l'} d^l X_{l'} -- evaluated
    pair by pair from the definitions (PAPER.md:1017-1023 expanded)."""
    vs = small_case
    A, B = vs.volumes[2].astype(np.complex128), vs.target.astype(np.complex128)
    HC, HD = 5, 4
    U, _ = ov.vol_basis(ov.vol_kernel_C(B, vs.w), HC)
    V, _ = ov.vol_basis(ov.vol_kernel_D(B, vs.w, vs.L), HD)
    Pr = (U @ U.T) * np.sqrt(np.outer(vs.w, vs.w))
    Pd = V @ V.T
    L, P = vs.L, vs.P
    beta = vs.betas[2]
    d = ov.wigner_d(L, beta)
    F = np.zeros((2 * L + 1, 2 * L + 1), np.complex128)
    for m1 in range(-L, L + 1):
        for m2 in range(-L, L + 1):
            s = 0
            for l in range(max(abs(m1), abs(m2)), L + 1):
                for lp in range(max(abs(m1), abs(m2)), L + 1):
                    x = A[:, lp * lp + lp + m1].conj() @ Pr @ B[:, lp * lp + lp + m2]
                    s += Pd[l, lp] * d[l][m1 + l, m2 + l] * x
            F[m1 + L, m2 + L] = s
    m = np.arange(-L, L + 1)
    a, g = 7, 22
    want = np.sum(np.exp(-2j * np.pi * m[:, None] * a / P) * np.exp(-2j * np.pi * m[None, :] * g / P) * F).real
    X = ov.vol_landscape_rank(A, B, vs.w, U, V, L, [beta], P)[0]
    assert abs(X[a, g] - want) < 1e-10 * np.abs(X).max()
