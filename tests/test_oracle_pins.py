"""Pins for the fp64 oracle (oracle/): each test ties an oracle function to something other than
itself -- a closed form, an identity of the mathematics, a textbook special case, a brute-force
evaluation of the paper's defining integral, or a hand-derived golden fixture.  The comment on each
test names the plausible oracle mistake it would catch.  CPU only (-m "not gpu")."""
import math
import os

import numpy as np
import pytest

from oracle import ref
from synth import make_dataset, radial_grid

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load_gold(name):
    return np.loadtxt(os.path.join(GOLD, name), comments="#")


def _rand_rings(rng, n, R, Q):
    return rng.standard_normal((n, R, Q)) + 1j * rng.standard_normal((n, R, Q))


def _all_pairs(na, nb):
    ia, ib = np.meshgrid(np.arange(na), np.arange(nb), indexing="ij")
    return ia.ravel(), ib.ravel()


def _rand_orth(rng, R):
    q, _ = np.linalg.qr(rng.standard_normal((R, R)))
    return q


# ------------------------------------------------------------------ radial quadrature (harness)
def test_gauss_jacobi_golden_R2():
    """Hand-derived 2-point Gauss-Jacobi(0,1) rule. Catches a wrong (alpha,beta)
    or a wrong k/w mapping in the generator."""
    g = _load_gold("gauss_jacobi_R2.txt")
    k, w = radial_grid(2)
    np.testing.assert_allclose(k, g[:, 3], rtol=0, atol=1e-15)
    np.testing.assert_allclose(w, g[:, 4], rtol=0, atol=1e-15)


@pytest.mark.parametrize("R", [3, 16, 64, 128])
def test_radial_quadrature_exactness(R):
    """sum_r w_r p(k_r) = int_0^K p(k) k dk for deg p <= 2R-1; sum w = K^2/2."""
    k, w = radial_grid(R)
    K = R - 1
    assert abs(w.sum() - K * K / 2) <= 1e-12 * K * K
    for n in [1, 2, R, 2 * R - 1]:
        # int_0^K (k/K)^n k dk / K^2 = 1 / (n + 2)
        approx = (w * (k / K) ** n).sum() / (K * K)
        assert abs(approx - 1.0 / (n + 2)) <= 1e-11 / (n + 2)


# ------------------------------------------------------------------ O1 / O2 / P8
def test_P5_single_ring_closed_form():
    """P5: one-ring content gives X_k = 2 pi w_r e^{-i p gamma_k} (golden).  Catches a missing dpsi,
    a conj on the wrong operand (would flip the phase sign) or a wrong shift direction."""
    g = _load_gold("single_ring_landscape.txt")
    R, Q, p = 3, 8, 2
    w = np.array([0.5, 1.25, 2.0])
    psi = 2 * np.pi * np.arange(Q) / Q
    a = np.zeros((1, R, Q), complex)
    a[0, 1] = np.exp(1j * p * psi)
    X = ref.landscape_full(a, a, w, [0], [0])[0]
    np.testing.assert_allclose(X.real, g[:, 1], atol=1e-13)
    np.testing.assert_allclose(X.imag, g[:, 2], atol=1e-13)


def test_P2_on_grid_rotation_peaks_at_k0():
    """P2: image = template rotated by +gamma_k0 (a[r,j] = b[r,(j-k0)]) peaks at
    k0 with X = ||b||_w^2 exactly (Cauchy-Schwarz).  Catches a reversed shift (peak at Q-k0)."""
    rng = np.random.default_rng(1)
    R, Q = 5, 32
    k, w = radial_grid(R)
    b = _rand_rings(rng, 1, R, Q)
    for k0 in [0, 1, 7, 31]:
        a = np.roll(b, k0, axis=-1)                 # a[j] = b[j - k0]
        X = ref.landscape_full(a, b, w, [0], [0])[0]
        assert ref.argmax_first(X.real) == k0
        nb = (w[:, None] * (2 * np.pi / Q) * np.abs(b[0]) ** 2).sum()
        assert abs(X[k0] - nb) <= 1e-13 * nb


def test_P2_analytic_rotation_generator():
    """P2 via the analytic generator: a noiseless image whose planted angle is on-grid equals the
    template cyclically shifted (A2), and its landscape peaks at that index."""
    d = make_dataset("tiny", complex128=True, noise=False)
    Q = d.Q
    m = 3
    t = int(d.t_true[m])
    k0 = int(round(float(d.gamma[m]) / (2 * np.pi / Q))) % Q
    # re-evaluate that image exactly on-grid by using the planted template with a cyclic shift
    b = d.templates[t].numpy()
    a_shift = np.roll(b, k0, axis=-1)[None]
    X = ref.landscape_full(a_shift, b[None], d.w.numpy(), [0], [0])[0]
    assert ref.argmax_first(X.real) == k0
    # the off-grid analytic image peaks within one sample of its planted angle
    Xo = ref.landscape_full(d.images.numpy()[m:m + 1], b[None], d.w.numpy(), [0], [0])[0]
    kk = ref.argmax_first(Xo.real)
    g = float(d.gamma[m]) / (2 * np.pi / Q)
    assert min(abs(kk - g), Q - abs(kk - g)) <= 1.0


def test_P8_fourier_bessel_form_equals_direct_sum():
    """P8: Eq. image_innerproduct_0 with the direct DFT and ahat = DFT/Q (G1)
    equals O1.  Catches a 2 pi / dpsi normalization slip or the inverse-FFT sign (G3)."""
    rng = np.random.default_rng(2)
    for (R, Q) in [(4, 16), (7, 24), (3, 64)]:
        k, w = radial_grid(R)
        A = _rand_rings(rng, 3, R, Q)
        B = _rand_rings(rng, 2, R, Q)
        ia, ib = _all_pairs(3, 2)
        X1 = ref.landscape_full(A, B, w, ia, ib)
        X8 = ref.landscape_fb(A, B, w, ia, ib)
        assert np.abs(X1 - X8).max() <= 1e-13 * np.abs(X1).max()


def test_P1_full_rank_equals_uncompressed():
    """P1: H = R with ANY orthogonal U reproduces O1.  Catches eta_r = sqrt(w dpsi)
    (would scale by dpsi, G2) or a missing sqrt(w)."""
    rng = np.random.default_rng(3)
    R, Q = 9, 32
    k, w = radial_grid(R)
    A = _rand_rings(rng, 2, R, Q)
    B = _rand_rings(rng, 3, R, Q)
    U = _rand_orth(rng, R)
    ia, ib = _all_pairs(2, 3)
    X1 = ref.landscape_full(A, B, w, ia, ib)
    X2 = ref.landscape_rank(A, B, w, U, ia, ib)
    assert np.abs(X1 - X2).max() <= 1e-13 * np.abs(X1).max()


def test_P3_parseval_over_q():
    """P3: sum_k |X_k|^2 = 4 pi^2 Q sum_q |S_q|^2 with S_q = sum_r w_r conj(ahat) bhat (direct DFT),
    and ring Plancherel sum_j |a_j|^2 dpsi = 2 pi sum_q |ahat_q|^2."""
    rng = np.random.default_rng(4)
    R, Q = 6, 40
    k, w = radial_grid(R)
    A = _rand_rings(rng, 1, R, Q)
    B = _rand_rings(rng, 1, R, Q)
    X = ref.landscape_full(A, B, w, [0], [0])[0]
    j = np.arange(Q)
    F = np.exp(-2j * np.pi * np.outer(j, j) / Q)
    ah = A[0] @ F.T / Q
    bh = B[0] @ F.T / Q
    S = (w[:, None] * np.conj(ah) * bh).sum(0)
    lhs = (np.abs(X) ** 2).sum()
    rhs = 4 * np.pi ** 2 * Q * (np.abs(S) ** 2).sum()
    assert abs(lhs - rhs) <= 1e-12 * rhs
    ring = (np.abs(A[0]) ** 2).sum(1) * (2 * np.pi / Q)
    assert np.allclose(ring, 2 * np.pi * (np.abs(ah) ** 2).sum(1), rtol=1e-13)


def test_P4_mean_over_gamma():
    """P4: (1/Q) sum_k X_k = 2 pi sum_r w_r conj(abar_r) bbar_r (ring means)."""
    rng = np.random.default_rng(5)
    R, Q = 4, 16
    k, w = radial_grid(R)
    A = _rand_rings(rng, 1, R, Q)
    B = _rand_rings(rng, 1, R, Q)
    X = ref.landscape_full(A, B, w, [0], [0])[0]
    rhs = 2 * np.pi * (w * np.conj(A[0].mean(1)) * B[0].mean(1)).sum()
    assert abs(X.mean() - rhs) <= 1e-13 * abs(X).max()


def test_P6_conjugate_symmetry():
    """P6: X(gamma; A, B) = conj X(-gamma; B, A).  Catches conj applied to the shifted operand."""
    rng = np.random.default_rng(6)
    R, Q = 5, 16
    k, w = radial_grid(R)
    A = _rand_rings(rng, 1, R, Q)
    B = _rand_rings(rng, 1, R, Q)
    Xab = ref.landscape_full(A, B, w, [0], [0])[0]
    Xba = ref.landscape_full(B, A, w, [0], [0])[0]
    minus = (-np.arange(Q)) % Q
    assert np.abs(Xab - np.conj(Xba[minus])).max() <= 1e-13 * np.abs(Xab).max()


def test_P11_hermitian_data_gives_real_landscape():
    """P11: noiseless templates are Fourier transforms of real functions, so X is real
    (PAPER.md:410-411 conjugacy); Im X <= 1e-13 max|X|."""
    d = make_dataset("tiny", complex128=True, noise=False)
    B = d.templates.numpy()
    ia, ib = _all_pairs(B.shape[0], B.shape[0])
    X = ref.landscape_full(B, B, d.w.numpy(), ia, ib)
    assert np.abs(X.imag).max() <= 1e-13 * np.abs(X).max()


def test_P10_whole_tiny_config_brute_force():
    """P10: whole Tiny config: O1, O2 at H = R (oracle basis) and P8 agree on all 64 pairs."""
    d = make_dataset("tiny")
    A, B, w = d.images.numpy(), d.templates.numpy(), d.w.numpy()
    ia, ib = _all_pairs(8, 8)
    X1 = ref.landscape_full(A, B, w, ia, ib)
    U, lam = ref.basis(ref.kernel_C(B, w), d.R)
    X2 = ref.landscape_rank(A, B, w, U, ia, ib)
    X8 = ref.landscape_fb(A, B, w, ia, ib)
    s = np.abs(X1).max()
    assert np.abs(X1 - X2).max() <= 1e-12 * s
    assert np.abs(X1 - X8).max() <= 1e-12 * s


def test_rank_landscape_depends_only_on_projector():
    """O2 depends on U only through P = U U^T: rotating the basis inside its span changes nothing."""
    rng = np.random.default_rng(7)
    R, Q, H = 8, 16, 3
    k, w = radial_grid(R)
    A = _rand_rings(rng, 2, R, Q)
    B = _rand_rings(rng, 2, R, Q)
    U = _rand_orth(rng, R)[:, :H]
    Rh = _rand_orth(rng, H)
    ia, ib = _all_pairs(2, 2)
    X = ref.landscape_rank(A, B, w, U, ia, ib)
    Y = ref.landscape_rank(A, B, w, U @ Rh, ia, ib)
    assert np.abs(X - Y).max() <= 1e-13 * np.abs(X).max()


# ------------------------------------------------------------------ O3 kernel / basis
def test_kernel_golden_single_frequency_rings():
    """O3 on single-frequency rings (golden): catches including q = 0 (ring 2 would be nonzero),
    using w instead of sqrt(w) sqrt(w') off the diagonal, or a 1/Q^2 normalization slip."""
    g = _load_gold("two_ring_kernel.txt")
    R, Q = 3, 16
    w = np.array([1.0, 2.0, 3.0])
    c = np.array([1 + 1j, 2.0, 0.5j])
    p = np.array([3, 3, 0])
    psi = 2 * np.pi * np.arange(Q) / Q
    b = (c[:, None] * np.exp(1j * p[:, None] * psi[None, :]))[None]
    np.testing.assert_allclose(ref.kernel_C(b, w), g, atol=1e-14)


def test_kernel_equals_brute_force_rotation_average():
    """Eq. Image_single_kern brute force: average over on-grid gamma, gamma' of
    sum_q [R_g b - R_g' b]^dagger [R_g b' - R_g' b'] dpsi, weights sqrt(w_r w_r'), equals C up to
    one positive constant.  Catches a kernel that forgets the q = 0 exclusion (:665)."""
    rng = np.random.default_rng(8)
    R, Q, T = 4, 12, 3
    k, w = radial_grid(R)
    Bt = _rand_rings(rng, T, R, Q) + 3.0            # strong ring means (q = 0 content)
    brute = np.zeros((R, R))
    for t in range(T):
        x = np.sqrt(w)[:, None] * Bt[t]
        for g in range(Q):
            for gp in range(Q):
                d = np.roll(x, g, axis=1) - np.roll(x, gp, axis=1)
                brute += (np.conj(d) @ d.T).real
    brute /= T
    C = ref.kernel_C(Bt, w)
    scale = brute.trace() / C.trace()
    assert scale > 0
    assert np.abs(brute - scale * C).max() <= 1e-10 * np.abs(brute).max()


def test_P9_kernel_symmetric_psd_rotation_invariant():
    """P9: C symmetric PSD; invariant under rotating any template (phase cancellation, SPEC-style
    invariant); trace = sum of eigenvalues."""
    d = make_dataset("tiny", complex128=True, noise=False)
    B, w = d.templates.numpy(), d.w.numpy()
    C = ref.kernel_C(B, w)
    assert np.abs(C - C.T).max() == 0.0
    U, lam = ref.basis(C, d.R)
    assert lam.min() >= -1e-12 * lam.max()
    assert abs(lam.sum() - np.trace(C)) <= 1e-12 * abs(np.trace(C))
    Br = B.copy()
    Br[2] = np.roll(Br[2], 5, axis=-1)
    Br[5] = np.roll(Br[5], 17, axis=-1)
    assert np.abs(ref.kernel_C(Br, w) - C).max() <= 1e-13 * np.abs(C).max()
    res = np.linalg.norm(C @ U - U * lam[None, :])
    assert res <= 1e-12 * lam[0]


def test_P7_truncation_bounded_by_eigenvalues():
    """P7 (i) Eckart-Young: sum_t ||(I-P_H) B'_t||^2 over q != 0 = T sum_{h>H} lambda_h;
    (ii) per pair max_k |dX_k - dX^(q=0)| <= 2 pi ||(I-P)A'||_F ||(I-P)B'||_F (q != 0 norms).
    Catches a kernel with the wrong weights or with q = 0 included."""
    d = make_dataset("tiny")
    A, B, w = d.images.numpy(), d.templates.numpy(), d.w.numpy()
    T, R, Q = B.shape
    C = ref.kernel_C(B, w)
    for H in [1, 2, 4, 8]:
        U, lam = ref.basis(C, H)
        P = ref.projector(U)
        Bp = np.sqrt(w)[None, :, None] * ref.fb_coefficients(B)
        resid = np.einsum("rs,tsq->trq", np.eye(R) - P, Bp)[:, :, 1:]
        lhs = (np.abs(resid) ** 2).sum()
        rhs = T * lam[H:].sum()
        assert abs(lhs - rhs) <= 1e-10 * max(rhs, 1e-300) + 1e-12 * lam[0]
        ia, ib = _all_pairs(A.shape[0], T)
        Xf = ref.landscape_full(A, B, w, ia, ib)
        Xh = ref.landscape_rank(A, B, w, U, ia, ib)
        Ap = np.sqrt(w)[None, :, None] * ref.fb_coefficients(A)
        ra = np.einsum("rs,tsq->trq", np.eye(R) - P, Ap)
        rb = np.einsum("rs,tsq->trq", np.eye(R) - P, Bp)
        dq0 = 2 * np.pi * (np.conj(ra[ia, :, 0]) * rb[ib, :, 0]).sum(1)
        lhs2 = np.abs((Xf - Xh) - dq0[:, None]).max(1)
        na = np.sqrt((np.abs(ra[:, :, 1:]) ** 2).sum((1, 2)))
        nb = np.sqrt((np.abs(rb[:, :, 1:]) ** 2).sum((1, 2)))
        bound = 2 * np.pi * na[ia] * nb[ib]
        assert np.all(lhs2 <= bound * (1 + 1e-9) + 1e-12 * np.abs(Xf).max())


# ------------------------------------------------------------------ O4 / O5
def test_O4_reductions_tie_breaks():
    x = np.array([[1.0, 3.0, 3.0, 2.0], [5.0, 5.0, 5.0, 5.0]])
    assert list(ref.argmax_first(x)) == [1, 0]
    assert list(ref.top2_gap(np.array([[1.0, 4.0, 2.5]]))) == [1.5]
    Xre = np.array([[1.0, 7.0], [7.0, 0.0]])            # tie between (t0,k1) and (t1,k0)
    assert ref.per_image_winner(Xre) == (7.0, 0, 1)
    assert bool(ref.near_tie_ok(np.array([1.0, 2.0, 1.999]), np.array(2), 0.01))
    assert not bool(ref.near_tie_ok(np.array([1.0, 2.0, 1.9]), np.array(2), 0.01))


def test_O5_metrics_identities():
    """Frobenius / correlation / backward-error f identities."""
    rng = np.random.default_rng(9)
    full = rng.standard_normal((5, 16))
    assert ref.rel_frobenius(full, full) == 0.0
    assert abs(ref.rel_frobenius(np.zeros_like(full), full) - 1.0) < 1e-15
    assert abs(ref.rel_frobenius(2 * full, full) - 1.0) < 1e-15
    assert abs(ref.correlation(full, full) - 1.0) < 1e-14
    assert abs(ref.correlation(-full, full) + 1.0) < 1e-14
    assert abs(ref.correlation(3 * full + 7, full) - 1.0) < 1e-14
    assert np.all(ref.backward_fraction(full, full) == 1.0)
    # literal counting loop
    appr = rng.standard_normal((5, 16))
    f = ref.backward_fraction(appr, full)
    for p in range(5):
        ke = int(np.argmax(appr[p]))
        assert f[p] == sum(1 for k in range(16) if full[p, k] <= full[p, ke]) / 16


# ------------------------------------------------------------------ generator (harness)
def test_noise_variance_calibration():
    """Per-node noise variance = sigma_hat^2 / (w_r dpsi) within 2% (G11)."""
    d0 = make_dataset("small", M=32, T=4, noise=False, complex128=True)
    d1 = make_dataset("small", M=32, T=4, noise=True, complex128=True)
    nz = (d1.images - d0.images).numpy()
    Q = d1.Q
    var = (np.abs(nz) ** 2).mean(axis=(0, 2))                 # per ring
    expect = d1.sigma_hat2 / (d1.w.numpy() * 2 * np.pi / Q)
    np.testing.assert_allclose(var, expect, rtol=0.06)       # 4096 samples per ring
    pooled = (np.abs(nz) ** 2 / expect[None, :, None]).mean()
    assert abs(pooled - 1.0) < 0.02                           # 131072 samples
    # SNR definition G11: Pbar / E||noise||_w^2 = SNR
    assert abs(d1.meta["pbar"] / (d1.sigma_hat2 * d1.R * Q) - 0.5) < 1e-12


def test_generator_rotation_is_cyclic_shift():
    """A2: evaluating the analytic slice at psi - 2 pi k0/Q equals the cyclic
    shift of the unrotated samples (to fp64 rounding)."""
    import torch
    from synth.generator import _slice_rows, molecule_centres, view_frames
    k, w = radial_grid(8)
    kt = torch.tensor(k)
    c = torch.tensor(molecule_centres(0, 5))
    e1, e2 = view_frames(0, 2, "random")
    p1 = torch.tensor(e1) @ c.T
    p2 = torch.tensor(e2) @ c.T
    Q, k0 = 32, 5
    b0 = _slice_rows(p1, p2, torch.zeros(2, dtype=torch.float64), kt, Q).numpy()
    b1 = _slice_rows(p1, p2, torch.full((2,), 2 * np.pi * k0 / Q, dtype=torch.float64), kt, Q).numpy()
    assert np.abs(b1 - np.roll(b0, k0, axis=-1)).max() <= 1e-12 * np.abs(b0).max()


# ------------------------------------------------------------------ F1: finer gamma
def test_F1_fine_equals_O2_on_the_coarse_grid():
    """At Q_out = Q the zero-padded evaluation is the plain rank-H landscape (a direct correlation
    sum, O2), and at Q_out = 4Q every 4th sample is.  Catches a wrong frequency sign, a missing
    1/Q or 2 pi, a mis-indexed negative frequency or a doubled Nyquist term."""
    rng = np.random.default_rng(11)
    R, Q, H = 5, 16, 3
    A, B = _rand_rings(rng, 2, R, Q), _rand_rings(rng, 3, R, Q)
    k, w = radial_grid(R)
    U = _rand_orth(rng, R)[:, :H]
    ia, ib = _all_pairs(2, 3)
    X2 = ref.landscape_rank(A, B, w, U, ia, ib).real
    F = ref.landscape_rank_fine(A, B, w, U, ia, ib, Q)
    np.testing.assert_allclose(F, X2, atol=1e-12 * np.abs(X2).max())
    F4 = ref.landscape_rank_fine(A, B, w, U, ia, ib, 4 * Q)
    np.testing.assert_allclose(F4[:, ::4], X2, atol=1e-12 * np.abs(X2).max())


@pytest.mark.parametrize("p", [1, 3, -5])
def test_F1_single_frequency_is_exact_off_grid(p):
    """A single angular frequency p (|p| < Q/2) on one ring has the band-limited landscape
    2 pi w_r cos(p gamma) for EVERY gamma (P5 continued off the grid): the zero-padded samples must
    reproduce it at gamma = 2 pi k / Q_out.  Catches an interpolation that is not the trigonometric
    polynomial of the coefficients (e.g. a missing conjugate-frequency term)."""
    R, Q, r = 4, 16, 2
    k, w = radial_grid(R)
    psi = 2 * np.pi * np.arange(Q) / Q
    a = np.zeros((1, R, Q), complex)
    a[0, r] = np.exp(1j * p * psi)
    U = np.eye(R)
    Qo = 8 * Q
    F = ref.landscape_rank_fine(a, a, w, U, [0], [0], Qo)[0]
    gam = 2 * np.pi * np.arange(Qo) / Qo
    np.testing.assert_allclose(F, 2 * np.pi * w[r] * np.cos(p * gam), atol=1e-12)


def test_F1_nyquist_bin_is_split():
    """Reading G4 for f1: the unpaired bin Q/2 contributes cos(Q gamma/2) S_{Q/2}.  With
    a = (-1)^j and b = i (-1)^j on one ring, S_{Q/2} = i w_r (purely imaginary), so the split gives
    Re X = 0 at every gamma (the one-sided '+Q/2' or '-Q/2' readings would give -+2 pi w_r sin(Q gamma/2))."""
    R, Q, r = 3, 8, 1
    k, w = radial_grid(R)
    alt = (-1.0) ** np.arange(Q)
    a = np.zeros((1, R, Q), complex)
    b = np.zeros((1, R, Q), complex)
    a[0, r] = alt
    b[0, r] = 1j * alt
    F = ref.landscape_rank_fine(a, b, w, np.eye(R), [0], [0], 4 * Q)[0]
    np.testing.assert_allclose(F, 0.0, atol=1e-13)
    # and a real Nyquist ring gives 2 pi w_r cos(Q gamma / 2)
    F2 = ref.landscape_rank_fine(a, a, w, np.eye(R), [0], [0], 4 * Q)[0]
    gam = 2 * np.pi * np.arange(4 * Q) / (4 * Q)
    np.testing.assert_allclose(F2, 2 * np.pi * w[r] * np.cos(Q / 2 * gam), atol=1e-12)


def test_F1_argmax_refine_spec_examples():
    """SPEC.md argmax_refine examples: unique max at index 5 of 98 with symmetric neighbours ->
    2 pi 5/98; constant landscape -> 0 (smallest index, zero curvature); samples of a parabola with
    its vertex between grid points -> the analytic vertex (exact for a parabola); wrap-around at k=0."""
    x = np.zeros(98)
    x[4], x[5], x[6] = 1.0, 2.0, 1.0
    assert abs(ref.argmax_refine(x) - 2 * np.pi * 5 / 98) < 1e-15
    assert ref.argmax_refine(np.full(17, 3.0)) == 0.0
    Q, v = 64, 20.3
    kk = np.arange(Q)
    par = 5.0 - (kk - v) ** 2
    assert abs(ref.argmax_refine(par) - 2 * np.pi * v / Q) < 1e-12
    cyc = np.zeros(Q)
    cyc[0], cyc[1], cyc[-1] = 4.0, 1.0, 3.0                     # vertex left of 0 -> wraps near 2 pi
    g = ref.argmax_refine(cyc)
    d = (3.0 - 1.0) / (2 * (3.0 - 8.0 + 1.0))
    assert abs(g - np.mod(2 * np.pi * d / Q, 2 * np.pi)) < 1e-12


# ------------------------------------------------------------------ F2: translations
def test_F2_translate_is_the_shift_theorem_of_the_analytic_templates():
    """translate() (reading G15) against the generator's analytic transform: moving every atom of a
    slice by (dx, dy) must equal ramping the unmoved slice.  Catches a sign error in the ramp (it
    would move the atoms the other way), swapped cos/sin or a missing k_r."""
    import torch
    from synth.generator import _slice_rows
    R, Q = 6, 32
    k, w = radial_grid(R)
    rng = np.random.default_rng(5)
    p1 = torch.tensor(rng.uniform(-0.3, 0.3, (1, 7)))
    p2 = torch.tensor(rng.uniform(-0.3, 0.3, (1, 7)))
    kt = torch.tensor(k)
    g0 = torch.zeros(1, dtype=torch.float64)
    base = _slice_rows(p1, p2, g0, kt, Q).numpy()
    shifts = np.array([[0.02, -0.03], [-0.05, 0.0], [0.0, 0.0]])
    tr = ref.translate(base, k, shifts)
    for s, (dx, dy) in enumerate(shifts):
        moved = _slice_rows(p1 + dx, p2 + dy, g0, kt, Q).numpy()[0]
        np.testing.assert_allclose(tr[s], moved, atol=1e-12 * np.abs(moved).max())


def test_F2_translation_averaged_kernel_reduces_to_O3():
    """With the single shift (0, 0) the translation-averaged kernel is O3's kernel; with shifts the
    kernel stays symmetric PSD and rotation-invariant (each translated template's C contribution is
    invariant to rotating it, P9).  Catches a mis-normalised average over shifts."""
    rng = np.random.default_rng(6)
    R, Q = 5, 16
    k, w = radial_grid(R)
    B = _rand_rings(rng, 4, R, Q)
    C0 = ref.kernel_C(B, w)
    np.testing.assert_allclose(ref.kernel_C(ref.translate(B, k, [[0.0, 0.0]]), w), C0, atol=1e-14 * np.abs(C0).max())
    sh = [[0.01, 0.0], [0.0, -0.02], [0.015, 0.015]]
    Ct = ref.kernel_C(ref.translate(B, k, sh), w)
    assert np.abs(Ct - Ct.T).max() <= 1e-15 * np.abs(Ct).max()
    assert np.linalg.eigvalsh(Ct).min() >= -1e-12 * np.abs(Ct).max()
    # averaging over the 3 shifts == averaging the 3 single-shift kernels
    Cs = sum(ref.kernel_C(ref.translate(B, k, [s]), w) for s in sh) / 3
    np.testing.assert_allclose(Ct, Cs, atol=1e-13 * np.abs(Ct).max())


# ------------------------------------------------------------------ F3: per-CTF-group bases
def test_F3_ctf_group_kernel_is_diagonally_scaled():
    """For targets multiplied ring-wise by a radial CTF c(k_r), O3's kernel is diag(c) C diag(c):
    every term of C is bilinear in one ring r and one ring r'.  Catches a CTF applied to the weights
    instead of the rings (c^2 on the diagonal only) or a transposed scaling."""
    from synth import toy_ctf
    rng = np.random.default_rng(8)
    R, Q = 6, 16
    k, w = radial_grid(R)
    B = _rand_rings(rng, 5, R, Q)
    c = toy_ctf(k, 0.05)
    assert np.all(np.abs(c) > 1e-3)                      # not degenerate at these k
    C = ref.kernel_C(B, w)
    Cg = ref.kernel_C(B * c[None, :, None], w)
    np.testing.assert_allclose(Cg, c[:, None] * C * c[None, :], atol=1e-13 * np.abs(Cg).max())


def test_F3_library_ctf_basis_matches_oracle(lib_built=None):
    """Host entry rsvd_eigen_basis_ctf (no GPU): its U is the oracle basis of the CTF-corrected
    targets' kernel (projector agreement), and U_tmpl = diag(c) U."""
    from synth import toy_ctf
    from paper_2202_07235_b200 import api, build
    build.build()
    rng = np.random.default_rng(9)
    R, Q, H = 8, 16, 4
    k, w = radial_grid(R)
    B = _rand_rings(rng, 40, R, Q)
    c = toy_ctf(k, 0.05)
    U, Ut, lam = api.eigen_basis_ctf(ref.kernel_C(B, w), c, H)
    Ur, lr = ref.basis(ref.kernel_C(B * c[None, :, None], w), H)
    assert np.abs(lam - lr).max() <= 1e-12 * lr[0]
    assert np.linalg.norm(U @ U.T - Ur @ Ur.T, 2) <= 1e-9 / ((lr[H - 1] - lr[H]) / lr[0])
    np.testing.assert_allclose(Ut, c[:, None] * U, rtol=0, atol=1e-15)


# ------------------------------------------------------------------------------ T1 (row f2, closed form)
def _slices_analytic(atoms, k, Q, views, shifts, sig_a):
    """Central slices of sum_a exp(-sig^2 k^2/2) exp(-i kvec . c_a) on the polar grid, viewing direction
    v, translated in-plane by (dx, dy) (Fourier shift theorem), evaluated directly (test helper)."""
    psi = 2 * np.pi * np.arange(Q) / Q
    out = np.empty((len(views), len(k), Q), np.complex128)
    for i, (v, (dx, dy)) in enumerate(zip(views, shifts)):
        v = v / np.linalg.norm(v)
        a = np.cross(v, [0.3, 0.5, 0.8])
        a /= np.linalg.norm(a)
        b = np.cross(v, a)
        dirs = np.cos(psi)[:, None] * a + np.sin(psi)[:, None] * b
        kv = k[:, None, None] * dirs[None]
        F = np.exp(-0.5 * sig_a ** 2 * k ** 2)[:, None] * np.exp(-1j * (kv @ atoms.T)).sum(-1)
        out[i] = F * np.exp(-1j * k[:, None] * (dx * np.cos(psi) + dy * np.sin(psi))[None])
    return out


def test_T1_E_minus_is_a_gaussian():
    """The printed E-(k) (modified Bessel functions of order -+1/2) equals exp(-k^2 sigma^2 / 2):
    I_{-1/2}(x) - I_{1/2}(x) = sqrt(2/(pi x)) e^{-x} (textbook closed forms of the half-order I)."""
    k = np.linspace(0.0, 60.0, 41)
    for sig in [0.005, 0.02, 0.05]:
        assert np.allclose(ref.E_minus(k, sig), np.exp(-0.5 * (k * sig) ** 2), rtol=1e-12, atol=1e-300)
    assert np.array_equal(ref.E_minus(k, 0.0), np.ones_like(k))


def test_T1_E_plus_is_the_translation_average_along_a_ray():
    """E+(k, k') = E_delta[exp(-i (k - k') u . delta)] for an isotropic Gaussian delta (std sigma per
    axis) and any unit u: u . delta ~ N(0, sigma^2), evaluated here by Gauss-Hermite quadrature."""
    x, wq = np.polynomial.hermite_e.hermegauss(80)
    wq = wq / wq.sum()
    k = np.linspace(1.0, 40.0, 9)
    for sig in [0.01, 0.03]:
        avg = np.array([[np.sum(wq * np.exp(-1j * (a - b) * sig * x)) for b in k] for a in k])
        assert np.abs(avg.imag).max() < 1e-14
        assert np.allclose(ref.E_plus(k, k, sig), avg.real, rtol=1e-12, atol=1e-15)


def test_T1_closed_form_against_the_view_average():
    """sigma_d = 0: the O3 kernel of central slices at uniform random views converges (as the views
    are averaged) to (1/4 pi) sum_lm conj(B_lm) B_lm' minus the view average of the ring
    mean, which by Funk-Hecke is (1/4 pi) sum_{even l} P_l(0)^2 sum_m conj(B_lm) B_lm'.  T1 keeps the l = 0
    mean term only (as printed), so T1 plus the even l >= 2 terms (computed here independently) must
    match the Monte-Carlo kernel; the printed form alone misses by the size of those terms (reading T1)."""
    from scipy.special import eval_legendre
    from synth.volumes import ball_points, sh_coefficients
    rng = np.random.default_rng(11)
    atoms = ball_points(rng, 20, 0.3)
    R, Q, L, nt = 12, 64, 30, 3000
    k = np.linspace(2.0, 40.0, R)
    w = np.linspace(0.5, 2.0, R)
    B = sh_coefficients(atoms, k, L, sigma=0.05)
    views = rng.standard_normal((nt, 3))
    C_mc = ref.kernel_C(_slices_analytic(atoms, k, Q, views, np.zeros((nt, 2)), 0.05), w)
    C_t1 = ref.kernel_translated_sh(B, k, w, 0.0) / (4 * np.pi)
    even = np.zeros((R, R))
    for l in range(2, L + 1, 2):
        c = B[:, l * l:(l + 1) * (l + 1)]
        even += eval_legendre(l, 0.0) ** 2 * np.einsum("rm,sm->rs", np.conj(c), c).real
    even *= np.sqrt(np.outer(w, w)) / (4 * np.pi)
    err_exact = np.linalg.norm(C_mc - (C_t1 - even)) / np.linalg.norm(C_mc)
    err_printed = np.linalg.norm(C_mc - C_t1) / np.linalg.norm(C_mc)
    assert err_exact < 0.02                       # Monte-Carlo error ~ 1/sqrt(nt)
    assert err_printed > 3 * err_exact            # the printed mean term is an approximation (reading T1)
