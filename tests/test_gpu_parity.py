"""CUDA path vs the fp64 oracle, element by element (-m gpu).  Every call goes through the C ABI
(librsvd.so via the ctypes binding).  Tolerances: DESIGN.md "Tolerance rules"."""
import numpy as np
import pytest
import torch

from oracle import ref
from synth import make_dataset, radial_grid, sample_pairs
from tests.gpu_helpers import (TOL_FP32, assert_argmax_gated, assert_landscape_close, assert_per_image,
                               cuda, to_np)

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2202_07235_b200.api")


@pytest.fixture(autouse=True, params=["simt", "tc"])
def contraction_path(request):
    """Every parity test runs on both contraction paths (FP32 SIMT and tcgen05 with the error-compensated fp16 hi/lo split)."""
    api.set_path(api.PATH_SIMT if request.param == "simt" else api.PATH_TC)
    yield request.param
    api.set_path(api.PATH_AUTO)


def _gpu_path(images, templates, w, U, H, landscape=True, per_pair=True, per_image=True, work_bytes=None):
    """images/templates: complex64 numpy or torch; w: fp64 [R]; U: fp64 [R, H]."""
    A = cuda(images)
    B = cuda(templates)
    M, R, Q = A.shape
    T = B.shape[0]
    wd, Ud = cuda(w, torch.float64), cuda(U, torch.float64)
    ib = api.compress(A, wd, Ud, api.SIDE_IMAGE)
    tb = api.compress(B, wd, Ud, api.SIDE_TEMPLATE)
    nb = work_bytes or api.align_workspace_bytes(M, T, Q, H)
    work = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
    out = {}
    if landscape:
        out["X"] = to_np(api.align_landscape(ib, M, tb, T, Q, H, work))
    if per_pair:
        v, k = api.align_argmax(ib, M, tb, T, Q, H, api.PER_PAIR, work)
        out["val"], out["k"] = to_np(v), to_np(k)
    if per_image:
        keys = torch.zeros(M, dtype=torch.int64, device="cuda")
        api.winners_reset(keys)
        api.align_argmax(ib, M, tb, T, Q, H, api.PER_IMAGE, work, best_key=keys)
        v, t, k = api.winners_unpack(keys, Q)
        out["img"] = (to_np(v), to_np(t), to_np(k))
    torch.cuda.synchronize()
    return out


def _check_all(out, X_ref, tol=TOL_FP32):
    M, T, Q = X_ref.shape
    tol_abs = tol * np.abs(X_ref).max()
    if "X" in out:
        assert_landscape_close(out["X"], X_ref, tol)
    if "val" in out:
        assert np.abs(out["val"] - X_ref.max(-1)).max() <= tol_abs
        assert_argmax_gated(out["k"].reshape(-1), X_ref.reshape(-1, Q), tol_abs)
    if "img" in out:
        assert_per_image(*out["img"], X_ref, tol_abs)


def _all_pairs(M, T):
    ia, ib = np.meshgrid(np.arange(M), np.arange(T), indexing="ij")
    return ia.ravel(), ib.ravel()


# ------------------------------------------------------------------ Tiny: everything, all pairs
def test_tiny_all_pairs_rank_H_and_full_rank():
    d = make_dataset("tiny")
    A, B, w = to_np(d.images), to_np(d.templates), to_np(d.w)
    M, T, Q, R = A.shape[0], B.shape[0], d.Q, d.R
    ia, ib = _all_pairs(M, T)
    for H in [4, R]:
        U, lam = api.build_basis(cuda(B), w, H)
        X_ref = ref.landscape_rank(A, B, w, U, ia, ib).real.reshape(M, T, Q)
        _check_all(_gpu_path(A, B, w, U, H), X_ref)
    # H = R: the library path reproduces the uncompressed direct sum O1
    X_full = ref.landscape_full(A, B, w, ia, ib).real.reshape(M, T, Q)
    U, _ = api.build_basis(cuda(B), w, R)
    out = _gpu_path(A, B, w, U, R, per_pair=False, per_image=False)
    assert_landscape_close(out["X"], X_full)


def test_basis_parity_and_determinism():
    for name, T in [("tiny", None), ("small", 256)]:
        d = make_dataset(name, T=T, M=8)
        B, w = to_np(d.templates), to_np(d.w)
        R = d.R
        U, lam = api.build_basis(cuda(B), w, R)
        U2, lam2 = api.build_basis(cuda(B), w, R)
        assert np.array_equal(U, U2) and np.array_equal(lam, lam2)        # bitwise reproducible
        C_ref = ref.kernel_C(B, w)
        Ur, lr = ref.basis(C_ref, R)
        assert np.abs(lam - lr).max() <= 1e-12 * lr[0]
        assert np.linalg.norm(C_ref @ U - U * lam[None, :]) <= 1e-12 * lr[0]
        # projector agreement on the non-null eigenspace up to each well-separated gap
        nz = int((lr > 1e-9 * lr[0]).sum())
        for h in range(1, nz):
            relgap = (lr[h - 1] - lr[h]) / lr[0]
            if relgap < 1e-6:
                continue
            P = U[:, :h] @ U[:, :h].T
            Pr = Ur[:, :h] @ Ur[:, :h].T
            assert np.linalg.norm(P - Pr, 2) <= 1e-10 / relgap, (name, h, relgap)


def test_basis_parity_multi_tile():
    """R = 128 (2 x 2 tiles of the partials grid: off-diagonal and diagonal tiles, every warp block of the
    fp64 tensor-core Gram) and R = 96 (a ragged second tile), T not a multiple of the 8-template chunk:
    the same SURVEY.md 8(c) O3 gates against the oracle's C and eigenbasis."""
    for name, T, R_use in [("large", 45, 128), ("medium", 37, 64)]:
        d = make_dataset(name, T=T, M=8)
        B, w = to_np(d.templates), to_np(d.w)
        for R in sorted({R_use, 96 if R_use == 128 else R_use}):
            Bs, ws = np.ascontiguousarray(B[:, :R]), np.ascontiguousarray(w[:R])
            U, lam = api.build_basis(cuda(Bs), ws, 24)
            C_ref = ref.kernel_C(Bs, ws)
            Ur, lr = ref.basis(C_ref, 24)
            assert np.abs(lam - lr).max() <= 1e-12 * lr[0], (name, R)
            assert np.linalg.norm(C_ref @ U - U * lam[None, :24]) <= 1e-12 * lr[0], (name, R)
            for h in range(1, 24):
                relgap = (lr[h - 1] - lr[h]) / lr[0]
                if relgap < 1e-6:
                    continue
                P, Pr = U[:, :h] @ U[:, :h].T, Ur[:, :h] @ Ur[:, :h].T
                assert np.linalg.norm(P - Pr, 2) <= 1e-10 / relgap, (name, R, h, relgap)


def test_device_eigen_solver():
    """rsvd_eigen_basis_device (row a0 without the host round trip) against the oracle's C and eigenbasis at
    the SURVEY.md 8(c) O3 gates, for every ring count of the BASELINE configs (R = 16, 32, 64, 128) and the
    H of each, plus H = R / 2 at R = 128 and a 5-template C (fast-decaying spectrum, clustered near-null
    eigenvalues); the sign rule
    and eigenvalues agree with the host solver; bitwise reproducible; info = 0."""
    cases = [("tiny", None, 4), ("small", 256, 8), ("medium", 48, 16), ("medium", 40, 64), ("large", 45, 24),
             ("large", 45, 64), ("small", 5, 8)]
    for name, T, H in cases:
        d = make_dataset(name, T=T, M=8)
        B, w = to_np(d.templates), to_np(d.w)
        R = d.R
        C = api.kernel_reduce(api.kernel_partials(cuda(B)), B.shape[0], d.Q, cuda(w, torch.float64))
        U, lam, info = api.eigen_basis_device(C, H)
        U2, lam2, info2 = api.eigen_basis_device(C, H)
        torch.cuda.synchronize()
        assert int(info.item()) == 0 and int(info2.item()) == 0, (name, H)
        U, lam = to_np(U), to_np(lam)
        assert np.array_equal(U, to_np(U2)) and np.array_equal(lam, to_np(lam2))      # bitwise reproducible
        Uh, lamh = api.eigen_basis(to_np(C), H)                                         # host solver, same C
        assert np.abs(lam - lamh).max() <= 1e-13 * lamh[0], (name, H)
        C_ref = ref.kernel_C(B, w)
        Ur, lr = ref.basis(C_ref, H)
        assert np.abs(lam - lr).max() <= 1e-12 * lr[0], (name, H)
        assert np.linalg.norm(C_ref @ U - U * lam[None, :H]) <= 1e-12 * lr[0], (name, H)
        assert np.abs(U.T @ U - np.eye(H)).max() <= 1e-12, (name, H)
        for h in range(1, H + 1):
            relgap = (lr[h - 1] - lr[h]) / lr[0] if h < R else 1.0
            if relgap < 1e-6:
                continue
            P, Pr = U[:, :h] @ U[:, :h].T, Ur[:, :h] @ Ur[:, :h].T
            assert np.linalg.norm(P - Pr, 2) <= 1e-10 / relgap, (name, H, h, relgap)
            # well-separated single vectors: same sign rule as the host solver
            gap_below = relgap
            gap_above = (lr[h - 2] - lr[h - 1]) / lr[0] if h >= 2 else 1.0
            if gap_below >= 1e-6 and gap_above >= 1e-6:
                assert float(U[:, h - 1] @ Uh[:, h - 1]) > 0.5, (name, H, h)


def test_device_eigen_solver_edge_shapes():
    """rsvd_eigen_basis_device on shapes the configs never reach: R = 1, 2, 3, 5 (no or one Householder
    step), exactly repeated eigenvalues (a 3-fold and a 4-fold cluster: Gram-Schmidt keeps the cluster
    vectors orthonormal and spanning their eigenspace), a rank-deficient PSD matrix (a null space of
    dimension R - 4), and R = 128 with H = 64.  Reference: numpy eigh (LAPACK) of the same matrix."""
    rng = np.random.default_rng(20220723)

    def check(C, H, tag):
        R = C.shape[0]
        U, lam, info = api.eigen_basis_device(cuda(C, torch.float64), H)
        torch.cuda.synchronize()
        assert int(info.item()) == 0, tag
        U, lam = to_np(U), to_np(lam)
        lr, V = np.linalg.eigh(C)
        lr, V = lr[::-1], V[:, ::-1]
        scale = max(abs(lr[0]), abs(lr[-1]), 1e-300)
        assert np.abs(lam - lr).max() <= 1e-12 * scale, tag
        assert np.linalg.norm(C @ U - U * lam[None, :H]) <= 1e-12 * scale * max(1.0, np.sqrt(R)), tag
        assert np.abs(U.T @ U - np.eye(H)).max() <= 1e-12, tag
        # projector onto each complete cluster of (numerically) equal eigenvalues among the top H
        h = 0
        while h < H:
            g = h
            while g + 1 < R and abs(lr[g + 1] - lr[h]) <= 1e-9 * scale:
                g += 1
            if g < H:
                P, Pr = U[:, h:g + 1] @ U[:, h:g + 1].T, V[:, h:g + 1] @ V[:, h:g + 1].T
                assert np.linalg.norm(P - Pr, 2) <= 1e-9, (tag, h, g)
            h = g + 1

    for R in (1, 2, 3, 5):
        A = rng.standard_normal((R, R + 2))
        check(A @ A.T, R, f"R={R}")
    Qm, _ = np.linalg.qr(rng.standard_normal((16, 16)))
    ev = np.array([5.0, 3.0, 3.0, 3.0, 2.0, 1.0, 1.0, 1.0, 1.0, 0.5, 0.25, 0.2, 0.1, 0.05, 0.02, 0.01])
    check((Qm * ev) @ Qm.T, 10, "clusters")
    A = rng.standard_normal((32, 4))
    check(A @ A.T, 8, "rank 4")
    A = rng.standard_normal((128, 300))
    check(A @ A.T / 300.0, 64, "R=128 H=64")


@pytest.fixture(params=[1, 2, 0], ids=["auto", "mma", "ffma"])
def compress_mode(request):
    """Step 1 kernel choice (rsvd_set_compress_mma): auto, tensor-core projection forced, FFMA2 forced."""
    api.set_compress_mma(request.param)
    yield request.param
    api.set_compress_mma(1)


def test_compress_parity(compress_mode):
    d = make_dataset("small", M=40, T=24)
    A, B, w = to_np(d.images), to_np(d.templates), to_np(d.w)
    for H, rings, side in [(8, A, api.SIDE_IMAGE), (8, B, api.SIDE_TEMPLATE), (12, A, api.SIDE_IMAGE),
                           (24, B, api.SIDE_TEMPLATE), (20, A, api.SIDE_IMAGE)]:
        U, _ = api.build_basis(cuda(B), w, H)         # 4 | H > 8: rows split over groups of 8 rings
        blocks = api.compress(cuda(rings), cuda(w, torch.float64), cuda(U, torch.float64), side)
        got = to_np(api.blocks_unpack(blocks, rings.shape[0], d.Q, H, side))       # [n, Q, H]
        coef = ref.fb_coefficients(rings)                                           # [n, R, Q]
        want = np.einsum("rh,nrq->nqh", U * np.sqrt(w)[:, None], coef)
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err <= 2e-6, err


@pytest.mark.parametrize("Q,R,H,n", [(256, 40, 6, 9), (512, 100, 16, 5), (1024, 24, 12, 3), (512, 128, 32, 4),
                                     (128, 16, 3, 7), (512, 128, 24, 150)])
def test_compress_shapes(Q, R, H, n, compress_mode):
    """Compress (both sides) against the oracle's coefficients on shapes that exercise the tensor-core
    projection's edges: R not a multiple of the 8-ring stage (TMA zero fill), H not a multiple of 4 in
    one epilogue chunk, several chunks, Q = 1024 (four passes), N padded to 16 / 32, more rows than SMs."""
    rng = np.random.default_rng(1000 + Q + R + H)
    rings = (rng.standard_normal((n, R, Q)) + 1j * rng.standard_normal((n, R, Q))).astype(np.complex64)
    rings *= np.exp(rng.uniform(-3, 3, (n, 1, 1))).astype(np.float32)        # rows of very different scale
    U = np.linalg.qr(rng.standard_normal((R, H)))[0]
    w = radial_grid(R)[1]
    coef = ref.fb_coefficients(rings)
    want = np.einsum("rh,nrq->nqh", U * np.sqrt(w)[:, None], coef)
    for side in (api.SIDE_IMAGE, api.SIDE_TEMPLATE):
        args = (cuda(rings), cuda(w, torch.float64), cuda(U, torch.float64), side)
        blocks = api.compress(*args)
        for _ in range(3):                                   # race proxy: repeat runs bitwise identical
            assert torch.equal(api.compress(*args).view(torch.int32), blocks.view(torch.int32))
        got = to_np(api.blocks_unpack(blocks, n, Q, H, side))
        for i in range(n):                                   # gate per row (each row has its own scale)
            err = np.abs(got[i] - want[i]).max() / np.abs(want[i]).max()
            assert err <= 2e-6, (side, i, err)


def test_small_full_argmax_sampled_pairs():
    d = make_dataset("small", device="cuda")
    H = 8
    U, _ = api.build_basis(d.templates, to_np(d.w), H)
    M, T, Q = d.images.shape[0], d.templates.shape[0], d.Q
    out = _gpu_path(d.images, d.templates, to_np(d.w), U, H, landscape=False, per_image=True)
    m, t = sample_pairs("small", M, T, 4096, 1024, to_np(d.t_true))
    A, B, w = to_np(d.images), to_np(d.templates), to_np(d.w)
    X_ref = ref.landscape_rank(A, B, w, U, m, t).real
    tol_abs = TOL_FP32 * np.abs(X_ref).max()
    assert np.abs(out["val"][m, t] - X_ref.max(-1)).max() <= tol_abs
    assert_argmax_gated(out["k"][m, t], X_ref, tol_abs)
    # per-image winners of a few images over all templates
    for mm in [0, 1, 517, 1023]:
        Xi = ref.landscape_rank(A, B, w, U, np.full(T, mm), np.arange(T)).real
        v, tt, kk = (x[mm:mm + 1] for x in out["img"])
        assert_per_image(v, tt, kk, Xi[None], TOL_FP32 * max(np.abs(Xi).max(), np.abs(X_ref).max()))


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("M,T,R,Q,H", [
    (1, 1, 4, 32, 1),          # minimum Q, H = 1, single pair
    (70, 130, 9, 32, 9),       # ragged tiles, H = R, odd R
    (65, 3, 16, 64, 5),        # ragged, tiny T
    (3, 67, 12, 128, 7),
    (2, 5, 8, 1024, 3),        # maximum Q
    (9, 11, 33, 256, 33),      # K = 2H not a multiple of 16
    (20, 30, 24, 512, 12),     # zero-padded k-block
    (17, 40, 40, 256, 20),
    (5, 9, 36, 1024, 32),      # H x Q block too large for one CTA: row split over 4 groups of 8 rings
    (4, 7, 64, 1024, 28),      # split, last group of 4, zero-padded k-block
    (6, 10, 64, 512, 52),      # split at Q = 512 (7 groups)
    (3, 300, 24, 64, 16),
])
def test_edge_shapes_random_rings(M, T, R, Q, H):
    rng = np.random.default_rng(M * 1000 + T)
    A = (rng.standard_normal((M, R, Q)) + 1j * rng.standard_normal((M, R, Q))).astype(np.complex64)
    B = (rng.standard_normal((T, R, Q)) + 1j * rng.standard_normal((T, R, Q))).astype(np.complex64)
    k, w = radial_grid(R)
    U, _ = api.build_basis(cuda(B), w, H)
    ia, ib = _all_pairs(M, T)
    X_ref = ref.landscape_rank(A, B, w, U, ia, ib).real.reshape(M, T, Q)
    _check_all(_gpu_path(A, B, w, U, H), X_ref)


@pytest.mark.parametrize("Q", [32, 64, 128, 256, 512, 1024])
def test_many_items_per_cta_all_modes(Q):
    """Tens of FFT work items per CTA (so every slot of the Step-3 TMA ring is reused many times and
    warp groups drift apart): sampled landscapes against the oracle, and the per-pair / per-image
    argmax outputs against the landscape the same launch configuration produced."""
    M, T, R, H = 600, 300, 16, 4
    rng = np.random.default_rng(Q)
    A = (rng.standard_normal((M, R, Q)) + 1j * rng.standard_normal((M, R, Q))).astype(np.complex64)
    B = (rng.standard_normal((T, R, Q)) + 1j * rng.standard_normal((T, R, Q))).astype(np.complex64)
    k, w = radial_grid(R)
    U, _ = api.build_basis(cuda(B), w, H)
    out = _gpu_path(A, B, w, U, H)
    m = rng.integers(0, M, 160)
    t = rng.integers(0, T, 160)
    X_ref = ref.landscape_rank(A, B, w, U, m, t).real
    tol_abs = TOL_FP32 * np.abs(X_ref).max()
    assert np.abs(out["X"][m, t] - X_ref).max() <= tol_abs
    assert np.abs(out["val"][m, t] - X_ref.max(-1)).max() <= tol_abs
    assert_argmax_gated(out["k"][m, t], X_ref, tol_abs)
    # every pair: argmax outputs agree with the landscape kernel's own values
    X = out["X"]
    assert np.abs(out["val"] - X.max(-1)).max() <= 1e-6 * np.abs(X).max()
    kk = out["k"]
    assert np.all(X[np.arange(M)[:, None], np.arange(T)[None, :], kk] >= X.max(-1) - 1e-6 * np.abs(X).max())
    v, ti, ki = out["img"]
    assert np.abs(v - out["val"].max(1)).max() <= 1e-6 * np.abs(X).max()
    assert np.all(out["val"][np.arange(M), ti] == v)


def test_small_workspace_many_chunks():
    """Minimum workspace forces many small chunks: results identical to one big chunk."""
    d = make_dataset("small", M=200, T=150)
    A, B, w = to_np(d.images), to_np(d.templates), to_np(d.w)
    U, _ = api.build_basis(cuda(B), w, 8)
    big = _gpu_path(A, B, w, U, 8, landscape=True)
    small = _gpu_path(A, B, w, U, 8, landscape=True, work_bytes=api.align_min_workspace_bytes(d.Q))
    for key in ["X", "val", "k"]:
        assert np.array_equal(big[key], small[key])
    for a, b in zip(big["img"], small["img"]):
        assert np.array_equal(a, b)


def test_ties_smallest_index():
    """Constant landscapes (all-zero rings): per-pair k = 0, per-image (t, k) = (0, 0)."""
    M, T, R, Q, H = 3, 5, 4, 64, 2
    A = np.zeros((M, R, Q), np.complex64)
    B = np.zeros((T, R, Q), np.complex64)
    k, w = radial_grid(R)
    U = np.eye(R)[:, :H]
    out = _gpu_path(A, B, w, U, H)
    assert np.all(out["k"] == 0) and np.all(out["val"] == 0)
    v, t, kk = out["img"]
    assert np.all(t == 0) and np.all(kk == 0)


def test_on_grid_rotation_recovered_exactly():
    """P2 through the library: image = template cyclically shifted by k0 -> argmax k0 (H = R)."""
    rng = np.random.default_rng(11)
    R, Q = 8, 128
    B = (rng.standard_normal((4, R, Q)) + 1j * rng.standard_normal((4, R, Q))).astype(np.complex64)
    shifts = np.array([0, 1, 77, 127])
    A = np.stack([np.roll(B[i], s, axis=-1) for i, s in enumerate(shifts)])
    k, w = radial_grid(R)
    U, _ = api.build_basis(cuda(B), w, R)
    out = _gpu_path(A, B, w, U, R, landscape=False)
    assert list(np.diag(out["k"])) == list(shifts)
    v, t, kk = out["img"]
    assert list(t) == [0, 1, 2, 3] and list(kk) == list(shifts)


def test_empty_problems_are_noops():
    R, Q, H = 4, 64, 2
    k, w = radial_grid(R)
    wd, Ud = cuda(w, torch.float64), cuda(np.eye(R)[:, :H], torch.float64)
    blocks = torch.empty(16, dtype=torch.float32, device="cuda")
    lib = api._lib.lib()
    assert lib.rsvd_compress(blocks.data_ptr(), 0, R, Q, wd.data_ptr(), Ud.data_ptr(), H, 0,
                             blocks.data_ptr(), None) == 0
    work = torch.empty(api.align_min_workspace_bytes(Q) // 4, dtype=torch.float32, device="cuda")
    assert lib.rsvd_align_argmax(blocks.data_ptr(), 0, blocks.data_ptr(), 5, 0, Q, H, 0, work.data_ptr(),
                                 work.numel() * 4, None, None, None, None) == 0


def test_error_paths():
    R, Q, H = 4, 64, 2
    k, w = radial_grid(R)
    lib = api._lib.lib()
    rings = torch.zeros((2, R, Q), dtype=torch.complex64, device="cuda")
    wd, Ud = cuda(w, torch.float64), cuda(np.eye(R)[:, :H], torch.float64)
    blocks = torch.empty(api.block_bytes(2, Q, H, api.SIDE_TEMPLATE) // 4, dtype=torch.float32, device="cuda")
    p = rings.data_ptr()
    assert lib.rsvd_compress(p, 2, R, 48, wd.data_ptr(), Ud.data_ptr(), H, 0, blocks.data_ptr(), None) == 2
    assert lib.rsvd_compress(p, 2, R, 16, wd.data_ptr(), Ud.data_ptr(), H, 0, blocks.data_ptr(), None) == 2
    assert lib.rsvd_compress(p, 2, R, Q, wd.data_ptr(), Ud.data_ptr(), R + 1, 0, blocks.data_ptr(), None) == 2
    assert lib.rsvd_compress(p, -1, R, Q, wd.data_ptr(), Ud.data_ptr(), H, 0, blocks.data_ptr(), None) == 1
    assert lib.rsvd_compress(None, 2, R, Q, wd.data_ptr(), Ud.data_ptr(), H, 0, blocks.data_ptr(), None) == 1
    assert lib.rsvd_compress(p + 8, 2, R, Q, wd.data_ptr(), Ud.data_ptr(), H, 0, blocks.data_ptr(), None) == 1
    assert lib.rsvd_compress(p, 2, R, Q, wd.data_ptr(), Ud.data_ptr(), H, 7, blocks.data_ptr(), None) == 1
    bad_w = w.copy()
    bad_w[1] = np.nan
    U = np.zeros((R, H))
    assert lib.rsvd_build_basis(p, 2, R, Q, bad_w.ctypes.data, H, U.ctypes.data, None, None) == 1
    bad_w[1] = -1.0
    assert lib.rsvd_build_basis(p, 2, R, Q, bad_w.ctypes.data, H, U.ctypes.data, None, None) == 1
    work = torch.empty(1024, dtype=torch.float32, device="cuda")
    b = blocks.data_ptr()
    assert lib.rsvd_align_argmax(b, 2, b, 2, 0, Q, H, 0, work.data_ptr(), 4096, b, b, None, None) == 1  # small work
    big = torch.empty(api.align_min_workspace_bytes(Q) // 4, dtype=torch.float32, device="cuda")
    assert lib.rsvd_align_argmax(b, 2, b, 2, 0, Q, H, 0, big.data_ptr(), big.numel() * 4, None, None, None, None) == 1
    assert lib.rsvd_align_argmax(b, 2, b, 2, 0, Q, H, 1, big.data_ptr(), big.numel() * 4, None, None, None, None) == 1
    assert lib.rsvd_align_argmax(b, 2, b, 2, 1 << 30, Q, H, 1, big.data_ptr(), big.numel() * 4, None, None, b,
                                 None) == 2
    assert lib.rsvd_align_argmax(b, 2, b, 2, 0, Q, H, 9, big.data_ptr(), big.numel() * 4, b, b, b, None) == 1
    assert len(lib.rsvd_last_error()) > 0


def test_streamed_host_path_matches_device_path(contraction_path):
    """dist.align_from_host (host->device copies of template / image blocks overlapped with the
    compute) returns exactly the winners of the device-resident path, including ragged blocks."""
    from paper_2202_07235_b200 import dist as pdist
    d = make_dataset("small", M=700, T=300, device="cuda")
    H, Q = 8, d.Q
    w = d.w.contiguous()
    h_img = d.images.cpu().pin_memory()
    h_tmp = d.templates.cpu().pin_memory()
    d_img, d_tmp = torch.empty_like(d.images), torch.empty_like(d.templates)
    (keys, val, t, k), U = pdist.align_from_host(h_img, h_tmp, 300, 0, w, H, d_img, d_tmp, img_block=256,
                                                   tmpl_block=64)
    U2, _ = pdist.basis_from_shards(d.templates, 300, w, H)
    assert np.array_equal(U, U2)
    Ud = cuda(U2, torch.float64)
    ib = api.compress(d.images, w, Ud, api.SIDE_IMAGE)
    tb = api.compress(d.templates, w, Ud, api.SIDE_TEMPLATE)
    work = torch.empty(api.align_workspace_bytes(700, 300, Q, H) // 4, dtype=torch.float32, device="cuda")
    ref_keys = api.align_argmax(ib, 700, tb, 300, Q, H, api.PER_IMAGE, work)
    assert torch.equal(keys, ref_keys)


@pytest.mark.parametrize("Q,p", [(32, 1), (64, 2), (128, 1), (256, 1), (512, 1)])
def test_fine_gamma_landscape_and_refined_argmax(Q, p):
    """Row f1: the landscape on the zero-padded grid Q_out = Q 2^p against the oracle's
    term-by-term evaluation (F1), the per-pair argmax / parabolic-refined angle against the same
    launch's landscape, and per-image winners on the fine grid."""
    M, T, R, H = 70, 45, 12, 5
    rng = np.random.default_rng(Q + p)
    A = (rng.standard_normal((M, R, Q)) + 1j * rng.standard_normal((M, R, Q))).astype(np.complex64)
    B = (rng.standard_normal((T, R, Q)) + 1j * rng.standard_normal((T, R, Q))).astype(np.complex64)
    k, w = radial_grid(R)
    U, _ = api.build_basis(cuda(B), w, H)
    wd, Ud = cuda(w, torch.float64), cuda(U, torch.float64)
    ib = api.compress(cuda(A), wd, Ud, api.SIDE_IMAGE)
    tb = api.compress(cuda(B), wd, Ud, api.SIDE_TEMPLATE)
    Qo = Q << p
    work = torch.empty(api.align_workspace_bytes(M, T, Qo, H) // 4, dtype=torch.float32, device="cuda")
    X = to_np(api.align_landscape_fine(ib, M, tb, T, Q, H, Qo, work))
    m, t = rng.integers(0, M, 120), rng.integers(0, T, 120)
    X_ref = ref.landscape_rank_fine(A, B, w, U, m, t, Qo)
    tol_abs = TOL_FP32 * np.abs(X_ref).max()
    assert np.abs(X[m, t] - X_ref).max() <= tol_abs
    # the coarse landscape is the fine one's every 2^p-th sample
    Xc = to_np(api.align_landscape(ib, M, tb, T, Q, H, work))
    assert np.abs(X[:, :, ::(1 << p)] - Xc).max() <= 2 * TOL_FP32 * np.abs(Xc).max()
    val, kk, gam = (to_np(x) for x in api.align_argmax_fine(ib, M, tb, T, Q, H, Qo, api.PER_PAIR, work))
    assert np.abs(val - X.max(-1)).max() <= 1e-6 * np.abs(X).max()
    assert_argmax_gated(kk[m, t], X_ref, tol_abs)
    same = kk == ref.argmax_first(X)                          # where the launch agrees with its landscape
    assert same.mean() > 0.95
    g_ref = ref.argmax_refine(X)
    dg = np.abs(np.angle(np.exp(1j * (gam - g_ref))))
    assert dg[same].max() <= 1e-3 * 2 * np.pi / Qo + 1e-5
    assert np.all((gam >= 0) & (gam < 2 * np.pi))
    keys = api.align_argmax_fine(ib, M, tb, T, Q, H, Qo, api.PER_IMAGE, work)
    v, ti, ki = (to_np(x) for x in api.winners_unpack(keys, Qo))
    assert np.abs(v - val.max(1)).max() <= 1e-6 * np.abs(X).max()
    assert np.all(val[np.arange(M), ti] == v)


def test_translations_fused_into_compress():
    """Row f2: rsvd_compress_translated builds the S phase-ramped copies of each base ring in the
    compress kernel.  Its coefficients match compressing the materialised copies, and the alignment
    of the fused blocks matches the oracle on rings translated in fp64 by the test itself
    (a exp(-i k_r (dx cos psi + dy sin psi)), reading G15)."""
    d = make_dataset("translations", M=20, T=40, device="cuda")
    H, Q, R = 16, d.Q, d.R
    S = 9
    base = d.images[4::S].contiguous()                     # shift 4 is (0, 0): the base images
    shifts = d.shift[:S].contiguous()
    w, kr = d.w.contiguous(), d.k.contiguous()
    U, _ = api.build_basis(d.templates, to_np(w), H)
    Ud = cuda(U, torch.float64)
    fused = api.compress_translated(base, w, kr, Ud, shifts, api.SIDE_IMAGE)
    mat = api.compress(d.images, w, Ud, api.SIDE_IMAGE)
    M = base.shape[0] * S
    cf = to_np(api.blocks_unpack(fused, M, Q, H, api.SIDE_IMAGE))
    cm = to_np(api.blocks_unpack(mat, M, Q, H, api.SIDE_IMAGE))
    assert np.abs(cf - cm).max() <= 2e-6 * np.abs(cm).max()
    tb = api.compress(d.templates, w, Ud, api.SIDE_TEMPLATE)
    T = d.templates.shape[0]
    work = torch.empty(api.align_workspace_bytes(M, T, Q, H) // 4, dtype=torch.float32, device="cuda")
    val, k = (to_np(x) for x in api.align_argmax(fused, M, tb, T, Q, H, api.PER_PAIR, work))
    # oracle: translate the base rings in fp64 here, then the rank-H direct sum
    psi = 2 * np.pi * np.arange(Q) / Q
    sh, kk = to_np(shifts), to_np(kr)
    b64 = to_np(base).astype(np.complex128)
    A = np.stack([b64[b] * np.exp(-1j * kk[:, None] * (sh[s, 0] * np.cos(psi) + sh[s, 1] * np.sin(psi))[None, :])
                  for b in range(base.shape[0]) for s in range(S)])
    rng = np.random.default_rng(3)
    m, t = rng.integers(0, M, 150), rng.integers(0, T, 150)
    X_ref = ref.landscape_rank(A, to_np(d.templates), to_np(w), U, m, t).real
    tol_abs = TOL_FP32 * np.abs(X_ref).max()
    assert np.abs(val[m, t] - X_ref.max(-1)).max() <= tol_abs
    assert_argmax_gated(k[m, t], X_ref, tol_abs)


def test_translation_averaged_basis():
    """Row f2: rsvd_build_basis_translated (fp64 ramps on the device, every template's S translated
    copies in the kernel partials) against the oracle's kernel of the fp64-translated templates."""
    d = make_dataset("small", T=96, M=8)
    B, w, k = to_np(d.templates), to_np(d.w), to_np(d.k)
    R = d.R
    shifts = np.array([[0.0, 0.0], [0.03, 0.0], [0.0, -0.03], [0.02, 0.02]])
    U, lam = api.build_basis_translated(cuda(B), w, k, shifts, R)
    C_ref = ref.kernel_C(ref.translate(B, k, shifts), w)
    Ur, lr = ref.basis(C_ref, R)
    assert np.abs(lam - lr).max() <= 1e-12 * lr[0]
    assert np.linalg.norm(C_ref @ U - U * lam[None, :]) <= 1e-12 * lr[0]
    nz = int((lr > 1e-9 * lr[0]).sum())
    for h in range(1, nz):
        relgap = (lr[h - 1] - lr[h]) / lr[0]
        if relgap < 1e-6:
            continue
        P = U[:, :h] @ U[:, :h].T
        Pr = Ur[:, :h] @ Ur[:, :h].T
        assert np.linalg.norm(P - Pr, 2) <= 1e-9 / relgap, (h, relgap)
    # shifts change the kernel (the test is not vacuous)
    U0, lam0 = api.build_basis(cuda(B), w, R)
    assert np.abs(lam0 - lam).max() > 1e-6 * lam0[0]


def test_ctf_group_bases_end_to_end():
    """Row f3: two CTF groups sharing one kernel-partials pass.  Group g's images carry c_g; its
    targets are the raw templates compressed with diag(c_g) U_g; the alignment equals the oracle's
    rank-H landscape of (images_g, c_g * templates) through U_g."""
    from synth import toy_ctf
    d = make_dataset("small", M=24, T=60, device="cuda")
    H, Q, R = 8, d.Q, d.R
    k = to_np(d.k)
    ctfs = np.stack([toy_ctf(k, 0.02), toy_ctf(k, 0.035)])
    w = d.w.contiguous()
    bases = api.ctf_group_bases(d.templates, w, ctfs, H)
    T = d.templates.shape[0]
    work = torch.empty(api.align_workspace_bytes(24, T, Q, H) // 4, dtype=torch.float32, device="cuda")
    B = to_np(d.templates)
    for g, (U, Ut, lam) in enumerate(bases):
        c = torch.tensor(ctfs[g], dtype=torch.complex64, device="cuda")
        imgs = (d.images * c[None, :, None]).contiguous()
        ib = api.compress(imgs, w, cuda(U, torch.float64), api.SIDE_IMAGE)
        tb = api.compress(d.templates, w, cuda(Ut, torch.float64), api.SIDE_TEMPLATE)
        X = to_np(api.align_landscape(ib, 24, tb, T, Q, H, work))
        rng = np.random.default_rng(g)
        m, t = rng.integers(0, 24, 80), rng.integers(0, T, 80)
        Bg = (B.astype(np.complex128) * ctfs[g][None, :, None])
        X_ref = ref.landscape_rank(to_np(imgs), Bg, to_np(w), U, m, t).real
        assert np.abs(X[m, t] - X_ref).max() <= TOL_FP32 * np.abs(X_ref).max()


def test_ctf_grouped_align_three_groups():
    """Row f3, rsvd_align_argmax_grouped: three CTF groups (images of group g carry c_g; targets are the
    raw templates compressed with diag(c_g) U_g) in ONE call, PER_PAIR and PER_IMAGE, against the
    oracle's rank-H landscape of (images_g, c_g * templates) through U_g on all pairs, and bitwise
    equal to three separate rsvd_align_argmax calls."""
    from synth import toy_ctf
    G, Mg = 3, 40
    d = make_dataset("small", M=G * Mg, T=72, device="cuda")
    H, Q = 8, d.Q
    k = to_np(d.k)
    ctfs = np.stack([toy_ctf(k, lam) for lam in (0.015, 0.025, 0.04)])
    w = d.w.contiguous()
    bases = api.ctf_group_bases(d.templates, w, ctfs, H)
    T = d.templates.shape[0]
    work = torch.empty(api.align_workspace_bytes(Mg, T, Q, H) // 4, dtype=torch.float32, device="cuda")
    B = to_np(d.templates)
    groups, refs = [], []
    for g, (U, Ut, lam) in enumerate(bases):
        c = torch.tensor(ctfs[g], dtype=torch.complex64, device="cuda")
        imgs = (d.images[g * Mg:(g + 1) * Mg] * c[None, :, None]).contiguous()
        ib = api.compress(imgs, w, cuda(U, torch.float64), api.SIDE_IMAGE)
        tb = api.compress(d.templates, w, cuda(Ut, torch.float64), api.SIDE_TEMPLATE)
        groups.append(dict(img_blocks=ib, M=Mg, tmpl_blocks=tb, T=T, t_offset=g * T))
        ia, it = _all_pairs(Mg, T)
        Bg = B.astype(np.complex128) * ctfs[g][None, :, None]
        refs.append(ref.landscape_rank(to_np(imgs), Bg, to_np(w), U, ia, it).real.reshape(Mg, T, Q))
    outs = api.align_argmax_grouped(groups, Q, H, api.PER_PAIR, work)
    keys = api.align_argmax_grouped(groups, Q, H, api.PER_IMAGE, work)
    for g, ((val, kk), key, X_ref) in enumerate(zip(outs, keys, refs)):
        tol_abs = TOL_FP32 * np.abs(X_ref).max()
        assert np.abs(to_np(val) - X_ref.max(-1)).max() <= tol_abs
        assert_argmax_gated(to_np(kk).ravel(), X_ref.reshape(-1, Q), tol_abs)
        v1, k1 = api.align_argmax(groups[g]["img_blocks"], Mg, groups[g]["tmpl_blocks"], T, Q, H, api.PER_PAIR, work)
        assert torch.equal(v1, val) and torch.equal(k1, kk)
        vi, ti, ki = (to_np(x) for x in api.winners_unpack(key, Q))
        assert np.all((ti >= g * T) & (ti < (g + 1) * T))
        assert_per_image(vi, ti - g * T, ki, X_ref, tol_abs)


def test_closed_form_translation_kernel_matches_oracle():
    """Row f2, closed form: rsvd_kernel_translated_sh vs the oracle T1 at several
    translation widths, then the basis from it through rsvd_eigen_basis vs the oracle's on the
    leading (well-separated) eigenspace."""
    from synth.volumes import ball_points, sh_coefficients
    from synth import radial_grid
    rng = np.random.default_rng(21)
    atoms = ball_points(rng, 40, 0.3)
    R, L = 32, 40
    kk, ww = radial_grid(R)
    B = sh_coefficients(atoms, kk, L, sigma=0.05)
    Bd = torch.tensor(B, dtype=torch.complex128, device="cuda")
    kd, wd = cuda(kk, torch.float64), cuda(ww, torch.float64)
    for sig in [0.0, 0.01, 0.03]:
        C = api.kernel_translated_sh(Bd, kd, wd, sig).cpu().numpy()
        C_ref = ref.kernel_translated_sh(B, kk, ww, sig)
        assert np.abs(C - C_ref).max() <= 1e-12 * np.abs(C_ref).max(), sig
        assert np.array_equal(C, C.T)
        C2 = api.kernel_translated_sh(Bd, kd, wd, sig).cpu().numpy()
        assert np.array_equal(C, C2)                                   # deterministic
        U, lam = api.eigen_basis(C, 8)
        Ur, lr = ref.basis(C_ref, 8)
        assert np.abs(lam[:8] - lr[:8]).max() <= 1e-10 * lr[0]
        h = 4
        assert np.abs(U[:, :h] @ U[:, :h].T - Ur[:, :h] @ Ur[:, :h].T).max() <= 1e-8
    with pytest.raises(api.RsvdError):
        api.kernel_translated_sh(Bd, kd, wd, -1.0)


@pytest.mark.parametrize("path", ["tc", "simt", "fused"])
def test_repeat_runs_bitwise_identical(path, monkeypatch):
    """Race-detection proxy (compute-sanitizer is closed on this pool): the same align call repeated
    20 times on the same inputs gives bitwise identical per-pair values/indices, landscapes and
    per-image keys.  A shared-memory or mbarrier race in the contraction / transform pipelines shows
    up as run-to-run differences at these sizes (several chunks, ragged tails, many CTAs per SM
    pipeline).  "fused": the persistent one-launch kernel (RSVD_FUSED=1), which must also reproduce
    the two-kernel TC path bit for bit (same K order per (pair, q), same transform code)."""
    api.set_path(api.PATH_SIMT if path == "simt" else api.PATH_TC)
    ref_out = None
    if path == "fused":
        monkeypatch.setenv("RSVD_FUSED", "0")
    try:
        d = make_dataset("small", M=300, T=260, device="cuda")
        w = d.w.contiguous()
        U, _ = api.build_basis(d.templates, w.cpu().numpy(), 8)
        Ud = cuda(U, torch.float64)
        M, T, Q = 300, 260, d.Q
        ib = api.compress(d.images, w, Ud, api.SIDE_IMAGE)
        tb = api.compress(d.templates, w, Ud, api.SIDE_TEMPLATE)
        work = torch.empty(api.align_min_workspace_bytes(Q) // 4, dtype=torch.float32, device="cuda")
        if path == "fused":
            ref_out = (api.align_argmax(ib, M, tb, T, Q, 8, api.PER_PAIR, work),
                       api.align_landscape(ib, M, tb, T, Q, 8, work))
            monkeypatch.setenv("RSVD_FUSED", "1")
            work = torch.empty(api.align_workspace_bytes(M, T, Q, 8) // 4, dtype=torch.float32, device="cuda")
        v0, k0 = api.align_argmax(ib, M, tb, T, Q, 8, api.PER_PAIR, work)
        X0 = api.align_landscape(ib, M, tb, T, Q, 8, work)
        key0 = api.align_argmax(ib, M, tb, T, Q, 8, api.PER_IMAGE, work)
        for _ in range(20):
            v, k = api.align_argmax(ib, M, tb, T, Q, 8, api.PER_PAIR, work)
            X = api.align_landscape(ib, M, tb, T, Q, 8, work)
            key = api.align_argmax(ib, M, tb, T, Q, 8, api.PER_IMAGE, work)
            assert torch.equal(v, v0) and torch.equal(k, k0)
            assert torch.equal(X, X0)
            assert torch.equal(key, key0)
        if ref_out is not None:
            assert torch.equal(ref_out[0][0], v0) and torch.equal(ref_out[0][1], k0)
            assert torch.equal(ref_out[1], X0)
    finally:
        api.set_path(api.PATH_AUTO)
