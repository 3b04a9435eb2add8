"""Row f4 (volume alignment, §5) on the GPU vs the fp64 oracle (oracle/vol.py), element by
element, through the C ABI (include/rsvd_vol.h).  Tolerances: fp64 kernels 1e-12 relative; fp32
tables / shells / landscapes 1e-5 of the reference's max (DESIGN.md f4 tolerance); argmax exact where
the reference top-2 gap exceeds that tolerance."""
import numpy as np
import pytest
import torch

from oracle import vol as ov
from synth import volumes as sv
from tests.gpu_helpers import TOL_FP32, to_np

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2202_07235_b200.api")


def dev(x, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(x))
    return t.to("cuda", dtype=dtype) if dtype else t.to("cuda")


def _ref_table(L, betas, V):
    """[nb][HD][m2 + L][m1 + L] (the library's layout, include/rsvd_vol.h)."""
    M = 2 * L + 1
    T = np.zeros((len(betas), V.shape[1], M, M))
    for ib, b in enumerate(betas):
        d = ov.wigner_d(L, b)                                              # d[l][m1 + l, m2 + l]
        for l in range(L + 1):
            T[ib, :, L - l:L + l + 1, L - l:L + l + 1] += V[l][:, None, None] * d[l].T[None]
    return T


def test_kernels_match_oracle():
    vs = sv.make_volumes(12, 14, 1, nb=4, atoms=9, K=9.0, seed=11)
    B = np.stack([vs.target, vs.volumes[0]])                               # two targets: the average
    C, D = api.vol_kernels(dev(B), dev(vs.w), vs.L)
    Cr, Dr = ov.vol_kernel_C(B, vs.w), ov.vol_kernel_D(B, vs.w, vs.L)
    assert np.abs(to_np(C) - Cr).max() <= 1e-12 * np.abs(Cr).max()
    assert np.abs(to_np(D) - Dr).max() <= 1e-12 * np.abs(Dr).max()


@pytest.mark.parametrize("L,HD", [(10, 5), (31, 16), (63, 32)])
def test_wigner_table_matches_oracle(L, HD):
    """Seeds + three-term recurrence in fp64 vs the J_y exponential, up to the maximum L = 63."""
    rng = np.random.default_rng(L)
    V, _ = np.linalg.qr(rng.standard_normal((L + 1, HD)))
    betas = np.array([-np.pi, -2.3, -0.4, 0.0, 1e-3, 0.9, 2.0, np.pi - 1e-3])
    T = to_np(api.vol_wigner_table(dev(betas), L, dev(V)))
    Tr = _ref_table(L, betas, V)
    assert np.abs(T - Tr).max() <= 2e-6 * np.abs(Tr).max()


def test_compress_matches_oracle():
    vs = sv.make_volumes(9, 11, 3, nb=4, atoms=8, K=7.0, seed=12)
    U, _ = ov.vol_basis(ov.vol_kernel_C(vs.target, vs.w), 7)
    sh = to_np(api.vol_compress(dev(vs.volumes), dev(vs.w), dev(U), vs.L))          # [n, HC, NC]
    for i in range(3):
        want = ov.vol_shells(vs.volumes[i], vs.w, U)
        assert np.abs(sh[i] - want).max() <= TOL_FP32 * np.abs(want).max()


def _gpu_pipeline(vs, HC, HD, landscape=True, P=None):
    P = P or vs.P
    al = api.VolumeAligner(dev(vs.target), dev(vs.w), vs.L, HC, HD, dev(vs.betas), P=P)
    X, (val, b, a, g) = al.align(dev(vs.volumes), landscape=landscape)
    return al, (to_np(X) if X is not None else None), to_np(val), to_np(b), to_np(a), to_np(g)


@pytest.mark.parametrize("L,R,n,nb,HC,HD,jitter", [
    (10, 12, 5, 6, 6, 5, 0.01),       # compressed ranks, jittered volumes
    (8, 10, 3, 4, 10, 9, 0.0),        # full ranks (HC = R, HD = L + 1): the uncompressed landscape
    (15, 16, 2, 3, 1, 1, 0.02),       # rank 1 / 1, M = 31 < P = 32
    (20, 18, 2, 5, 8, 8, 0.01),       # P = 64
])
def test_landscape_matches_oracle(L, R, n, nb, HC, HD, jitter):
    vs = sv.make_volumes(L, R, n, nb=nb, atoms=12, K=L / 1.2, seed=L, jitter=jitter)
    al, X, val, b, a, g = _gpu_pipeline(vs, HC, HD)
    U, V = to_np(al.U), to_np(al.V)
    for i in range(n):
        Xr = ov.vol_landscape_rank(vs.volumes[i], vs.target, vs.w, U, V, L, vs.betas, vs.P)
        scale = np.abs(Xr).max()
        assert np.abs(X[i] - Xr).max() <= TOL_FP32 * scale, i
        rv, ridx = ov.vol_best(Xr[None])
        assert abs(val[i] - rv[0]) <= TOL_FP32 * scale
        flat = (b[i] * vs.P + a[i]) * vs.P + g[i]
        srt = np.sort(Xr.ravel())
        if srt[-1] - srt[-2] > TOL_FP32 * scale:
            assert flat == ridx[0]
        else:
            assert Xr.ravel()[flat] >= srt[-1] - TOL_FP32 * scale
    if HC == R and HD == L + 1:                                              # full rank == Eq. volume_innerproduct
        Xf = ov.vol_landscape_full(vs.volumes[0], vs.target, vs.w, L, vs.betas, vs.P)
        assert np.abs(X[0] - Xf).max() <= TOL_FP32 * np.abs(Xf).max()


def test_rotation_recovered_on_grid():
    """Exactly rotated copies of the target, full ranks: the per-volume winner is the applied rotation.
    At beta = 0 or +-pi the Euler angles are degenerate (only alpha +- gamma matters), so the winner is
    compared as a rotation matrix."""
    vs = sv.make_volumes(12, 14, 6, nb=8, atoms=10, K=10.0, seed=21)
    _, _, val, b, a, g = _gpu_pipeline(vs, 14, 13, landscape=False)
    for i in range(6):
        tb, ta, tg = vs.tau_index[i]
        R_true = sv.rotation(2 * np.pi * ta / vs.P, vs.betas[tb], 2 * np.pi * tg / vs.P)
        R_found = sv.rotation(2 * np.pi * a[i] / vs.P, vs.betas[b[i]], 2 * np.pi * g[i] / vs.P)
        assert np.abs(R_found - R_true).max() < 1e-9, (i, (b[i], a[i], g[i]), (tb, ta, tg))
        norm = np.sum(vs.w[:, None] * np.abs(vs.volumes[i].astype(np.complex128)) ** 2)
        assert abs(val[i] / norm - 1) < 1e-4


def test_max_size_sampled():
    """L = 63 (M = 127, P = 128), ranks 16 / 16: two volumes against the oracle at three betas."""
    vs = sv.make_volumes(63, 64, 2, nb=3, atoms=30, seed=5, jitter=0.01)
    al, X, val, b, a, g = _gpu_pipeline(vs, 16, 16)
    U, V = to_np(al.U), to_np(al.V)
    for i in range(2):
        Xr = ov.vol_landscape_rank(vs.volumes[i], vs.target, vs.w, U, V, 63, vs.betas, vs.P)
        assert np.abs(X[i] - Xr).max() <= TOL_FP32 * np.abs(Xr).max()


def test_errors_and_empty():
    L = 10
    Y = torch.zeros(1, 4, 21, 21, dtype=torch.complex64, device="cuda")
    T = torch.zeros(2, 4, 21, 21, dtype=torch.float32, device="cuda")
    with pytest.raises(api.RsvdError):
        api.vol_align(Y, T, L, 16)                                           # P < 2L+1 / not supported
    with pytest.raises(api.RsvdError):
        api.vol_wigner_table(dev(np.zeros(2)), L, dev(np.zeros((L + 1, L + 2))))  # HD > L + 1
    with pytest.raises(api.RsvdError):
        api.vol_kernels(torch.zeros(1, 4, 64 * 64 + 128, dtype=torch.complex64, device="cuda"),
                        dev(np.ones(4)), 64)                                 # L > 63
    X, _ = api.vol_align(Y[:0], T, L, 32)                                    # n = 0: no launch
    assert X.shape[0] == 0
