"""Steps 3-4 with pass 1 on the tensor cores (rsvd_fftc.cuh, RSVD_FFTC=1), -m gpu: the 1e-5 gate of the
fp32-grade path against the oracle at the Medium (Q = 256) and Large (Q = 512) shapes, several chunks
with ragged tails, per-pair and per-image modes, and the Large bench configuration's winners."""
import numpy as np
import pytest
import torch

from oracle import ref
from synth import make_dataset, sample_pairs
from tests.gpu_helpers import TOL_FP32, assert_argmax_gated, assert_per_image, cuda, to_np

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2202_07235_b200.api")


@pytest.fixture
def fftc(monkeypatch):
    api.set_path(api.PATH_TC)
    monkeypatch.setenv("RSVD_FFTC", "1")
    yield
    api.set_path(api.PATH_AUTO)


@pytest.mark.parametrize("name,M,T,H", [("medium", 300, 270, 16), ("large", 200, 140, 24)])
def test_fftc_small_shapes(fftc, name, M, T, H):
    d = make_dataset(name, M=M, T=T, device="cuda")
    Q = d.Q
    w = to_np(d.w)
    U, _ = api.build_basis(d.templates, w, H)
    wd, Ud = d.w.contiguous(), cuda(U, torch.float64)
    ib = api.compress(d.images, wd, Ud, api.SIDE_IMAGE)
    tb = api.compress(d.templates, wd, Ud, api.SIDE_TEMPLATE)
    work = torch.empty(api.align_min_workspace_bytes(Q) // 4, dtype=torch.float32, device="cuda")
    val, k = api.align_argmax(ib, M, tb, T, Q, H, api.PER_PAIR, work)
    keys = api.align_argmax(ib, M, tb, T, Q, H, api.PER_IMAGE, work)
    ia, it = np.meshgrid(np.arange(M), np.arange(T), indexing="ij")
    X_ref = ref.landscape_rank(to_np(d.images), to_np(d.templates), w, U, ia.ravel(), it.ravel()).real.reshape(M, T, Q)
    tol_abs = TOL_FP32 * np.abs(X_ref).max()
    err = np.abs(to_np(val) - X_ref.max(-1)).max()
    assert err <= tol_abs, err / np.abs(X_ref).max()
    assert_argmax_gated(to_np(k).ravel(), X_ref.reshape(-1, Q), tol_abs)
    v, t, kk = (to_np(x) for x in api.winners_unpack(keys, Q))
    assert_per_image(v, t, kk, X_ref, tol_abs)
    print(f"\nfftc {name}: max-value error {err / np.abs(X_ref).max():.2e} of max|X_ref|")


def test_fftc_large_bench_configuration(fftc):
    d = make_dataset("large", device="cuda")
    M, T, Q, H = d.images.shape[0], d.templates.shape[0], d.Q, 24
    w = to_np(d.w)
    U, _ = api.build_basis(d.templates, w, H)
    wd, Ud = d.w.contiguous(), cuda(U, torch.float64)
    ib = api.compress(d.images, wd, Ud, api.SIDE_IMAGE)
    tb = api.compress(d.templates, wd, Ud, api.SIDE_TEMPLATE)
    work = torch.empty(api.align_workspace_bytes(M, T, Q, H) // 4, dtype=torch.float32, device="cuda")
    keys = api.winners_reset(torch.zeros(M, dtype=torch.int64, device="cuda"))
    api.align_argmax(ib, M, tb, T, Q, H, api.PER_IMAGE, work, best_key=keys)
    val, tw, kw = (to_np(x) for x in api.winners_unpack(keys, Q))
    B = d.templates.cpu().numpy()
    for m in [11, 9999]:
        A = d.images[m:m + 1].cpu().numpy()
        X = ref.landscape_rank(A, B, w, U, np.zeros(T, np.int64), np.arange(T)).real
        v_ref, _, _ = ref.per_image_winner(X)
        tol_abs = TOL_FP32 * np.abs(X).max()
        assert abs(float(val[m]) - v_ref) <= tol_abs
        assert X[tw[m], kw[m]] >= v_ref - tol_abs
    bv, bk = api.align_argmax(ib, M, tb, T, Q, H, api.PER_PAIR, work)
    mm, tt = sample_pairs("large", M, T, 512, 0)
    um, im_ = np.unique(mm, return_inverse=True)
    ut, it_ = np.unique(tt, return_inverse=True)
    Xs = ref.landscape_rank(d.images[torch.as_tensor(um, device="cuda")].cpu().numpy(),
                            d.templates[torch.as_tensor(ut, device="cuda")].cpu().numpy(), w, U, im_, it_).real
    tol_abs = TOL_FP32 * np.abs(Xs).max()
    sel = (torch.as_tensor(mm, device="cuda"), torch.as_tensor(tt, device="cuda"))
    assert np.abs(to_np(bv[sel]) - Xs.max(-1)).max() <= tol_abs
    assert_argmax_gated(to_np(bk[sel]), Xs, tol_abs)
