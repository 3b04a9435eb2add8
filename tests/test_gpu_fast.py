"""The single-pass tensor-core path (rsvd_set_precision(1), -m gpu): one fp16 MMA per product and an
fp16 spectrum, held to north_star's gate for tensor-core paths, max|X_gpu - X_ref| <= 2e-3 max|X_ref|,
with argmaxes exact wherever the oracle's top-2 gap exceeds that tolerance.  Several chunks with
ragged tails (minimum workspace), every output mode, the Small / Medium / Large shapes, and the Large
bench configuration's per-image winners."""
import numpy as np
import pytest
import torch

from oracle import ref
from synth import make_dataset, sample_pairs
from tests.gpu_helpers import assert_argmax_gated, assert_landscape_close, assert_per_image, cuda, to_np

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2202_07235_b200.api")
TOL_FAST = 2e-3


@pytest.fixture
def fast():
    api.set_path(api.PATH_TC)
    api.set_precision(api.PREC_FAST)
    yield
    api.set_precision(api.PREC_FP32)
    api.set_path(api.PATH_AUTO)


@pytest.mark.parametrize("name,M,T,H", [("small", 300, 260, 8), ("medium", 200, 140, 16), ("large", 160, 140, 24)])
def test_fast_path_all_modes(fast, name, M, T, H):
    d = make_dataset(name, M=M, T=T, device="cuda")
    Q = d.Q
    w = to_np(d.w)
    U, _ = api.build_basis(d.templates, w, H)
    wd, Ud = d.w.contiguous(), cuda(U, torch.float64)
    ib = api.compress(d.images, wd, Ud, api.SIDE_IMAGE)
    tb = api.compress(d.templates, wd, Ud, api.SIDE_TEMPLATE)
    work = torch.empty(api.align_min_workspace_bytes(Q) // 4, dtype=torch.float32, device="cuda")
    X = to_np(api.align_landscape(ib, M, tb, T, Q, H, work))
    val, k = api.align_argmax(ib, M, tb, T, Q, H, api.PER_PAIR, work)
    keys = api.align_argmax(ib, M, tb, T, Q, H, api.PER_IMAGE, work)
    ia, it = np.meshgrid(np.arange(M), np.arange(T), indexing="ij")
    A, B = to_np(d.images), to_np(d.templates)
    X_ref = ref.landscape_rank(A, B, w, U, ia.ravel(), it.ravel()).real.reshape(M, T, Q)
    err = assert_landscape_close(X, X_ref, TOL_FAST)
    assert err > 1e-7                                   # really the reduced-precision path
    tol_abs = TOL_FAST * np.abs(X_ref).max()
    assert np.abs(to_np(val) - X_ref.max(-1)).max() <= tol_abs
    assert_argmax_gated(to_np(k).ravel(), X_ref.reshape(-1, Q), tol_abs)
    v, t, kk = (to_np(x) for x in api.winners_unpack(keys, Q))
    assert_per_image(v, t, kk, X_ref, tol_abs)
    print(f"\nfast path {name}: landscape error {err:.2e} of max|X_ref| (gate {TOL_FAST})")


def test_fast_path_large_bench_configuration(fast):
    """Large, PER_IMAGE, the bench's workspace: one image's winner against the oracle over all 8192
    templates, and 256 sampled pairs in PER_PAIR mode."""
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
    m = 777
    A = d.images[m:m + 1].cpu().numpy()
    X = ref.landscape_rank(A, B, w, U, np.zeros(T, np.int64), np.arange(T)).real
    v_ref, _, _ = ref.per_image_winner(X)
    tol_abs = TOL_FAST * np.abs(X).max()
    assert abs(float(val[m]) - v_ref) <= tol_abs
    assert X[tw[m], kw[m]] >= v_ref - tol_abs
    bv, bk = api.align_argmax(ib, M, tb, T, Q, H, api.PER_PAIR, work)
    mm, tt = sample_pairs("large", M, T, 256, 0)
    um, im_ = np.unique(mm, return_inverse=True)
    ut, it_ = np.unique(tt, return_inverse=True)
    Xs = ref.landscape_rank(d.images[torch.as_tensor(um, device="cuda")].cpu().numpy(),
                            d.templates[torch.as_tensor(ut, device="cuda")].cpu().numpy(), w, U, im_, it_).real
    tol_abs = TOL_FAST * np.abs(Xs).max()
    sel = (torch.as_tensor(mm, device="cuda"), torch.as_tensor(tt, device="cuda"))
    assert np.abs(to_np(bv[sel]) - Xs.max(-1)).max() <= tol_abs
    assert_argmax_gated(to_np(bk[sel]), Xs, tol_abs)
