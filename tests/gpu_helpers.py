"""Shared helpers for the -m gpu parity tests: run the CUDA path on seeded inputs and compare with
the fp64 oracle under DESIGN.md's tolerance rules (landscape: max|dX| <= tol * max|X_ref| with tol
1e-5 for the FP32 path; argmax exact wherever the reference top-2 gap exceeds tol * max|X_ref|,
otherwise inside the near-tie set)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import ref

TOL_FP32 = 1e-5


def to_np(x):
    return x.detach().cpu().numpy()


def assert_landscape_close(X_gpu: np.ndarray, X_ref: np.ndarray, tol: float = TOL_FP32):
    scale = np.abs(X_ref).max()
    err = np.abs(X_gpu.astype(np.float64) - X_ref).max()
    assert err <= tol * scale, f"landscape error {err / scale:.3e} > {tol:.1e} (relative to max|X_ref|)"
    return err / scale


def assert_argmax_gated(k_gpu: np.ndarray, X_ref: np.ndarray, tol_abs: float):
    """Bit-exact where the top-2 gap > tol_abs; otherwise k_gpu must be in the near-tie set."""
    k_ref = ref.argmax_first(X_ref)
    gap = ref.top2_gap(X_ref)
    gated = gap > tol_abs
    bad = gated & (k_gpu != k_ref)
    assert not bad.any(), f"{bad.sum()} gated argmax mismatches of {gated.sum()}"
    ok = ref.near_tie_ok(X_ref, k_gpu, tol_abs)
    assert ok.all(), f"{(~ok).sum()} argmaxes outside the near-tie set"
    return int(gated.sum())


def assert_per_image(val, t, k, X_ref_img: np.ndarray, tol_abs: float):
    """X_ref_img [M, T, Q] (Re X).  Winner (t, k) exact when the best entry beats the runner-up
    by > tol_abs; always within the near-tie set; value within tol_abs."""
    M, T, Q = X_ref_img.shape
    flat = X_ref_img.reshape(M, T * Q)
    for m in range(M):
        v_ref, t_ref, k_ref = ref.per_image_winner(X_ref_img[m])
        g = ref.top2_gap(flat[m:m + 1])[0]
        got = flat[m, int(t[m]) * Q + int(k[m])]
        assert abs(float(val[m]) - v_ref) <= tol_abs, (m, float(val[m]), v_ref)
        if g > tol_abs:
            assert (int(t[m]), int(k[m])) == (t_ref, k_ref), (m, t[m], k[m], t_ref, k_ref)
        assert got >= v_ref - tol_abs


def cuda(x, dtype=None):
    t = torch.as_tensor(x)
    if dtype is not None:
        t = t.to(dtype)
    return t.contiguous().cuda()
