"""CPU-only checks of the C ABI: the library builds for sm_100a, loads, exports every symbol that
include/rsvd.h declares (and the binding declares them all), and its host-only entry points
(sizes, the fp64 eigen-solver, argument validation that fails before any launch) behave."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2202_07235_b200 import build
    build.build()
    from paper_2202_07235_b200 import _lib
    return _lib.lib()


def _declared():
    inc = os.path.join(ROOT, "include")
    src = "".join(open(os.path.join(inc, f)).read() for f in sorted(os.listdir(inc)) if f.endswith(".h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsvd_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported_and_bound(lib):
    from paper_2202_07235_b200 import _lib
    names = _declared()
    assert len(names) >= 20
    bound = {n for n, _, _ in _lib.SIGNATURES}
    for n in names:
        assert hasattr(lib, n), f"{n} declared in rsvd.h but not exported"
        assert n in bound, f"{n} not bound in _lib.SIGNATURES"


def test_sizes(lib):
    from paper_2202_07235_b200 import api
    api.set_path(api.PATH_SIMT)
    try:
        assert api.path_for(512, 24) == api.PATH_SIMT
        assert api.block_bytes(16384, 512, 24) == 257 * 48 * 16384 * 8
        assert api.block_bytes(1, 32, 1) == 17 * 16 * 64 * 8
        api.set_path(api.PATH_TC)
        assert api.path_for(512, 24) == api.PATH_TC
        # TC layout: (N+1) q x KB = ceil(4H/32) k-blocks x {hi, lo} x operand rows of 32 fp16 (64 B);
        # images: 2 rows (Re, Im embedding) per image, padded to 128 images; templates padded to 256;
        # then one float scale per padded row, rounded up to 256 B
        assert api.block_bytes(16384, 512, 24, api.SIDE_IMAGE) == 257 * 3 * 2 * 32768 * 64 + 16384 * 4
        assert api.block_bytes(8192, 512, 24, api.SIDE_TEMPLATE) == 257 * 3 * 2 * 8192 * 64 + 8192 * 4
        assert api.block_bytes(10, 64, 4, api.SIDE_TEMPLATE) == 33 * 1 * 2 * 256 * 64 + 1024
        assert api.block_bytes(10, 64, 4, api.SIDE_IMAGE) == 33 * 1 * 2 * 256 * 64 + 512
        assert api.path_for(1024, 255) == api.PATH_SIMT        # H x Q block too large for the TC compress
        assert api.path_for(1024, 256) == api.PATH_TC          # 4 | H: the row splits into groups of 8 rings
    finally:
        api.set_path(api.PATH_AUTO)
    assert api.path_for(512, 24) == api.PATH_TC
    assert api.kernel_chunk() == 8
    assert api.kernel_partials_bytes(8192, 128) == 8192 // api.kernel_chunk() * 128 * 128 * 8
    assert api.align_min_workspace_bytes(512) == 128 * 256 * 256 * 8
    assert lib.rsvd_abi_version() == 6


def test_eigen_solver_matches_lapack(lib):
    from paper_2202_07235_b200 import api
    rng = np.random.default_rng(0)
    for R in [1, 3, 16, 64, 128, 256]:
        A = rng.standard_normal((R, R + 2))
        C = A @ A.T
        U, lam = api.eigen_basis(C, R)
        ref = np.sort(np.linalg.eigvalsh(C))[::-1]
        assert np.abs(lam - ref).max() <= 1e-13 * ref[0]
        assert np.linalg.norm(C @ U - U * lam) <= 1e-12 * ref[0]
        assert np.abs(U.T @ U - np.eye(R)).max() <= 1e-13
        # sign rule: largest-|.| entry of each column is positive
        assert np.all(U[np.abs(U).argmax(0), np.arange(R)] > 0)
    # low-rank PSD (the synthetic kernels are numerically low-rank): deterministic, orthonormal
    A = rng.standard_normal((128, 13))
    C = A @ A.T
    U1, l1 = api.eigen_basis(C, 64)
    U2, l2 = api.eigen_basis(C, 64)
    assert np.array_equal(U1, U2) and np.array_equal(l1, l2)
    assert np.abs(U1.T @ U1 - np.eye(64)).max() <= 1e-13


def test_eigen_solver_errors(lib):
    from paper_2202_07235_b200 import api
    with pytest.raises(api.RsvdError) as e:
        api.eigen_basis(np.full((4, 4), np.inf), 2)
    assert e.value.status == 4
    with pytest.raises(api.RsvdError) as e:
        api.eigen_basis(np.eye(4), 5)
    assert e.value.status == 2


def test_validation_before_launch(lib):
    """Bad arguments are rejected on the host (no device needed)."""
    assert lib.rsvd_compress(None, 4, 8, 48, None, None, 2, 0, None, None) == 2       # Q not pow2
    assert lib.rsvd_compress(None, 4, 8, 2048, None, None, 2, 0, None, None) == 2     # Q too large
    assert lib.rsvd_compress(None, 4, 300, 64, None, None, 2, 0, None, None) == 2     # R > 256
    assert lib.rsvd_compress(None, 4, 8, 64, None, None, 9, 0, None, None) == 2       # H > R
    assert lib.rsvd_compress(None, -1, 8, 64, None, None, 2, 0, None, None) == 1      # negative n
    assert lib.rsvd_compress(None, 4, 8, 64, None, None, 2, 0, None, None) == 1       # NULL
    assert lib.rsvd_compress(None, 0, 8, 64, None, None, 2, 0, None, None) == 0       # empty: no-op
    assert lib.rsvd_align_argmax(None, 0, None, 0, 0, 64, 2, 0, None, 0, None, None, None, None) == 0
    assert lib.rsvd_align_argmax(None, 3, None, 3, 0, 96, 2, 0, None, 0, None, None, None, None) == 2
    assert lib.rsvd_kernel_reduce(None, 0, 8, 1, 64, None, None, None) == 1
    assert b"Q" in lib.rsvd_last_error() or len(lib.rsvd_last_error()) > 0
    assert lib.rsvd_eigen_basis_device(None, 129, 8, None, None, None, None) == 2     # R > 128
    assert lib.rsvd_eigen_basis_device(None, 128, 65, None, None, None, None) == 2    # H * R > 8192
    assert lib.rsvd_eigen_basis_device(None, 64, 0, None, None, None, None) == 2      # H < 1
    assert lib.rsvd_eigen_basis_device(None, 64, 8, None, None, None, None) == 1      # NULL
    out = ctypes.c_double(0.0)
    assert lib.rsvd_probe_fp32(6, 1000, ctypes.byref(out), None) == 1                 # kinds 0..5 (3 = DFMA, 4/5 = DMMA)
    assert lib.rsvd_probe_fp32(3, 8, ctypes.byref(out), None) == 1                    # iters < 16
    assert lib.rsvd_probe_fp32(3, 1000, None, None) == 1                              # NULL result


def test_eigen_solver_top_h_path(lib):
    """H <= R/2 takes the top-H path (QR without vector updates + inverse iteration on the tridiagonal
    form): eigenvalues bitwise those of the full path, residual and orthonormality at fp64 level, the
    leading well-separated projector equal to LAPACK's, also for a numerically low-rank kernel whose
    top-H block reaches into the null cluster (as the Large kernel does at H = 24)."""
    from paper_2202_07235_b200 import api
    rng = np.random.default_rng(5)
    Qm, _ = np.linalg.qr(rng.standard_normal((128, 128)))
    spectra = [np.logspace(0, -15, 128), np.concatenate([np.logspace(0, -13, 18), np.full(110, 1e-16)]),
               np.sort(rng.random(128))[::-1]]
    for ev in spectra:
        C = (Qm * ev) @ Qm.T
        C = 0.5 * (C + C.T)
        U_full, lam_full = api.eigen_basis(C, 128)
        for H in [8, 24, 64]:
            U, lam = api.eigen_basis(C, H)
            assert np.array_equal(lam, lam_full)                 # same QR arithmetic on (d, e)
            assert np.linalg.norm(C @ U - U * lam[:H]) <= 1e-13 * lam[0]
            assert np.abs(U.T @ U - np.eye(H)).max() <= 1e-13
            assert np.all(U[np.abs(U).argmax(0), np.arange(H)] > 0)
            k = 6
            w, V = np.linalg.eigh(C)
            V = V[:, ::-1]
            assert np.abs(U[:, :k] @ U[:, :k].T - V[:, :k] @ V[:, :k].T).max() <= 1e-9


def test_grouped_align_validates_before_any_launch(lib):
    """rsvd_align_argmax_grouped (row f3) rejects bad descriptors with a status code and a message
    before enqueuing anything (no GPU needed: validation precedes every launch)."""
    from paper_2202_07235_b200 import _lib
    arr = (_lib.AlignGroup * 2)()
    arr[0] = _lib.AlignGroup(None, 8, None, 8, 0, None, None, None)
    assert lib.rsvd_align_argmax_grouped(ctypes.addressof(arr), -1, 64, 4, 0, None, 0, None) == 1
    assert lib.rsvd_align_argmax_grouped(None, 1, 64, 4, 0, None, 0, None) == 1
    assert lib.rsvd_align_argmax_grouped(ctypes.addressof(arr), 1, 64, 4, 0, None, 0, None) == 1
    assert b"group 0" in lib.rsvd_last_error()
    assert lib.rsvd_align_argmax_grouped(ctypes.addressof(arr), 1, 48, 4, 0, None, 0, None) == 2   # Q not a power of 2
    assert lib.rsvd_align_argmax_grouped(ctypes.addressof(arr), 0, 64, 4, 0, None, 0, None) == 0


def test_process_settings_roundtrip(lib):
    """Host-only setters of include/rsvd.h: precision (0 / 1) and the Step-1 kernel choice (0 / 1 / 2,
    out-of-range values fall back to the default 1); both are process-global and need no GPU."""
    p0, c0 = lib.rsvd_precision(), lib.rsvd_compress_mma_mode()
    try:
        for v in (1, 0):
            lib.rsvd_set_precision(v)
            assert lib.rsvd_precision() == v
        for v, want in ((2, 2), (0, 0), (7, 1), (-3, 1), (1, 1)):
            lib.rsvd_set_compress_mma(v)
            assert lib.rsvd_compress_mma_mode() == want
    finally:
        lib.rsvd_set_precision(p0)
        lib.rsvd_set_compress_mma(c0)
