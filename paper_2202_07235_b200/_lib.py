"""ctypes binding of librsvd.so (include/rsvd.h).  Argument marshalling only: every step of the
path runs in the library's kernels.  There is no CPU fallback: a missing library, a missing GPU
or a non-OK status raises RsvdError."""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

LIB_PATH = os.environ.get("RSVD_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "librsvd.so")
STATUS = {0: "RSVD_OK", 1: "RSVD_ERR_ARG", 2: "RSVD_ERR_UNSUPPORTED", 3: "RSVD_ERR_CUDA",
          4: "RSVD_ERR_NUMERIC"}
SIDE_IMAGE, SIDE_TEMPLATE = 0, 1
PER_PAIR, PER_IMAGE = 0, 1

# (name, restype, argtypes) -- mirrors include/rsvd.h
_P, _I32, _I64, _D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
SIGNATURES = [
    ("rsvd_last_error", ctypes.c_char_p, []),
    ("rsvd_abi_version", _I32, []),
    ("rsvd_block_bytes", _I64, [_I64, _I32, _I32, _I32]),
    ("rsvd_path_for", _I32, [_I32, _I32]),
    ("rsvd_set_path", None, [_I32]),
    ("rsvd_set_precision", None, [_I32]),
    ("rsvd_precision", _I32, []),
    ("rsvd_set_compress_mma", None, [_I32]),
    ("rsvd_compress_mma_mode", _I32, []),
    ("rsvd_kernel_chunk", _I64, []),
    ("rsvd_kernel_partials_bytes", _I64, [_I64, _I32]),
    ("rsvd_align_workspace_bytes", _I64, [_I64, _I64, _I32, _I32]),
    ("rsvd_align_min_workspace_bytes", _I64, [_I32]),
    ("rsvd_kernel_partials", _I32, [_P, _I64, _I32, _I32, _P, _P]),
    ("rsvd_kernel_reduce", _I32, [_P, _I64, _I32, _I64, _I32, _P, _P, _P]),
    ("rsvd_eigen_basis", _I32, [_P, _I32, _I32, _P, _P]),
    ("rsvd_eigen_basis_ctf", _I32, [_P, _I32, _P, _I32, _P, _P, _P]),
    ("rsvd_eigen_basis_device", _I32, [_P, _I32, _I32, _P, _P, _P, _P]),
    ("rsvd_build_basis", _I32, [_P, _I64, _I32, _I32, _P, _I32, _P, _P, _P]),
    ("rsvd_build_basis_translated", _I32, [_P, _I64, _I32, _I32, _P, _P, _P, _I32, _I32, _P, _P, _P]),
    ("rsvd_kernel_translated_sh", _I32, [_P, _I32, _I32, _P, _P, ctypes.c_double, _P, _P]),
    ("rsvd_compress", _I32, [_P, _I64, _I32, _I32, _P, _P, _I32, _I32, _P, _P]),
    ("rsvd_blocks_unpack", _I32, [_P, _I64, _I32, _I32, _I32, _P, _P]),
    ("rsvd_compress_translated", _I32, [_P, _I64, _I32, _I32, _P, _P, _P, _I32, _P, _I32, _I32, _P, _P]),
    ("rsvd_align_argmax", _I32, [_P, _I64, _P, _I64, _I64, _I32, _I32, _I32, _P, _I64, _P, _P, _P, _P]),
    ("rsvd_align_landscape", _I32, [_P, _I64, _P, _I64, _I32, _I32, _P, _I64, _P, _I64, _I64, _P]),
    ("rsvd_align_argmax_fine", _I32, [_P, _I64, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P, _I64, _P, _P, _P, _P, _P]),
    ("rsvd_align_argmax_grouped", _I32, [_P, _I32, _I32, _I32, _I32, _P, _I64, _P]),
    ("rsvd_align_landscape_fine", _I32, [_P, _I64, _P, _I64, _I32, _I32, _I32, _P, _I64, _P, _I64, _I64, _P]),
    ("rsvd_winners_reset", _I32, [_P, _I64, _P]),
    ("rsvd_winners_unpack", _I32, [_P, _I64, _I32, _P, _P, _P, _P]),
    ("rsvd_combine_winners", _I32, [_P, _I32, _I64, _I32, _P, _P, _P, _P, _P]),
    ("rsvd_launch_count", _I64, []),
    ("rsvd_timing_enable", None, [_I32]),
    ("rsvd_timing_read", _I32, [_P, _P, _I32]),
    ("rsvd_probe_fp32", _I32, [_I32, _I32, _P, _P]),
    # row f4 (include/rsvd_vol.h)
    ("rsvd_vol_ncoef", _I64, [_I32]),
    ("rsvd_vol_kernels", _I32, [_P, _I64, _I32, _I32, _P, _P, _P, _P]),
    ("rsvd_vol_compress", _I32, [_P, _I64, _I32, _I32, _P, _P, _I32, _P, _P]),
    ("rsvd_vol_wigner_table", _I32, [_P, _I32, _I32, _P, _I32, _P, _P]),
    ("rsvd_vol_degrees", _I32, [_P, _I64, _P, _I32, _I32, _P, _I32, _P, _P]),
    ("rsvd_vol_align", _I32, [_P, _I64, _P, _I32, _I32, _I32, _I32, _P, _P, _P]),
]


class AlignGroup(ctypes.Structure):
    """rsvd_align_group (include/rsvd.h, row f3)."""
    _fields_ = [("img_blocks", ctypes.c_void_p), ("M", ctypes.c_int64), ("tmpl_blocks", ctypes.c_void_p),
                ("T", ctypes.c_int64), ("t_offset", ctypes.c_int64), ("best_val", ctypes.c_void_p),
                ("best_k", ctypes.c_void_p), ("best_key", ctypes.c_void_p)]


class RsvdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lock = threading.Lock()
_lib = None


def lib():
    """Load librsvd.so (in-tree).  Raises if it is missing -- build it with __graft_entry__.build()."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RsvdError(3, f"{LIB_PATH} not built (run python -c 'import __graft_entry__ as g; g.build()')")
            L = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def check(status: int):
    if status != 0:
        raise RsvdError(status, lib().rsvd_last_error().decode())


def ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    """The caller's stream, else the current device's current stream (require_cuda has checked that
    the tensors live on the current device, so the work lands on the tensors' device)."""
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda(*tensors):
    if not torch.cuda.is_available():
        raise RsvdError(3, "no CUDA device: librsvd has no CPU fallback")
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise RsvdError(1, "expected a CUDA tensor")
        if t is not None and not t.is_contiguous():
            raise RsvdError(1, "expected a contiguous tensor")
        if t is not None and t.device.index != torch.cuda.current_device():
            raise RsvdError(1, f"tensor on {t.device} but the current device is cuda:{torch.cuda.current_device()} "
                               "(library work goes to the current device's stream: torch.cuda.set_device first)")
