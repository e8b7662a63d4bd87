"""ctypes binding of the in-tree CUDA C-ABI library (include/conesplit_b200.h).

This is the only way the package computes anything: there is no CPU
fallback.  If the library is missing, or no CUDA device is visible, the
first operator call raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

__all__ = ["lib", "check", "NativeLibraryError", "ConesplitCudaError",
           "LIB_PATH", "SYMBOLS", "dptr", "hptr", "stream_ptr"]

LIB_PATH = os.environ.get("CS_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libconesplit_b200.so")


class NativeLibraryError(RuntimeError):
    """The CUDA library could not be loaded (not built, or no GPU)."""


class ConesplitCudaError(RuntimeError):
    """A C-ABI call returned an error code (``code``: CS_ERR_*)."""

    def __init__(self, msg: str, code: int = 0):
        super().__init__(msg)
        self.code = code


P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double
L = ctypes.c_int64

# name -> argtypes (restype int unless noted); mirrors include/conesplit_b200.h
SYMBOLS: dict[str, list] = {
    "cs_version": [],
    "cs_last_error": [],
    "cs_sync": [P],
    "cs_launch_count": [],
    "cs_release_cache": [],
    "cs_fwd_interp": [P, I, I, I, I, I, P, P, I, I, I, D, P, I, P],
    "cs_fwd_interp_residual": [P, I, I, I, P, P, I, I, I, D, P, P, P, P],
    "cs_fwd_siddon": [P, I, I, I, I, I, P, P, I, I, I, P, I, P],
    "cs_bwd_matched": [P, I, I, I, I, I, P, P, I, I, I, D, P, P],
    "cs_bwd_fdk": [P, I, I, I, I, P, P, I, D, D, D, D, D, D, I, I, P, P],
    "cs_ray_table": [I, I, I, P, P, I, I, I, D, P, P, P, P],
    "cs_tv_grad_sumsq": [P, I, I, I, I, I, P, P],
    "cs_tv_grad_norm": [P, I, I, I, I, I, P, P],
    "cs_tv_grad_store": [P, P, I, I, I, I, I, P, P],
    "cs_tv_step_g": [P, P, P, L, D, P, D, P],
    "cs_tv_gd_fused": [P, P, P, P, I, I, I, I, I, D, P, D, P, P],
    "cs_tv_step": [P, P, I, I, I, D, P, D, P],
    "cs_rof_iter": [P, P, P, I, I, I, D, P],
    "cs_rof_finish": [P, P, P, I, I, I, D, P],
    "cs_tv_norm": [P, I, I, I, P, P],
    "cs_dot": [P, P, L, P, P],
    "cs_axpy_ratio": [P, P, L, P, P, D, P],
    "cs_xpay_ratio": [P, P, L, P, P, P],
    "cs_guarded_inverse": [P, P, L, P],
    "cs_sart_update": [P, P, P, D, L, P],
    "cs_weighted_residual": [P, P, P, L, P],
    "cs_fill": [P, ctypes.c_float, L, P],
    "cs_sum_slices": [P, I, L, L, P, P, P, P],
    "cs_set_deterministic": [I],
    "cs_peer_enable": [I],
}

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and bind every exported symbol (no GPU
    needed to load)."""
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not built; run `python -m paper_1905_03748_b200.build` "
            "(or __graft_entry__.build())")
    L_ = ctypes.CDLL(path)
    for name, argtypes in SYMBOLS.items():
        fn = getattr(L_, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_char_p if name in (
            "cs_version", "cs_last_error") else (
            ctypes.c_longlong if name == "cs_launch_count" else ctypes.c_int)
    return L_


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch
                if not torch.cuda.is_available():
                    raise NativeLibraryError(
                        "no CUDA device visible: the conesplit B200 kernels "
                        "have no CPU fallback")
                _lib = load_library()
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.cs_last_error().decode() if _lib is not None else "?"
        raise ConesplitCudaError(f"conesplit_b200 error {rc}: {msg}", rc)


def dptr(t) -> int:
    """Device pointer of a contiguous CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def hptr(a: np.ndarray) -> int:
    """Host pointer of a C-contiguous numpy array."""
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("expected a C-contiguous host array")
    return a.ctypes.data


def stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
