"""ctypes binding of the C ABI in include/slideconv_b200.h.

The shared library is built in-tree (``paper_2310_05218_b200/libslideconv_b200.so``
by ``__graft_entry__.build()`` / ``make -C paper_2310_05218_b200/csrc``).  There is
no CPU fallback: if the library is missing every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SLIDECONV_B200_LIB: an alternative build of the same ABI (A/B timing tools)
LIB_PATH = os.environ.get("SLIDECONV_B200_LIB") or os.path.join(_HERE, "libslideconv_b200.so")

SC_OK = 0
SC_ERR_SHAPE = -1
SC_ERR_ARG = -2
SC_ERR_CUDA = -3
SC_ERR_UNSUPPORTED = -4
SC_ERR_CUBLAS = -5

POOL_SUM, POOL_AVG, POOL_MAX = 0, 1, 2
MODE_FAST, MODE_EXACT = 0, 1

_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/slideconv_b200.h exactly
SIGNATURES = {
    "sc_version": (_int, []),
    "sc_last_error": (ctypes.c_char_p, []),
    "sc_pool1d_f32": (_int, [_int, _vp, _i64, _i64, _i64, _int, _vp, _vp]),
    "sc_pool1d_pair_f32": (_int, [_int, _vp, _i64, _i64, _i64, _int, _vp, _vp, _vp]),
    "sc_pool1d_stages": (_i64, [_int, _i64]),
    "sc_conv1d_f32": (_int, [_vp, _i64, _i64, _vp, _i64, _int, _vp, _vp]),
    "sc_conv2d_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _int, _vp, _vp]),
    "sc_conv2d_segment_rows": (_i64, [_i64, _i64, _i64, _i64, _i64, _int]),
    "sc_conv2d_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp]),
    "sc_conv2d_nchw_f32": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64,
                                  _int, _vp, _vp]),
    "sc_im2col_f32": (_int, [_vp, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp]),
    "sc_gemm_f32": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "sc_conv2d_im2col_f32": (_int, [_vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _vp]),
    "sc_rowband_create": (_int, [_int, ctypes.POINTER(_int), ctypes.POINTER(_vp)]),
    "sc_rowband_destroy": (_int, [_vp]),
    "sc_rowband_conv2d_f32": (_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i64), _i64, _vp,
                                     _i64, _i64, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                     _int]),
    "sc_pool1d_f32_host": (_int, [_int, _vp, _i64, _i64, _i64, _int, _vp, _int]),
    "sc_pool1d_pair_f32_host": (_int, [_int, _vp, _i64, _i64, _i64, _int, _vp, _vp, _int]),
    "sc_conv2d_f32_host": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _int, _vp, _int]),
}

_lib = None
_load_error: str | None = None


class SlideconvCudaError(RuntimeError):
    """A CUDA / cuBLAS / argument failure reported by the native library."""


def load():
    """Load (once) and return the ctypes library; raise if it is missing."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        _load_error = (f"{LIB_PATH} not built: run __graft_entry__.build() or "
                       "`make -C paper_2310_05218_b200/csrc` (no CPU fallback exists)")
        raise ImportError(_load_error)
    import torch  # noqa: F401  -- load torch's CUDA libraries before ours
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().sc_last_error()
    return msg.decode() if msg else ""


def check(rc: int, shape_error=None):
    """Map a non-zero sc_status to the reference's exception classes."""
    if rc == SC_OK:
        return
    msg = last_error()
    if rc == SC_ERR_SHAPE:
        if shape_error is None:
            from .tensor import ShapeError as shape_error  # noqa: N813
        raise shape_error(msg)
    raise SlideconvCudaError(f"slideconv_b200 status {rc}: {msg}")
