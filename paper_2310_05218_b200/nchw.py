"""Multi-channel NCHW convolution with zero padding (new; BASELINE config 4).

No reference function exists (the reference is single-channel only,
SPEC.md:112); the semantics are the composition SURVEY 8(a) a12 fixes:
out[n, co] = sum over ci (ascending) of conv2d_reference(pad(x[n, ci]), w[co, ci]).
"""

from __future__ import annotations

from . import _ops
from .tensor import ShapeError, as_array


def conv2d_nchw(x, w, padding: int = 1, *, exact=None):
    """x (N, Cin, H, W), w (Cout, Cin, kh, kw) -> (N, Cout, H+2p-kh+1, W+2p-kw+1)."""
    x = as_array(x)
    w = as_array(w)
    if x.ndim != 4 or w.ndim != 4:
        raise ShapeError("conv2d_nchw expects x (N, C, H, W) and w (Cout, Cin, kh, kw)")
    if int(x.shape[1]) != int(w.shape[1]):
        raise ShapeError(f"channel mismatch: x has {x.shape[1]}, w expects {w.shape[1]}")
    p = int(padding)
    if p < 0:
        raise ShapeError("padding must be >= 0")
    if int(w.shape[2]) > int(x.shape[2]) + 2 * p or int(w.shape[3]) > int(x.shape[3]) + 2 * p:
        raise ShapeError("filter exceeds padded input")
    return _ops.conv2d_nchw(x, w, p, exact)
