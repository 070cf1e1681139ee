"""Naive entry points and the float64 oracle (mirrors reference.py:1-54).

All three run on the GPU: ``conv2d_reference`` / ``conv1d_reference`` through
the same sm_100a convolution kernels as the slide variants, ``oracle_conv2d``
through a float64 instantiation of the runtime-(kh, kw) kernel.
"""

from __future__ import annotations

import numpy as np

from . import _ops
from .tensor import ConvShape, ShapeError, as_array, as_filter2d, as_tensor2d, is_cuda_tensor


def _batched(x):
    """(H, W) -> (1, H, W) view; (B, H, W) passes through."""
    return x.reshape((1,) + tuple(x.shape)) if x.ndim == 2 else x.reshape((-1,) + tuple(x.shape[-2:]))


def _unbatch(y, lead):
    return y.reshape(tuple(lead) + tuple(y.shape[-2:]))


def conv2d(x, f, exact=None):
    """Validated valid conv, any leading batch dims; returns array/tensor."""
    x = as_tensor2d(x, allow_batch=True)
    f = as_filter2d(f)
    ConvShape.of(x, f)
    lead = tuple(x.shape[:-2])
    y = _ops.conv2d(_batched(x), f, exact)
    return _unbatch(y, lead) if lead else y[0]


def conv2d_reference(x, f, *, exact=True):
    """reference.py:26-30: 2-D valid convolution, float32, tap order (j, i).
    Upstream documents this entry point as the bit-for-bit multiply-then-add
    baseline, so it defaults to exact mode (bit-identical to the reference);
    exact=False / None selects the FFMA kernels (module default)."""
    return conv2d(x, f, exact)


def conv1d_reference(x, f, *, exact=True):
    """reference.py:33-39: height-1 input and filter (exact by default, as
    conv2d_reference)."""
    x = as_tensor2d(x)
    f = as_filter2d(f)
    if x.shape[0] != 1 or f.shape[0] != 1:
        raise ShapeError("conv1d_reference expects height-1 input and filter")
    return conv2d(x, f, exact)


def oracle_conv2d(x, f):
    """reference.py:42-47: the same formula evaluated entirely in float64."""
    xa = as_array(x, np.float64)
    if xa.ndim == 1:
        xa = xa.reshape(1, -1)
    fa = np.atleast_2d(np.asarray(f if not hasattr(f, "cpu") else f.cpu().numpy(), dtype=np.float64))
    ConvShape.of(xa, fa)
    lead = tuple(xa.shape[:-2])
    xb = xa.reshape((-1,) + tuple(xa.shape[-2:]))
    if not is_cuda_tensor(xb):
        xb = np.ascontiguousarray(xb)
    y = _ops.conv2d_f64(xb, fa)
    return y.reshape(lead + tuple(y.shape[-2:])) if len(lead) > 0 and xa.ndim > 2 else y[0]


def relative_error(got, want) -> float:
    """reference.py:50-54: max elementwise |got - want| / max(1, |want|)."""
    def host(a):
        return a.detach().cpu().numpy() if hasattr(a, "detach") else a
    got = np.asarray(host(got), dtype=np.float64)
    want = np.asarray(host(want), dtype=np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want)), initial=0.0))
