"""Sliding-window sum / max / mean pooling (mirrors pooling.py:1-78).

Same signatures and return values as the reference: ``(y, stages)`` with y
1-D for 1-D input and ``(1, m)`` for ``(1, n)`` input, and the reference's
stage count (doubling + combine, pooling.py:37-51 / :67-76).  The work runs in
one sm_100a kernel per call: the doubling schedule in registers (bit-exact
sums and maxima), or, in fast mode for wide windows, an O(1)-per-output
float64 tile prefix.  Superset: ``(B, n)`` inputs pool each row (the
reference raises ShapeError for B > 1); ``sliding_window_mean`` is new
(float32 sum / float32 k, IEEE division); ``sliding_window_sum_max`` /
``sliding_window_mean_max`` return what the two separate calls return, from
ONE pass over x (one read of the input on the device, one upload of a host
array).
"""

from __future__ import annotations

import numpy as np

from . import _lib, _ops
from .lanes import VectorModel
from .tensor import ShapeError, as_array


def _as_signal(x):
    """pooling.py:18-25, widened to (B, n)."""
    a = as_array(x)
    squeeze = a.ndim == 1
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if a.ndim < 2:
        raise ShapeError("pooling expects a 1-D signal or a height-1 row tensor")
    lead = tuple(a.shape[:-1])
    a = a.reshape(-1, a.shape[-1])
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a)
    else:
        a = a.contiguous()
    return a, squeeze, lead


def _pool(op, x, k, exact):
    a, squeeze, lead = _as_signal(x)
    n = int(a.shape[-1])
    k = int(k)
    if not 1 <= k <= n:
        raise ShapeError(f"window {k} out of range for length {n}")
    y = _ops.pool1d(op, a, k, exact)
    stages = _ops.pool_stages(_lib.POOL_MAX if op == _lib.POOL_MAX else _lib.POOL_SUM, k)
    if squeeze:
        return y.reshape(-1), stages
    return y.reshape(lead + (n - k + 1,)), stages


def sliding_window_sum(x, k: int, vm: VectorModel | None = None, *, exact=None):
    """pooling.py:28-53: y[i] = sum(x[i:i+k])."""
    return _pool(_lib.POOL_SUM, x, k, exact)


def sliding_window_max(x, k: int, vm: VectorModel | None = None, *, exact=None):
    """pooling.py:56-78: y[i] = max(x[i:i+k]); always bit-exact (np.maximum
    semantics: NaN propagates, +0/-0 ties resolve as the reference's order)."""
    return _pool(_lib.POOL_MAX, x, k, exact)


def sliding_window_mean(x, k: int, vm: VectorModel | None = None, *, exact=None):
    """Average pooling (new): float32(window sum) / float32(k)."""
    return _pool(_lib.POOL_AVG, x, k, exact)


def _pool_pair(op_a, x, k, exact):
    a, squeeze, lead = _as_signal(x)
    n = int(a.shape[-1])
    k = int(k)
    if not 1 <= k <= n:
        raise ShapeError(f"window {k} out of range for length {n}")
    ya, ym = _ops.pool1d_pair(op_a, a, k, exact)
    shape = (-1,) if squeeze else lead + (n - k + 1,)
    return ((ya.reshape(shape), _ops.pool_stages(_lib.POOL_SUM, k)),
            (ym.reshape(shape), _ops.pool_stages(_lib.POOL_MAX, k)))


def sliding_window_sum_max(x, k: int, vm: VectorModel | None = None, *, exact=None):
    """Fused (new): ``(sliding_window_sum(x, k), sliding_window_max(x, k))``
    -- pooling.py:28-53 and :56-78 -- bit-identical to the two calls, computed
    in one pass over x."""
    return _pool_pair(_lib.POOL_SUM, x, k, exact)


def sliding_window_mean_max(x, k: int, vm: VectorModel | None = None, *, exact=None):
    """Fused (new): ``(sliding_window_mean(x, k), sliding_window_max(x, k))``
    in one pass over x (BASELINE config 2's average + max pooling)."""
    return _pool_pair(_lib.POOL_AVG, x, k, exact)
