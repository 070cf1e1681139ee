"""The im2col + GEMM incumbent (mirrors gemm.py:1-74) on the GPU: a CUDA
im2col gather that materialises the full column matrix, then cuBLAS SGEMM
with TF32 disabled (the contrast column of every report)."""

from __future__ import annotations

import numpy as np

from . import _ops
from .tensor import ConvShape, CostCounters, ShapeError, as_array, as_filter2d, as_tensor2d


def im2col_2d(x, kh: int, kw: int, counters: CostCounters | None = None):
    """gemm.py:21-37: (out_h*out_w, kh*kw) column matrix."""
    x = as_tensor2d(x)
    s = ConvShape(int(x.shape[0]), int(x.shape[1]), kh, kw)
    cols = _ops.im2col(x, kh, kw)
    if counters is not None:
        counters.im2col_elems += s.out_h * s.out_w * kh * kw
    return cols


def gemm(a, b, counters: CostCounters | None = None):
    """gemm.py:40-59: float32 c = a @ b (cuBLAS SGEMM, IEEE fp32, no TF32)."""
    a = as_array(a)
    b = as_array(b)
    if a.ndim != 2 or b.ndim != 2:
        raise ShapeError("gemm expects 2-D matrices")
    m, k = (int(d) for d in a.shape)
    k2, n = (int(d) for d in b.shape)
    if k != k2:
        raise ShapeError(f"inner dimensions disagree: {tuple(a.shape)} x {tuple(b.shape)}")
    c = _ops.gemm(a if not isinstance(a, np.ndarray) else np.ascontiguousarray(a),
                  b if not isinstance(b, np.ndarray) else np.ascontiguousarray(b))
    if counters is not None:
        counters.macs += m * n * k
    return c


def conv2d_im2col(x, f, counters: CostCounters | None = None):
    """gemm.py:62-69: im2col then a (kh*kw, 1) GEMM; batched inputs loop."""
    x = as_tensor2d(x, allow_batch=True)
    f = as_filter2d(f)
    s = ConvShape.of(x, f)
    if x.ndim == 2:
        y = _ops.conv2d_im2col(x, f)
        units = 1
    else:
        flat = x.reshape((-1,) + tuple(x.shape[-2:]))
        ys = [_ops.conv2d_im2col(flat[i], f) for i in range(flat.shape[0])]
        if isinstance(ys[0], np.ndarray):
            y = np.stack(ys)
        else:
            import torch
            y = torch.stack(ys)
        y = y.reshape(tuple(x.shape[:-2]) + (s.out_h, s.out_w))
        units = flat.shape[0]
    if counters is not None:
        counters.im2col_elems += s.out_h * s.out_w * s.kh * s.kw * units
        counters.macs += s.out_h * s.out_w * s.kh * s.kw * units
    return y


def bloat_ratio(shape: ConvShape) -> float:
    """gemm.py:72-74."""
    return (shape.out_h * shape.out_w * shape.kh * shape.kw) / (shape.in_h * shape.in_w)
