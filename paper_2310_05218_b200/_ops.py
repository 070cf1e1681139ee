"""Thin typed calls into the C ABI (one per entry point family).

Inputs are already validated / coerced by the public modules; here only the
device-vs-host routing happens.  Every function runs a CUDA kernel.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import (device_index, host_output, mode_flag, on_device, ptr, require_cuda,
                      stream_of, to_device, torch_mod)
from .tensor import is_cuda_tensor


def _f32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def conv2d(x, f: np.ndarray, exact=None, shape_error=None):
    """x: (B, H, W) float32 numpy or CUDA tensor; f: (kh, kw) host float32."""
    lib = require_cuda()
    b, h, w = (int(d) for d in x.shape)
    kh, kw = (int(d) for d in f.shape)
    oh, ow = h - kh + 1, w - kw + 1
    f = _f32(f)
    mode = mode_flag(exact)
    if is_cuda_tensor(x):
        torch = torch_mod()
        y = torch.empty((b, oh, ow), dtype=torch.float32, device=x.device)
        with on_device(x):
            _lib.check(lib.sc_conv2d_f32(ptr(x), b, h, w, f.ctypes.data, kh, kw, mode, ptr(y),
                                         stream_of(x)), shape_error)
        return y
    y = host_output((b, oh, ow))
    _lib.check(lib.sc_conv2d_f32_host(ptr(x), b, h, w, f.ctypes.data, kh, kw, mode, ptr(y),
                                      device_index()), shape_error)
    return y


def conv2d_into(x, f: np.ndarray, y, exact=None):
    """CUDA-only: x (H, W) or (B, H, W) tensor -> write the valid conv into the
    preallocated contiguous CUDA tensor y (no allocation, current stream)."""
    lib = require_cuda()
    torch = torch_mod()
    xb = x.reshape((-1,) + tuple(x.shape[-2:]))
    b, h, w = (int(d) for d in xb.shape)
    kh, kw = (int(d) for d in f.shape)
    if tuple(y.shape[-2:]) != (h - kh + 1, w - kw + 1) or not y.is_contiguous():
        raise ValueError("conv2d_into: output view has the wrong shape or is not contiguous")
    f = _f32(f)
    with on_device(xb):
        _lib.check(lib.sc_conv2d_f32(ptr(xb), b, h, w, f.ctypes.data, kh, kw, mode_flag(exact),
                                     ptr(y), stream_of(xb)))
    return y


def conv1d(x, f: np.ndarray, exact=None):
    """x: (B, L) signals; f: (k,) taps -> (B, L - k + 1)."""
    lib = require_cuda()
    b, n = (int(d) for d in x.shape)
    f = _f32(f).reshape(-1)
    k = f.shape[0]
    mode = mode_flag(exact)
    if is_cuda_tensor(x):
        torch = torch_mod()
        y = torch.empty((b, n - k + 1), dtype=torch.float32, device=x.device)
        with on_device(x):
            _lib.check(lib.sc_conv1d_f32(ptr(x), b, n, f.ctypes.data, k, mode, ptr(y),
                                         stream_of(x)))
        return y
    y = host_output((b, n - k + 1))
    _lib.check(lib.sc_conv2d_f32_host(ptr(x), 1, b, n, f.ctypes.data, 1, k, mode, ptr(y),
                                      device_index()))
    return y


def conv2d_f64(x, f: np.ndarray):
    """float64 valid conv (oracle_conv2d); x (B, H, W) float64."""
    lib = require_cuda()
    torch = torch_mod()
    on_dev = is_cuda_tensor(x)
    xd = x if on_dev else to_device(x, np.float64)
    b, h, w = (int(d) for d in xd.shape)
    kh, kw = (int(d) for d in f.shape)
    f = np.ascontiguousarray(f, dtype=np.float64)
    y = torch.empty((b, h - kh + 1, w - kw + 1), dtype=torch.float64, device=xd.device)
    with on_device(xd):
        _lib.check(lib.sc_conv2d_f64(ptr(xd), b, h, w, f.ctypes.data, kh, kw, ptr(y),
                                     stream_of(xd)))
    return y if on_dev else y.cpu().numpy()


def pool1d(op: int, x, k: int, exact=None):
    """x: (B, L) float32 numpy or CUDA tensor -> (B, L - k + 1)."""
    lib = require_cuda()
    b, n = (int(d) for d in x.shape)
    mode = mode_flag(exact)
    if is_cuda_tensor(x):
        torch = torch_mod()
        y = torch.empty((b, n - k + 1), dtype=torch.float32, device=x.device)
        with on_device(x):
            _lib.check(lib.sc_pool1d_f32(op, ptr(x), b, n, k, mode, ptr(y), stream_of(x)))
        return y
    y = host_output((b, n - k + 1))
    _lib.check(lib.sc_pool1d_f32_host(op, ptr(x), b, n, k, mode, ptr(y), device_index()))
    return y


def pool1d_pair(op_a: int, x, k: int, exact=None):
    """x: (B, L) -> (y_a, y_max), each (B, L - k + 1), from one pass over x
    (op_a: POOL_SUM or POOL_AVG); host inputs cross the link once."""
    lib = require_cuda()
    b, n = (int(d) for d in x.shape)
    mode = mode_flag(exact)
    if is_cuda_tensor(x):
        torch = torch_mod()
        ya = torch.empty((b, n - k + 1), dtype=torch.float32, device=x.device)
        ym = torch.empty_like(ya)
        with on_device(x):
            _lib.check(lib.sc_pool1d_pair_f32(op_a, ptr(x), b, n, k, mode, ptr(ya), ptr(ym),
                                              stream_of(x)))
        return ya, ym
    ya = host_output((b, n - k + 1))
    ym = host_output((b, n - k + 1))
    _lib.check(lib.sc_pool1d_pair_f32_host(op_a, ptr(x), b, n, k, mode, ptr(ya), ptr(ym),
                                           device_index()))
    return ya, ym


def pool_stages(op: int, k: int) -> int:
    return int(_lib.load().sc_pool1d_stages(op, k))


def conv2d_nchw(x, wt, pad: int, exact=None):
    lib = require_cuda()
    torch = torch_mod()
    on_dev = is_cuda_tensor(x)
    xd = x if on_dev else to_device(x)
    wd = wt if is_cuda_tensor(wt) else to_device(wt)
    wd = wd.to(xd.device).contiguous()
    n, cin, h, w = (int(d) for d in xd.shape)
    cout, cin2, kh, kw = (int(d) for d in wd.shape)
    oh, ow = h + 2 * pad - kh + 1, w + 2 * pad - kw + 1
    y = torch.empty((n, cout, oh, ow), dtype=torch.float32, device=xd.device)
    with on_device(xd):
        _lib.check(lib.sc_conv2d_nchw_f32(ptr(xd), n, cin, h, w, ptr(wd), cout, kh, kw, pad,
                                          mode_flag(exact), ptr(y), stream_of(xd)))
    return y if on_dev else y.cpu().numpy()


def im2col(x, kh: int, kw: int):
    """x: (H, W) -> cols (oh*ow, kh*kw)."""
    lib = require_cuda()
    torch = torch_mod()
    on_dev = is_cuda_tensor(x)
    xd = x if on_dev else to_device(x)
    h, w = (int(d) for d in xd.shape)
    oh, ow = h - kh + 1, w - kw + 1
    cols = torch.empty((oh * ow, kh * kw), dtype=torch.float32, device=xd.device)
    with on_device(xd):
        _lib.check(lib.sc_im2col_f32(ptr(xd), h, w, kh, kw, 0, oh, ptr(cols), stream_of(xd)))
    return cols if on_dev else cols.cpu().numpy()


def gemm(a, b):
    lib = require_cuda()
    torch = torch_mod()
    on_dev = is_cuda_tensor(a)
    ad = a if on_dev else to_device(a)
    bd = (b if is_cuda_tensor(b) else to_device(b)).to(ad.device).contiguous()
    m, k = (int(d) for d in ad.shape)
    n = int(bd.shape[1])
    c = torch.empty((m, n), dtype=torch.float32, device=ad.device)
    with on_device(ad):
        _lib.check(lib.sc_gemm_f32(ptr(ad), ptr(bd), ptr(c), m, n, k, stream_of(ad)))
    return c if on_dev else c.cpu().numpy()


def conv2d_im2col(x, f: np.ndarray, max_cols_bytes: int = 8 << 30):
    """im2col + cuBLAS GEMM, chunked by output rows so the column matrix stays
    under max_cols_bytes.  x: (H, W)."""
    lib = require_cuda()
    torch = torch_mod()
    on_dev = is_cuda_tensor(x)
    xd = x if on_dev else to_device(x)
    h, w = (int(d) for d in xd.shape)
    kh, kw = (int(d) for d in f.shape)
    oh, ow = h - kh + 1, w - kw + 1
    fd = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float32).reshape(-1)).to(xd.device)
    row_bytes = ow * kh * kw * 4
    chunk = max(1, min(oh, max_cols_bytes // max(1, row_bytes)))
    cols = torch.empty((chunk * ow * kh * kw,), dtype=torch.float32, device=xd.device)
    y = torch.empty((oh, ow), dtype=torch.float32, device=xd.device)
    with on_device(xd):
        _lib.check(lib.sc_conv2d_im2col_f32(ptr(xd), h, w, ptr(fd), kh, kw, ptr(cols), chunk,
                                            ptr(y), stream_of(xd)))
    return y if on_dev else y.cpu().numpy()
