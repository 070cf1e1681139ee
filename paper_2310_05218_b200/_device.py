"""Marshalling between the reference's array-in / array-out API and the C ABI.

* torch CUDA tensors stay on their device: the device entry points run on the
  tensor's current stream and return a new CUDA tensor (no host sync).
* host arrays (numpy / lists / CPU tensors) go through the `*_host` entry
  points, which pipeline H2D / kernel / D2H in chunks; outputs are new
  float32 numpy arrays (pinned when small enough, so D2H runs at full speed).
No path computes on the CPU: without a CUDA device every call raises.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib

_PIN_LIMIT = 2 << 30  # outputs up to 2 GiB come back in pinned host memory
_DEFAULT_EXACT = os.environ.get("SLIDECONV_B200_EXACT", "0") not in ("", "0", "false", "False")


def set_default_mode(mode: str) -> None:
    """'fast' (fused multiply-add; O(1) wide-window sums) or 'exact' (the
    reference's operation order, bit-identical float32 results)."""
    global _DEFAULT_EXACT
    if mode not in ("fast", "exact"):
        raise ValueError("mode must be 'fast' or 'exact'")
    _DEFAULT_EXACT = mode == "exact"


def mode_flag(exact: bool | None) -> int:
    e = _DEFAULT_EXACT if exact is None else bool(exact)
    return _lib.MODE_EXACT if e else _lib.MODE_FAST


def torch_mod():
    import torch
    return torch


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    if not _CUDA_OK:
        torch = torch_mod()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2310_05218_b200 computes on a CUDA device (sm_100a); none "
                               "is visible and there is no CPU fallback")
        _CUDA_OK = True
    return _lib.load()


def stream_of(t) -> int:
    """Raw handle of the current stream on t's device (the call enqueues there)."""
    torch = torch_mod()
    return torch._C._cuda_getCurrentRawStream(t.get_device())


class on_device:
    """Make t's device current for the C call; free when it already is
    (the common case -- torch.cuda.device() costs microseconds per call)."""

    __slots__ = ("dev", "prev")

    def __init__(self, t):
        self.dev = t.get_device()
        self.prev = -1

    def __enter__(self):
        torch = torch_mod()
        cur = torch._C._cuda_getDevice()
        if cur != self.dev:
            self.prev = cur
            torch._C._cuda_setDevice(self.dev)
        return self

    def __exit__(self, *exc):
        if self.prev >= 0:
            torch_mod()._C._cuda_setDevice(self.prev)
        return False


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """A numpy array backed by page-locked host memory (torch's caching host
    allocator).  Inputs allocated this way skip the staging copy."""
    torch = torch_mod()
    tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
    return torch.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()


def host_output(shape, dtype=np.float32) -> np.ndarray:
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if 0 < nbytes <= _PIN_LIMIT:
        return pinned_empty(shape, dtype)
    return np.empty(shape, dtype=dtype)


def ptr(a) -> int:
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def cuda_empty_like_dev(shape, ref, dtype=None):
    torch = torch_mod()
    return torch.empty(tuple(shape), dtype=dtype or ref.dtype, device=ref.device)


def to_device(a, dtype=np.float32):
    """Host array -> new CUDA tensor on the current device (for the paths
    without a host pipeline)."""
    torch = torch_mod()
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to("cuda", non_blocking=False)
    return a.to(device="cuda", dtype=tdt).contiguous()


def device_index() -> int:
    return torch_mod().cuda.current_device()
