"""Fast-mode window sums / averages with non-finite and mixed-scale inputs.

The fast wide-window kernels (pool_wide.cu, 33 < k <= 2049; pool1d.cu
pool_prefix_kernel, 2049 < k <= 8192) must compute every output from its own
window's samples only: an inf / NaN / 1e30 elsewhere in the tile -- or at the
end of the previous signal when an unaligned batch is viewed as one flat
signal -- must not change it.  The reference (pooling.py:28-53) sums each
window by doubling, so its result is non-finite exactly when the window holds
a non-finite sample (or +inf and -inf: NaN), and finite windows carry a
rounding error of order eps * log2(k) * sum|window|.
"""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu

EPS32 = float(np.finfo(np.float32).eps)


def _window_abs_sum(x: np.ndarray, k: int) -> np.ndarray:
    """sum |x| over every window, float64, non-finite samples counted as 0;
    each window summed directly (a running-sum difference would itself lose
    the small windows after a 1e30 sample)."""
    a = np.where(np.isfinite(x), np.abs(x.astype(np.float64)), 0.0)
    m = a.shape[-1] - k + 1
    out = np.empty(a.shape[:-1] + (m,))
    chunk = max(1, (32 << 20) // (8 * k * max(1, a[..., 0].size)))
    for s in range(0, m, chunk):
        e = min(m, s + chunk)
        win = np.lib.stride_tricks.sliding_window_view(a[..., s:e + k - 1], k, axis=-1)
        out[..., s:e] = win.sum(axis=-1)
    return out


def _check(got: np.ndarray, want: np.ndarray, x: np.ndarray, k: int, op: str):
    assert got.shape == want.shape
    assert np.array_equal(np.isnan(got), np.isnan(want)), (op, k, "NaN pattern")
    assert np.array_equal(np.isposinf(got), np.isposinf(want)), (op, k, "+inf pattern")
    assert np.array_equal(np.isneginf(got), np.isneginf(want)), (op, k, "-inf pattern")
    fin = np.isfinite(want)
    bound = 2.0 * k * EPS32 * _window_abs_sum(x, k)
    if op == "avg":
        bound = bound / k + EPS32 * np.abs(want.astype(np.float64))
    err = np.abs(got[fin].astype(np.float64) - want[fin].astype(np.float64))
    worst = float(np.max(err - bound[fin])) if err.size else -1.0
    assert worst <= 1e-30, (op, k, "error beyond the window-local bound", worst)


def _spiky(b: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, n), dtype=np.float32)
    x[0, n // 3] = np.inf
    x[1 % b, n // 2] = np.nan
    x[2 % b, n // 4] = np.float32(1e30)          # huge but finite: must not leak
    x[3 % b, 100] = -np.inf
    x[3 % b, 100 + min(n - 101, 40)] = np.inf    # windows holding both: NaN
    x[4 % b, n - 3] = np.inf                     # at the end of a signal: the next
    x[5 % b, n - 1] = np.float32(-3e29)          # signal (flat view) must not see it
    return x


@pytest.mark.parametrize("k", [34, 65, 100, 255, 256, 511, 1000, 2049, 2050, 4097, 8192])
@pytest.mark.parametrize("n", [32 * 1061, 9001])   # aligned, and unaligned (flat view)
def test_fast_sums_window_local(k, n):
    b = 32 if n % 32 else 6
    x = _spiky(b, n, 4242 + k + n)
    xd = torch.from_numpy(x).cuda()
    for op, fn in (("sum", sc.sliding_window_sum), ("avg", sc.sliding_window_mean)):
        want = O.pool_batched(x, k, op)
        got = fn(xd, k)[0].cpu().numpy()
        _check(got, want, x, k, op)


@pytest.mark.parametrize("k", [100, 255, 2049, 3000])
def test_fast_sums_small_after_large(k):
    """Small-valued windows right after 1e30 samples in the same tile keep
    their own precision (a tile-anchored prefix difference would return
    garbage of order 1e30 * eps for them)."""
    n = 32 * 512
    x = np.full((2, n), np.float32(1e-3), dtype=np.float32)
    x[:, 10:20] = np.float32(1e30)
    x[1, 30] = np.float32(-1e30)
    xd = torch.from_numpy(x).cuda()
    want = O.pool_batched(x, k, "sum")
    got = sc.sliding_window_sum(xd, k)[0].cpu().numpy()
    _check(got, want, x, k, "sum")
    # windows after the spikes: exactly k * 1e-3 up to float32 rounding
    tail = got[:, 40:]
    assert np.allclose(tail, want[:, 40:], rtol=1e-5, atol=0)
