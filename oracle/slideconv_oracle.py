"""CPU oracle for the sliding-window conv/pool hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's arithmetic
(arXiv 2310.05218 `slideconv`, pure Python + numpy).  It exists so that
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / reference
arm have a checker that travels to the GPU box (the reference tree does not).
The product package `paper_2310_05218_b200` never imports it.

Parity pin: every function below is checked bit-for-bit against golden vectors
produced by the *real* reference (`tests/golden/make_golden.py` imports
/root/reference/pkg/src in the build container and writes
`tests/golden/*.npz`; `tests/test_oracle_golden.py` replays them).

Each function cites the reference file:line whose arithmetic it restates.
The extensions the reference does not have (batching, average pooling, NCHW
with zero padding, row bands) are composed from the restated primitives the
way SURVEY.md section 8(c) prescribes; those compositions are "parity by
construction", not pinned by a reference test.
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# geometry / counters  (tensor.py:49-102, kernels.py:52-120)


def out_dims(h: int, w: int, kh: int, kw: int) -> tuple[int, int]:
    """Valid geometry, tensor.py:66-72."""
    return h - kh + 1, w - kw + 1


def mac_count(h: int, w: int, kh: int, kw: int) -> int:
    """tensor.py:100-102: out_h*out_w*kh*kw."""
    oh, ow = out_dims(h, w, kh, kw)
    return oh * ow * kh * kw


def counted_offsets(kw: int, lanes: int) -> int:
    """kernels.py:57-59: offsets 1..kw-1 except V cost one shuffle each."""
    return sum(1 for j in range(1, kw) if j != lanes)


def compound_width(kw: int, lanes: int) -> int:
    """kernels.py:52-54."""
    return math.ceil((lanes + kw - 1) / lanes)


def analytic_counters(variant: str, h: int, w: int, kh: int, kw: int, lanes: int):
    """kernels.py:100-120 -> (macs, slides, loads, im2col_elems)."""
    oh, ow = out_dims(h, w, kh, kw)
    macs = oh * ow * kh * kw
    if variant == "im2col_gemm":
        return macs, 0, 0, oh * ow * kh * kw
    if variant == "naive":
        return macs, 0, 0, 0
    nvec = math.ceil(ow / lanes) if ow >= lanes else 0
    if nvec == 0:
        return macs, 0, 0, 0
    if variant == "slide_generic":
        return (macs, oh * kh * counted_offsets(kw, lanes) * nvec,
                oh * kh * nvec * (2 if kw > 1 else 1), 0)
    if variant == "slide_compound":
        m = compound_width(kw, lanes)
        return macs, oh * kh * nvec * m * (kw - 1), oh * kh * nvec * m, 0
    # custom3 / custom5
    return macs, h * counted_offsets(kw, lanes) * nvec, 2 * h * nvec, 0


def pool_sum_stages(k: int) -> int:
    """Stage count of pooling.py:37-51: floor(log2 k) + popcount(k) - 1."""
    return int(k).bit_length() - 1 + bin(int(k)).count("1") - 1


def pool_max_stages(k: int) -> int:
    """Stage count of pooling.py:67-76: floor(log2 k) + [k not a power of 2]."""
    p = int(k).bit_length() - 1
    return p + (1 if (1 << p) != k else 0)


# ---------------------------------------------------------------------------
# convolution  (reference.py:15-47, gemm.py:21-69)


def accumulate_taps(x: np.ndarray, f: np.ndarray, dtype=np.float32) -> np.ndarray:
    """reference.py:15-23: for (j, i) ascending: acc += dtype(f[j,i]) * x[j:, i:].

    Multiply then add (two rounded numpy ops, never fused), acc starts at 0.
    """
    x = np.asarray(x).astype(dtype, copy=False)
    kh, kw = f.shape
    oh, ow = out_dims(x.shape[0], x.shape[1], kh, kw)
    acc = np.zeros((oh, ow), dtype=dtype)
    for j in range(kh):
        for i in range(kw):
            tap = dtype(f[j, i])
            acc += tap * x[j:j + oh, i:i + ow]
    return acc


def conv2d(x, f) -> np.ndarray:
    """conv2d_reference / the `fast` backend of every slide variant
    (reference.py:26-30, kernels.py:212-217): float32 accumulate_taps."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    f = np.ascontiguousarray(np.asarray(f, dtype=np.float32))
    if x.ndim == 1:
        x = x.reshape(1, -1)
    if f.ndim == 1:
        f = f.reshape(1, -1)
    return accumulate_taps(x, f, np.float32)


def oracle_conv2d(x, f) -> np.ndarray:
    """reference.py:42-47: same formula in float64."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    f = np.atleast_2d(np.asarray(f, dtype=np.float64))
    return accumulate_taps(x, f, np.float64)


def conv2d_batched(x, f) -> np.ndarray:
    """Batch extension: one reference call per leading unit."""
    x = np.asarray(x, dtype=np.float32)
    lead = x.shape[:-2]
    flat = x.reshape((-1,) + x.shape[-2:])
    outs = [conv2d(img, f) for img in flat]
    return np.stack(outs).reshape(lead + outs[0].shape)


def im2col_2d(x, kh: int, kw: int) -> np.ndarray:
    """gemm.py:21-37: row (r*out_w + c) = patch x[r:r+kh, c:c+kw] flattened."""
    x = np.asarray(x, dtype=np.float32)
    oh, ow = out_dims(x.shape[0], x.shape[1], kh, kw)
    cols = np.empty((oh * ow, kh * kw), dtype=np.float32)
    for j in range(kh):
        for i in range(kw):
            cols[:, j * kw + i] = x[j:j + oh, i:i + ow].reshape(-1)
    return cols


def gemm_k_ordered(a, b) -> np.ndarray:
    """gemm.py:40-59: c[m,n] accumulated over k ascending as rank-1 updates
    (mul then add).  The M/K blocking there does not change per-element order."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    c = np.zeros((a.shape[0], b.shape[1]), dtype=np.float32)
    for kk in range(a.shape[1]):
        c += a[:, kk:kk + 1] * b[kk:kk + 1, :]
    return c


def conv2d_im2col(x, f) -> np.ndarray:
    """gemm.py:62-69."""
    f = np.atleast_2d(np.asarray(f, dtype=np.float32))
    x = np.atleast_2d(np.asarray(x, dtype=np.float32))
    kh, kw = f.shape
    oh, ow = out_dims(x.shape[0], x.shape[1], kh, kw)
    return gemm_k_ordered(im2col_2d(x, kh, kw), f.reshape(kh * kw, 1)).reshape(oh, ow)


def conv2d_nchw(x, w, padding: int = 1) -> np.ndarray:
    """Multi-channel NCHW conv with zero padding (absent in the reference;
    SURVEY 8(a) a12).  Composed from the reference primitive: per (n, co) the
    output is sum over ci ascending of conv2d_reference(xpad[n, ci], w[co, ci]),
    acc starting at 0, one float32 add per ci."""
    x = np.asarray(x, dtype=np.float32)
    w = np.asarray(w, dtype=np.float32)
    n_, cin, h, wd = x.shape
    cout, cin2, kh, kw = w.shape
    assert cin == cin2
    p = int(padding)
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))
    oh, ow = out_dims(h + 2 * p, wd + 2 * p, kh, kw)
    out = np.zeros((n_, cout, oh, ow), dtype=np.float32)
    for n in range(n_):
        for co in range(cout):
            acc = np.zeros((oh, ow), dtype=np.float32)
            for ci in range(cin):
                acc += accumulate_taps(xp[n, ci], w[co, ci], np.float32)
            out[n, co] = acc
    return out


def conv2d_nchw_f64(x, w, padding: int = 1) -> np.ndarray:
    """Float64 ground truth for the NCHW composition (oracle_conv2d analogue)."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    p = int(padding)
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))
    n_, cin, hp, wp = xp.shape
    cout, _, kh, kw = w.shape
    oh, ow = out_dims(hp, wp, kh, kw)
    out = np.zeros((n_, cout, oh, ow), dtype=np.float64)
    for j in range(kh):
        for i in range(kw):
            patch = xp[:, :, j:j + oh, i:i + ow]               # n, ci, oh, ow
            out += np.einsum("nchw,oc->nohw", patch, w[:, :, j, i])
    return out


def rowband_conv2d(x, f, n_bands: int) -> np.ndarray:
    """Row-band evaluation: band g computes output rows
    [g*B, min((g+1)*B, oh)) from input rows [g*B, ... + kh - 1).  Banded ==
    whole-image bit-for-bit because each output row only reads its kh rows."""
    x = np.asarray(x, dtype=np.float32)
    f = np.atleast_2d(np.asarray(f, dtype=np.float32))
    kh = f.shape[0]
    h = x.shape[0]
    oh = h - kh + 1
    rows = h // n_bands
    parts = []
    for g in range(n_bands):
        r0 = g * rows
        r1 = (g + 1) * rows if g < n_bands - 1 else h
        o1 = min(r1, oh)
        if o1 > r0:
            parts.append(accumulate_taps(x[r0:o1 + kh - 1], f, np.float32))
    return np.concatenate(parts, axis=0)


# ---------------------------------------------------------------------------
# pooling  (pooling.py:28-78)


def sliding_window_sum(a, k: int) -> tuple[np.ndarray, int]:
    """pooling.py:28-53 on a 1-D float32 signal.

    Doubling S_2w(i) = S_w(i) + S_w(i+w) while 2w <= k, then combine the
    remaining bits of k largest first: acc(i) += S_b(i + width).
    """
    s1 = np.asarray(a, dtype=np.float32)
    n = s1.shape[0]
    parts = {1: s1}
    stages = 0
    w = 1
    while 2 * w <= k:
        prev = parts[w]
        parts[2 * w] = prev[:prev.shape[0] - w] + prev[w:]
        w *= 2
        stages += 1
    acc = parts[w]
    width = w
    b = w >> 1
    while b:
        if k & b:
            m = n - (width + b) + 1
            acc = acc[:m] + parts[b][width:width + m]
            width += b
            stages += 1
        b >>= 1
    return acc[:n - k + 1], stages


def sliding_window_max(a, k: int) -> tuple[np.ndarray, int]:
    """pooling.py:56-78: doubling max then one overlapping combine.
    np.maximum(a, b) returns b on ties (+0/-0) and NaN if either is NaN."""
    cur = np.asarray(a, dtype=np.float32)
    n = cur.shape[0]
    stages = 0
    w = 1
    while 2 * w <= k:
        cur = np.maximum(cur[:cur.shape[0] - w], cur[w:])
        w *= 2
        stages += 1
    if w < k:
        m = n - k + 1
        cur = np.maximum(cur[:m], cur[k - w:k - w + m])
        stages += 1
    return cur[:n - k + 1], stages


def sliding_window_mean(a, k: int) -> tuple[np.ndarray, int]:
    """Average pooling (absent in the reference):
    float32(sum) / float32(k), IEEE division."""
    s, stages = sliding_window_sum(a, k)
    return s / np.float32(k), stages


_POOL = {"sum": sliding_window_sum, "max": sliding_window_max, "avg": sliding_window_mean}


def pool_batched(x, k: int, op: str) -> np.ndarray:
    """Batch extension: one reference call per signal (row) of a 2-D array."""
    x = np.asarray(x, dtype=np.float32)
    fn = _POOL[op]
    return np.stack([fn(row, k)[0] for row in x.reshape(-1, x.shape[-1])]).reshape(
        x.shape[:-1] + (x.shape[-1] - k + 1,))


# ---------------------------------------------------------------------------
# error metrics  (reference.py:50-54, BASELINE.json north_star)


def relative_error(got, want) -> float:
    """reference.py:50-54: max |got-want| / max(1, |want|)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want)), initial=0.0))


def normwise_error(got, want) -> float:
    """||got - want||_2 / ||want||_2 (north-star tolerance metric)."""
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    den = float(np.linalg.norm(want))
    num = float(np.linalg.norm(got - want))
    return num / den if den > 0 else num


def north_star_tol(k: int, cin: int = 1) -> float:
    """1e-5 * k * sqrt(Cin) (BASELINE.json north_star)."""
    return 1e-5 * k * math.sqrt(cin)
