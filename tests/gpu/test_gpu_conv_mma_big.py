"""Large-filter tensor-core conv (csrc/conv2d_mma_big.cu; fast mode,
SC_CONV_MMA_BIG read per call: 0 off, 1 cost model, 2 forced) against the
oracle (reference.py:15-23 restated in oracle/): north-star tolerance
1e-5 * k normwise on sampled row bands (banded evaluation is exact), the
whole output against the exact-mode kernels, ragged widths / segments /
batches, the non-finite fallback, and that exact mode never takes it."""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu
VM = sc.VectorModel(16)


def _fast(xd, f, mode, monkeypatch, rows=None):
    monkeypatch.setenv("SC_CONV_MMA_BIG", str(mode))
    if rows:
        monkeypatch.setenv("SC_MMA_BIG_ROWS", str(rows))
    else:
        monkeypatch.delenv("SC_MMA_BIG_ROWS", raising=False)
    y = sc.conv2d_slide_compound(xd, f, VM, exact=False)[0]
    torch.cuda.synchronize()
    return y.cpu().numpy()


def _bands(oh, kh, nb=3, rows=5):
    """a few bands of output rows: first, last, and evenly spread"""
    starts = sorted({0, max(0, oh - rows)} | {int(v) for v in np.linspace(0, max(0, oh - rows), nb)})
    return [(s, min(rows, oh - s)) for s in starts]


@pytest.mark.parametrize("shape,kh,kw,rows", [
    ((2, 200, 1300), 11, 11, None),      # two strips, the second mostly empty
    ((1, 300, 2100), 17, 17, 37),        # ragged segments
    ((3, 256, 512), 25, 25, None),       # the paper's image size, batch
    ((1, 130, 1027), 51, 51, None),      # w % 4 != 0: scalar row loads
    ((1, 400, 1100), 53, 57, 64),        # the largest window (ring nearly full), 4 K blocks
    ((2, 90, 3000), 13, 31, 9),          # tiny segments: the window wraps the ring often
    ((1, 700, 777), 33, 10, None),
    ((1, 600, 1500), 40, 3, None),       # tall, narrow filter (one K block)
    ((1, 200, 2300), 2, 40, None),
    ((5, 64, 64), 21, 21, None),         # 16 images side by side in one strip (5 present)
    ((32, 512, 512), 51, 51, None),      # the paper's sweep shape: two images per strip
    ((7, 100, 203), 15, 9, 30),          # packed, odd width (pitch 208), ragged last group
    ((3, 80, 520), 11, 57, None),        # two images, the widest filter
])
def test_forced_mma_matches_oracle(shape, kh, kw, rows, monkeypatch):
    rng = np.random.default_rng(kh * 100 + kw)
    x = rng.uniform(-1, 1, shape).astype(np.float32)
    f = (rng.standard_normal((kh, kw)) / np.sqrt(kh * kw)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    got = _fast(xd, f, 2, monkeypatch, rows)
    oh = shape[1] - kh + 1
    assert got.shape == (shape[0], oh, shape[2] - kw + 1)
    tol = O.north_star_tol(max(kh, kw))
    for s, n in _bands(oh, kh):
        want = O.conv2d_batched(x[:, s:s + n + kh - 1], f)   # exact on a band (reference.py:19-22)
        assert O.normwise_error(got[:, s:s + n], want) <= tol, (s, n)
    # the whole output against the exact-mode kernels (bit-identical to the oracle)
    ref = sc.conv2d_slide_compound(xd, f, VM, exact=True)[0].cpu().numpy()
    assert O.normwise_error(got, ref) <= tol
    assert np.max(np.abs(got - ref)) <= 64 * tol * np.max(np.abs(ref))


def test_nonfinite_inputs_fall_back_per_cta(monkeypatch):
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (2, 300, 2100)).astype(np.float32)
    x[0, 17, 200] = np.inf
    x[1, 250, 1030] = np.nan
    x[1, 10, 2000] = -np.inf
    x[0, 120, 77] = 1e30
    x[0, 200, 1500] = 1e-42          # subnormal: outside what the split carries
    f = (rng.standard_normal((19, 23)) / 20).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    got = _fast(xd, f, 2, monkeypatch, 40)
    want = _fast(xd, f, 0, monkeypatch)          # the FFMA kernels (reference inf / NaN pattern)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(np.isinf(got), np.isinf(want))
    fin = np.isfinite(want)
    assert O.normwise_error(got[fin], want[fin]) <= O.north_star_tol(23)


def test_cost_model_and_exact_mode(monkeypatch):
    lib_calls = []
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (4, 1024, 1024)).astype(np.float32)
    f = (rng.standard_normal((25, 25)) / 25).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    auto = _fast(xd, f, 1, monkeypatch)
    forced = _fast(xd, f, 2, monkeypatch)
    off = _fast(xd, f, 0, monkeypatch)
    assert np.array_equal(auto, forced)            # the model picks the tensor-core kernel here
    assert not np.array_equal(auto, off)
    assert O.normwise_error(auto, off) <= O.north_star_tol(25)
    # exact mode is never served by it
    monkeypatch.setenv("SC_CONV_MMA_BIG", "2")
    band = sc.conv2d_slide_compound(xd[:1, :40], f, VM, exact=True)[0].cpu().numpy()
    assert np.array_equal(band, O.conv2d_batched(x[:1, :40], f))
    # small problems stay on the FFMA kernels under the model
    xs = torch.from_numpy(x[:1, :512, :512].copy()).cuda()
    assert np.array_equal(_fast(xs, f, 1, monkeypatch), _fast(xs, f, 0, monkeypatch))


def test_host_pipeline_with_large_filter(monkeypatch):
    """numpy in -> numpy out: the host pipeline's chunks (one image each here)
    go through the same dispatch and cost model"""
    rng = np.random.default_rng(77)
    x = rng.uniform(-1, 1, (3, 1100, 2048)).astype(np.float32)
    f = (rng.standard_normal((25, 25)) / 25).astype(np.float32)
    monkeypatch.setenv("SC_CONV_MMA_BIG", "1")
    monkeypatch.setenv("SC_HOST_CHUNK_MB", "32")     # chunks of whole images
    got = sc.conv2d_slide_compound(x, f, VM, exact=False)[0]
    assert isinstance(got, np.ndarray) and got.shape == (3, 1076, 2024)
    monkeypatch.setenv("SC_CONV_MMA_BIG", "0")
    ref = sc.conv2d_slide_compound(x, f, VM, exact=False)[0]
    assert not np.array_equal(got, ref)               # the tensor-core kernel did run
    assert O.normwise_error(got, ref) <= O.north_star_tol(25)
    want = O.conv2d_batched(x[:, 500:500 + 4 + 24], f)
    assert O.normwise_error(got[:, 500:504], want) <= O.north_star_tol(25)
