"""Multi-channel NCHW (config 4) and the im2col + cuBLAS contrast."""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu


def test_config4_full_size_within_tolerance():
    rng = np.random.default_rng([0x5EED, 4])
    x = rng.standard_normal((16, 64, 112, 112), dtype=np.float32)
    w = (rng.standard_normal((64, 64, 3, 3), dtype=np.float32) / np.float32(24.0)).astype(np.float32)
    got = sc.conv2d_nchw(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), 1).cpu().numpy()
    want = O.conv2d_nchw_f64(x, w, 1)
    assert O.normwise_error(got, want) <= O.north_star_tol(3, 64)


def test_config4_exact_matches_composed_oracle():
    rng = np.random.default_rng(41)
    x = rng.standard_normal((2, 64, 112, 112), dtype=np.float32)
    w = (rng.standard_normal((8, 64, 3, 3), dtype=np.float32) / np.float32(24.0)).astype(np.float32)
    got = sc.conv2d_nchw(x, w, 1, exact=True)
    assert np.array_equal(got, O.conv2d_nchw(x, w, 1))


def test_config4_full_size_exact_bit_identical():
    """Config 4 at full size (N 16, Cin = Cout = 64, 112^2, 3x3, pad 1) in
    exact mode against the composed oracle (per (n, co): sum over ci ascending
    of the reference's single-channel conv of the padded plane)."""
    rng = np.random.default_rng([0x5EED, 4])
    x = rng.standard_normal((16, 64, 112, 112), dtype=np.float32)
    w = (rng.standard_normal((64, 64, 3, 3), dtype=np.float32) / np.float32(24.0)).astype(np.float32)
    got = sc.conv2d_nchw(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), 1,
                         exact=True).cpu().numpy()
    want = O.conv2d_nchw(x, w, 1)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,cin,cout,h,w,k,p", [(1, 3, 5, 17, 23, 3, 1), (2, 7, 70, 33, 9, 3, 1),
                                                 (1, 4, 4, 10, 10, 5, 2), (1, 2, 3, 8, 8, 3, 0),
                                                 # tcgen05 bf16x3 path (Cin % 64, Cout % 64, W % 16):
                                                 # edge tiles, ragged H, several chunks / co-tiles
                                                 (2, 64, 64, 16, 32, 3, 1), (1, 64, 128, 21, 48, 3, 1),
                                                 (3, 128, 64, 9, 16, 3, 1), (1, 64, 64, 1, 16, 3, 1),
                                                 (2, 192, 128, 7, 48, 3, 1),
                                                 # weights-stationary (Cin 32 / 64): several
                                                 # column tiles with halos, 3 co-tiles, H = 1, 2
                                                 (2, 32, 64, 30, 224, 3, 1), (2, 32, 192, 17, 160, 3, 1),
                                                 (1, 64, 64, 2, 48, 3, 1), (3, 64, 128, 5, 96, 3, 1),
                                                 # weights-stationary, W % 16 != 0: one
                                                 # column tile padded to 16 pixels
                                                 (2, 64, 64, 20, 56, 3, 1), (3, 64, 128, 9, 28, 3, 1),
                                                 (1, 32, 64, 7, 12, 3, 1), (2, 64, 64, 5, 100, 3, 1),
                                                 (1, 32, 64, 3, 4, 3, 1),
                                                 # pixel-stationary (Cin 128 / 192), padded
                                                 # last column tile
                                                 (2, 128, 64, 11, 56, 3, 1), (1, 128, 128, 9, 28, 3, 1),
                                                 (1, 192, 64, 5, 20, 3, 1), (2, 128, 64, 3, 4, 3, 1),
                                                 # Cin % 64 != 0: zero-padded channel chunk
                                                 (2, 32, 64, 16, 32, 3, 1), (3, 96, 64, 9, 16, 3, 1),
                                                 (2, 48, 64, 10, 56, 3, 1), (1, 160, 128, 6, 28, 3, 1),
                                                 (1, 8, 64, 5, 16, 3, 1),
                                                 # Cout % 64 != 0: zero-padded output tile
                                                 (2, 64, 32, 9, 48, 3, 1), (1, 64, 96, 7, 56, 3, 1),
                                                 (2, 128, 40, 5, 32, 3, 1), (1, 32, 8, 6, 16, 3, 1),
                                                 # Cin % 8 != 0 -> CUDA-core kernel
                                                 (2, 3, 64, 12, 32, 3, 1)])
def test_nchw_shapes(n, cin, cout, h, w, k, p):
    rng = np.random.default_rng(n + cin + cout + h + w)
    x = rng.standard_normal((n, cin, h, w), dtype=np.float32)
    wt = rng.standard_normal((cout, cin, k, k), dtype=np.float32)
    fast = sc.conv2d_nchw(x, wt, p)
    assert O.normwise_error(fast, O.conv2d_nchw_f64(x, wt, p)) <= O.north_star_tol(k, cin)
    exact = sc.conv2d_nchw(x, wt, p, exact=True)
    assert np.array_equal(exact, O.conv2d_nchw(x, wt, p))


def test_im2col_exact_and_gemm():
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, (33, 47)).astype(np.float32)
    c = sc.CostCounters()
    cols = sc.im2col_2d(x, 5, 4, c)
    assert np.array_equal(cols, O.im2col_2d(x, 5, 4))
    assert c.im2col_elems == cols.size
    a = rng.uniform(-1, 1, (70, 30)).astype(np.float32)
    b = rng.uniform(-1, 1, (30, 9)).astype(np.float32)
    got = sc.gemm(a, b)
    assert np.allclose(got, a.astype(np.float64) @ b, rtol=0, atol=1e-5)
    kat = sc.im2col_2d(np.arange(1, 10, dtype=np.float32).reshape(3, 3), 2, 2)
    assert kat[0].tolist() == [1, 2, 4, 5]


def test_conv2d_im2col_matches_direct():
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (300, 700)).astype(np.float32)
    f = rng.uniform(-1, 1, (5, 5)).astype(np.float32)
    c = sc.CostCounters()
    y = sc.conv2d_im2col(x, f, c)
    assert sc.relative_error(y, O.oracle_conv2d(x, f)) < 1e-5
    assert c.im2col_elems == 296 * 696 * 25
    y2, c2 = sc.run_variant(sc.KernelVariant.IM2COL_GEMM, x, f, sc.VectorModel(16))
    assert c2.im2col_elems == c.im2col_elems


@pytest.mark.parametrize("shape", [(1, 64, 16, 32), (2, 32, 20, 112), (1, 128, 16, 32), (2, 64, 9, 56)])
def test_nonfinite_inputs(shape):
    # exact mode reproduces the reference's inf / NaN pattern bit for bit; the
    # fast tensor-core paths (weights-stationary for Cin <= 64, pixel-
    # stationary for Cin = 128) recompute the tiles whose inputs the bf16
    # split cannot carry with FMAs, so the pattern matches there too and every
    # finite output stays within tolerance (nchw_ws.cu / nchw_tc.cu)
    n, cin, h, w_ = shape
    rng = np.random.default_rng(12 + cin + h)
    x = rng.standard_normal(shape, dtype=np.float32)
    x[0, 5, 7, 9] = np.inf
    x[0, cin - 3, 2, w_ - 2] = np.nan
    x[n - 1, 1, h - 1, 0] = -np.inf
    x[n - 1, 2, h // 2, w_ // 2] = np.float32(3e38)        # |x| >= 2^127: not carried by the split
    w = (rng.standard_normal((64, cin, 3, 3), dtype=np.float32) / np.float32(3 * np.sqrt(cin))).astype(np.float32)
    want = O.conv2d_nchw(x, w, 1)
    exact = sc.conv2d_nchw(x, w, 1, exact=True)
    assert np.array_equal(exact, want, equal_nan=True)
    fast = sc.conv2d_nchw(x, w, 1)
    assert np.array_equal(np.isnan(fast), np.isnan(want))
    assert np.array_equal(np.isposinf(fast), np.isposinf(want))
    assert np.array_equal(np.isneginf(fast), np.isneginf(want))
    good = np.isfinite(want)
    ref64 = O.conv2d_nchw_f64(np.where(np.isfinite(x), x, 0).astype(np.float32), w, 1)
    assert np.allclose(fast[good], ref64[good], rtol=1e-4, atol=1e-4 * float(np.abs(ref64[good]).max()))
