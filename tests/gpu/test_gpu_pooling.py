"""Pooling kernels vs the oracle: BASELINE config 2 at full size, every
dispatch branch (register doubling static/runtime k, float64 tile prefix,
global passes), ragged shapes, NaN / signed-zero semantics, host pipeline."""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu

FNS = {"sum": sc.sliding_window_sum, "max": sc.sliding_window_max, "avg": sc.sliding_window_mean}


@pytest.fixture(scope="module")
def cfg2():
    rng = np.random.default_rng([0x5EED, 2])
    x = rng.standard_normal((256, 262144), dtype=np.float32)
    return x, torch.from_numpy(x).cuda()


@pytest.mark.parametrize("k", [16, 3, 64, 255])
@pytest.mark.parametrize("op", ["max", "sum", "avg"])
def test_config2_full_size(cfg2, op, k):
    x, xd = cfg2
    want = O.pool_batched(x, k, op)
    fast, st = FNS[op](xd, k)
    fast = fast.cpu().numpy()
    assert st == (O.pool_max_stages(k) if op == "max" else O.pool_sum_stages(k))
    if op == "max":
        assert np.array_equal(fast, want)
    else:
        assert O.normwise_error(fast, want) <= O.north_star_tol(k)
        if k in (16, 3):                    # register doubling: bit-exact even in fast mode
            assert np.array_equal(fast, want)
    exact, _ = FNS[op](xd, k, exact=True)
    assert np.array_equal(exact.cpu().numpy(), want)


@pytest.mark.parametrize("k", list(range(1, 40)) + [47, 63, 64, 65, 100, 127, 128, 129, 200, 255,
                                                     256, 257, 300, 511, 512, 1000, 4097, 9000])
@pytest.mark.parametrize("n", [12_345, 8192, 544])
def test_every_window_branch(k, n):
    rng = np.random.default_rng(k)
    n = n + (k if n == 12_345 else 0)          # ragged lengths hit the striped kernel,
    if k > n:                                   # multiples of 32 the TMA kernel
        pytest.skip("window longer than the signal")
    x = rng.standard_normal((3, n), dtype=np.float32)
    xd = torch.from_numpy(x).cuda()
    for op in ("sum", "max", "avg"):
        want = O.pool_batched(x, k, op)
        got = FNS[op](xd, k)[0].cpu().numpy()
        got_exact = FNS[op](xd, k, exact=True)[0].cpu().numpy()
        assert np.array_equal(got_exact, want), (op, k)
        if op == "max":
            assert np.array_equal(got, want)
        else:
            assert O.normwise_error(got, want) <= O.north_star_tol(k)


@pytest.mark.parametrize("n,k", [(1, 1), (5, 5), (7, 3), (31, 16), (32, 16), (33, 16),
                                 (497, 16), (498, 16), (1000, 255), (255, 255)])
def test_ragged_and_tiny_signals(n, k):
    rng = np.random.default_rng(n * 1000 + k)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    for op in ("sum", "max", "avg"):
        y, _ = FNS[op](x, k, exact=True)
        assert y.shape == (n - k + 1,)
        assert np.array_equal(y, O.pool_batched(x[None], k, op)[0])


# pool_block.cu runtime-K kernel (two block tilings): every window 33..512
# that is not B - 1 / B, on aligned signals long enough for several tiles
@pytest.mark.parametrize("k", [33, 34, 35, 47, 48, 49, 62, 65, 66, 95, 96, 97, 126, 129, 130,
                               160, 191, 192, 193, 254, 257, 258, 320, 383, 384, 385, 450, 510])
def test_block_max_runtime_window(k):
    rng = np.random.default_rng(7000 + k)
    x = rng.standard_normal((3, 32 * 1061), dtype=np.float32)
    x[1, ::7] = np.float32(2.5)                  # many exact ties
    want = O.pool_batched(x, k, "max")
    xd = torch.from_numpy(x).cuda()
    assert np.array_equal(sc.sliding_window_max(xd, k)[0].cpu().numpy(), want)
    assert np.array_equal(sc.sliding_window_max(xd, k, exact=True)[0].cpu().numpy(), want)


# pool_exact.cu: exact (bit-identical) sums / averages for 32 < k <= 512 on
# aligned signals -- the reference's doubling + largest-bit-first fold per tile
@pytest.mark.parametrize("k", [33, 37, 48, 63, 65, 100, 127, 128, 129, 200, 255, 256, 257, 300,
                               383, 450, 511, 512])
def test_exact_sum_block_kernel(k):
    rng = np.random.default_rng(9000 + k)
    x = rng.standard_normal((3, 32 * 1061), dtype=np.float32)
    x[0, 5000] = np.inf
    x[1, 7000:7003] = np.nan
    x[2, ::13] = np.float32(1e30)               # large magnitudes: order matters
    xd = torch.from_numpy(x).cuda()
    for op in ("sum", "avg"):
        want = O.pool_batched(x, k, op)
        got = FNS[op](xd, k, exact=True)[0].cpu().numpy()
        assert np.array_equal(np.isnan(got), np.isnan(want)), (op, k)
        m = ~np.isnan(want)
        assert np.array_equal(got[m].view(np.uint32), want[m].view(np.uint32)), (op, k)


# pool1d.cu launch_exact_big: exact sums / averages for k > 512 on aligned
# signals -- P_512 from the tile kernel, global doublings up to W, the kept
# partials of the bits in [512, W) folded by passes, the bits below 512 by the
# tile kernel reading the running fold (pooling.py:37-51, every add the same)
@pytest.mark.parametrize("k", [513, 600, 1000, 1023, 1024, 1025, 1536, 1537, 2048, 2560, 3000,
                               4095, 4096, 5000, 8191, 12289, 30000])
def test_exact_sum_wide_windows(k):
    rng = np.random.default_rng(9500 + k)
    x = rng.standard_normal((3, 32 * 1500), dtype=np.float32)
    x[0, 5000] = np.inf
    x[1, 7000:7003] = np.nan
    x[2, ::13] = np.float32(1e30)               # large magnitudes: order matters
    x[2, 1::13] = np.float32(-1e30)
    xd = torch.from_numpy(x).cuda()
    for op in ("sum", "avg"):
        want = O.pool_batched(x, k, op)
        got = FNS[op](xd, k, exact=True)[0].cpu().numpy()
        assert got.shape == want.shape
        assert np.array_equal(np.isnan(got), np.isnan(want)), (op, k)
        m = ~np.isnan(want)
        assert np.array_equal(got[m].view(np.uint32), want[m].view(np.uint32)), (op, k)


# edge geometries of the same path: window = signal length (one output),
# windows just past 512 / a power of two, single signal, odd batch counts
@pytest.mark.parametrize("b,n,k", [(1, 2048, 2048), (2, 3072, 3000), (5, 1024, 1024), (1, 1056, 513),
                                   (7, 4096, 4097 - 32), (3, 65536, 65535), (2, 8192, 1536 + 255)])
def test_exact_sum_wide_windows_edges(b, n, k):
    rng = np.random.default_rng(b * 100003 + n + k)
    x = rng.standard_normal((b, n), dtype=np.float32) * np.float32(1e3)
    xd = torch.from_numpy(x).cuda()
    for op in ("sum", "avg"):
        want = O.pool_batched(x, k, op)
        got = FNS[op](xd, k, exact=True)[0].cpu().numpy()
        assert got.shape == want.shape == (b, n - k + 1)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (op, b, n, k)


# signal length not a multiple of 32: the batch viewed as one flat signal
# (B L % 32 == 0), outputs straddling two signals dropped
@pytest.mark.parametrize("b,n", [(32, 4001), (64, 1031), (96, 2053), (32, 9001)])
@pytest.mark.parametrize("k", [34, 63, 64, 100, 127, 255, 256, 300, 511, 512, 1000, 1024, 1536, 2049,
                               3000])
def test_flat_batch_unaligned_signals(b, n, k):
    if k > n:
        pytest.skip("window longer than the signal")
    rng = np.random.default_rng(b * 7 + n + k)
    x = rng.standard_normal((b, n), dtype=np.float32)
    x[3, ::17] = np.float32(0.0)
    x[5, ::19] = np.float32(-0.0)
    xd = torch.from_numpy(x).cuda()
    for op in ("max", "sum", "avg"):
        want = O.pool_batched(x, k, op)
        got = FNS[op](xd, k)[0].cpu().numpy()
        if op == "max":
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (op, k)
        else:
            assert O.normwise_error(got, want) <= O.north_star_tol(k), (op, k)
            exact = FNS[op](xd, k, exact=True)[0].cpu().numpy()
            assert np.array_equal(exact.view(np.uint32), want.view(np.uint32)), (op, k)


def test_reference_kats():
    assert sc.sliding_window_sum([1, 2, 3, 4, 5], 3)[0].tolist() == [6, 9, 12]
    assert sc.sliding_window_max([3, 1, 4, 1, 5], 3)[0].tolist() == [4, 4, 5]
    x = np.arange(10, dtype=np.float32).reshape(1, 10)
    y, _ = sc.sliding_window_sum(x, 4)
    assert y.shape == (1, 7)
    y, st = sc.sliding_window_sum(np.arange(8, dtype=np.float32), 1)
    assert np.array_equal(y, np.arange(8, dtype=np.float32)) and st == 0


@pytest.mark.parametrize("n", [5000, 5024])
@pytest.mark.parametrize("k", [2, 3, 16, 17, 33, 40, 63, 64, 100, 127, 128, 200, 255, 256, 300,
                               400, 511, 512])
def test_max_nan_and_signed_zero_semantics(k, n):
    rng = np.random.default_rng(99 + k)
    x = rng.standard_normal((2, n), dtype=np.float32)
    x[:, ::97] = 0.0
    x[:, 5::89] = -0.0
    x[0, 1234] = np.nan
    x[1, 4000:4003] = np.nan
    x[0, 3000:3100:3] = -0.0                     # dense +0/-0 ties
    x[0, 3001:3100:3] = 0.0
    want = O.pool_batched(x, k, "max")
    got = sc.sliding_window_max(torch.from_numpy(x).cuda(), k)[0].cpu().numpy()
    assert np.array_equal(np.isnan(got), np.isnan(want))
    m = ~np.isnan(want)
    assert np.array_equal(got[m].view(np.uint32), want[m].view(np.uint32))  # +0 vs -0 too


def test_host_pipeline_multi_chunk_pageable_and_pinned():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((80, 262144), dtype=np.float32)     # 84 MB -> 2 chunks
    want = O.pool_batched(x, 16, "avg")
    assert np.array_equal(sc.sliding_window_mean(x, 16)[0], want)
    xp = sc.pinned_empty(x.shape)
    xp[...] = x
    assert np.array_equal(sc.sliding_window_mean(xp, 16)[0], want)


def test_host_pipeline_single_signal_larger_than_a_chunk():
    rng = np.random.default_rng(6)
    x = rng.standard_normal(20_000_000, dtype=np.float32)       # 80 MB, segmented
    want = O.sliding_window_max(x, 255)[0]
    assert np.array_equal(sc.sliding_window_max(x, 255)[0], want)
    want = O.sliding_window_sum(x, 16)[0]
    assert np.array_equal(sc.sliding_window_sum(x, 16)[0], want)


def test_host_pipeline_window_wider_than_a_chunk():
    """k - 1 larger than the host pipeline's chunk: segments grow with k (at
    least 3 (k - 1) outputs each) instead of degenerating to one output per
    chunk (host_stream.cu)."""
    rng = np.random.default_rng(61)
    x = rng.standard_normal(4_000_000, dtype=np.float32)       # 16 MB, chunk 8 MB
    k = 3_000_000
    assert np.array_equal(sc.sliding_window_max(x, k)[0], O.sliding_window_max(x, k)[0])
    got = sc.sliding_window_sum(x, k, exact=True)[0]
    assert np.array_equal(got, O.sliding_window_sum(x, k)[0])


def test_batch_leading_dims_and_empty_batch():
    x = np.random.default_rng(1).standard_normal((2, 3, 100), dtype=np.float32)
    y, _ = sc.sliding_window_sum(x, 5)
    assert y.shape == (2, 3, 96)
    assert np.array_equal(y.reshape(6, 96), O.pool_batched(x.reshape(6, 100), 5, "sum"))
    y, _ = sc.sliding_window_sum(np.zeros((0, 10), np.float32), 3)
    assert y.shape == (0, 8)


@pytest.mark.parametrize("k", [3, 5, 7, 9, 11, 13, 17, 31, 33])
def test_average_division_is_ieee(k):
    # avg = float32(sum) / float32(k); the TMA kernel divides by a reciprocal
    # plus an FMA correction, which must be bit-identical to IEEE division
    rng = np.random.default_rng(1000 + k)
    scale = np.exp(rng.uniform(-60, 60, (8, 1))).astype(np.float32)
    x = (rng.standard_normal((8, 16384), dtype=np.float32) * scale).astype(np.float32)
    got = sc.sliding_window_mean(torch.from_numpy(x).cuda(), k)[0].cpu().numpy()
    assert np.array_equal(got, O.pool_batched(x, k, "avg"))
