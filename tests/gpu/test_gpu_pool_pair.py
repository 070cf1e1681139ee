"""Fused sum/average + max pooling (sc_pool1d_pair_f32 / _host): each output
must be bit-identical to the single-op entry point (hence to the oracle:
pooling.py:28-53 and :56-78 in exact mode) on the fused TMA windows, on the
fallback shapes, with NaN / signed zeros, and through the host pipeline."""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu


def _same(a, b):
    """bit-identical (signed zeros included); NaNs match by position (their
    payload / sign is not defined by the reference)"""
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    return (a.shape == b.shape and np.array_equal(na, nb)
            and np.array_equal(a[~na].view(np.uint32), b[~nb].view(np.uint32)))


@pytest.mark.parametrize("k", [16, 3, 64])
def test_config2_full_size_pair(k):
    rng = np.random.default_rng([0x5EED, 2])
    x = rng.standard_normal((256, 262144), dtype=np.float32)
    xd = torch.from_numpy(x).cuda()
    (ya, sa), (ym, sm) = sc.sliding_window_mean_max(xd, k)
    assert sa == O.pool_sum_stages(k) and sm == O.pool_max_stages(k)
    assert _same(ya.cpu().numpy(), O.pool_batched(x, k, "avg"))
    assert _same(ym.cpu().numpy(), O.pool_batched(x, k, "max"))
    (ys, _), (ym2, _) = sc.sliding_window_sum_max(xd, k)
    assert _same(ys.cpu().numpy(), O.pool_batched(x, k, "sum"))
    assert _same(ym2.cpu().numpy(), ym.cpu().numpy())


@pytest.mark.parametrize("k", list(range(1, 36)) + [63, 64, 65, 255, 600])
@pytest.mark.parametrize("n", [32 * 1061, 12_345, 544])
def test_pair_equals_single_ops_every_window(k, n):
    """fused windows (k = 2..33, 64 on n % 32 == 0) and every fallback"""
    if k > n:
        pytest.skip("window longer than the signal")
    rng = np.random.default_rng(31 * k + n)
    x = rng.standard_normal((3, n), dtype=np.float32)
    xd = torch.from_numpy(x).cuda()
    for exact in (False, True):
        (ys, _), (ym, _) = sc.sliding_window_sum_max(xd, k, exact=exact)
        (ya, _), (ym2, _) = sc.sliding_window_mean_max(xd, k, exact=exact)
        assert _same(ys.cpu().numpy(), sc.sliding_window_sum(xd, k, exact=exact)[0].cpu().numpy())
        assert _same(ya.cpu().numpy(), sc.sliding_window_mean(xd, k, exact=exact)[0].cpu().numpy())
        assert _same(ym.cpu().numpy(), O.pool_batched(x, k, "max"))
        assert _same(ym2.cpu().numpy(), ym.cpu().numpy())
        if exact:
            assert _same(ys.cpu().numpy(), O.pool_batched(x, k, "sum"))
            assert _same(ya.cpu().numpy(), O.pool_batched(x, k, "avg"))


@pytest.mark.parametrize("k", [2, 7, 16, 33, 64])
def test_pair_nan_inf_signed_zero(k):
    rng = np.random.default_rng(900 + k)
    x = rng.standard_normal((4, 32 * 257), dtype=np.float32)
    x[0, ::97] = np.nan
    x[1, ::131] = np.inf
    x[1, 5::263] = -np.inf
    x[2] = np.where(rng.random(x.shape[1]) < 0.5, np.float32(0.0), np.float32(-0.0))
    x[3, ::11] = 0.0
    x[3, 3::11] = -0.0
    xd = torch.from_numpy(x).cuda()
    (ya, _), (ym, _) = sc.sliding_window_mean_max(xd, k, exact=True)
    with np.errstate(invalid="ignore"):
        assert _same(ym.cpu().numpy(), O.pool_batched(x, k, "max"))
        assert _same(ya.cpu().numpy(), O.pool_batched(x, k, "avg"))


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("shape,k", [((64, 262144), 16), ((5, 40_000), 16), ((1, 30_000_000), 16),
                                     ((3, 12_345), 7), ((2, 9_000), 300)])
def test_pair_host_pipeline(shape, k, pinned, monkeypatch):
    """numpy in -> numpy out: chunks of signals, segments of one long signal
    (k - 1 overlap), pinned and pageable buffers"""
    if shape[1] >= 30_000_000:
        monkeypatch.setenv("SC_HOST_CHUNK_MB", "16")
    rng = np.random.default_rng(shape[1] + k)
    x = rng.standard_normal(shape, dtype=np.float32)
    if pinned:
        xp = sc.pinned_empty(shape)
        xp[...] = x
    else:
        xp = x
    (ya, sa), (ym, sm) = sc.sliding_window_mean_max(xp, k, exact=True)
    assert isinstance(ya, np.ndarray) and isinstance(ym, np.ndarray)
    assert ya.shape == ym.shape == (shape[0], shape[1] - k + 1)
    assert sa == O.pool_sum_stages(k) and sm == O.pool_max_stages(k)
    assert _same(ya, O.pool_batched(x, k, "avg"))
    assert _same(ym, O.pool_batched(x, k, "max"))


def test_pair_shapes_and_errors():
    x = np.arange(40, dtype=np.float32)
    (ys, _), (ym, _) = sc.sliding_window_sum_max(x, 4)
    assert ys.shape == ym.shape == (37,)
    assert _same(ys, O.pool_batched(x[None], 4, "sum")[0])
    assert _same(ym, O.pool_batched(x[None], 4, "max")[0])
    (ys, _), (ym, _) = sc.sliding_window_sum_max(x.reshape(1, -1), 4)
    assert ys.shape == ym.shape == (1, 37)
    with pytest.raises(sc.ShapeError):
        sc.sliding_window_sum_max(x, 0)
    with pytest.raises(sc.ShapeError):
        sc.sliding_window_mean_max(x, 41)


def test_pair_abi_argument_checks():
    from paper_2310_05218_b200 import _lib
    lib = _lib.load()
    x = torch.zeros((2, 64), device="cuda")
    y = torch.zeros((2, 61), device="cuda")
    y2 = torch.zeros((2, 61), device="cuda")
    p = lambda t: t.data_ptr()
    assert lib.sc_pool1d_pair_f32(_lib.POOL_MAX, p(x), 2, 64, 4, 0, p(y), p(y2), None) == _lib.SC_ERR_ARG
    assert lib.sc_pool1d_pair_f32(_lib.POOL_SUM, p(x), 2, 64, 4, 0, p(y), p(y), None) == _lib.SC_ERR_ARG
    assert lib.sc_pool1d_pair_f32(_lib.POOL_SUM, p(x), 2, 64, 65, 0, p(y), p(y2), None) == _lib.SC_ERR_SHAPE
    assert lib.sc_pool1d_pair_f32(_lib.POOL_SUM, p(x), 2, 64, 4, 5, p(y), p(y2), None) == _lib.SC_ERR_ARG
    assert lib.sc_pool1d_pair_f32(_lib.POOL_AVG, None, 0, 64, 4, 0, None, None, None) == 0
    assert lib.sc_pool1d_pair_f32(_lib.POOL_AVG, p(x), 2, 64, 4, 0, p(y), p(y2), None) == 0
    torch.cuda.synchronize()
