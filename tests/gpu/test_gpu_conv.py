"""2-D / 1-D convolution kernels vs the oracle: every TMA specialisation and
the runtime-(kh, kw) kernel, exact mode bit-identical, fast mode within
tolerance, BASELINE configs 1 / 3 / 5 (full size where the oracle allows,
size-independent properties otherwise), edge shapes."""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu
VM = sc.VectorModel(16)


def rand(seed, shape, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, shape).astype(np.float32)


@pytest.mark.parametrize("kh,kw", [(3, 3), (5, 5), (7, 7), (1, 7), (1, 3), (2, 2), (4, 6),
                                   (11, 11), (1, 1), (7, 1), (17, 17), (33, 33)])
@pytest.mark.parametrize("h,w", [(300, 516), (64, 128), (257, 4100), (40, 41), (13, 29)])
def test_shapes_exact_and_fast(kh, kw, h, w):
    if kh > h or kw > w:
        pytest.skip("filter larger than input")
    x = rand(h * 7 + w, (2, h, w))
    f = rand(kh * 31 + kw, (kh, kw))
    want = O.conv2d_batched(x, f)
    xd = torch.from_numpy(x).cuda()
    got = sc.conv2d_reference(xd, f, exact=True).cpu().numpy()
    assert np.array_equal(got, want)
    fast = sc.conv2d_reference(xd, f, exact=False).cpu().numpy()
    ref64 = np.stack([O.oracle_conv2d(img, f) for img in x])
    assert O.normwise_error(fast, ref64) <= O.north_star_tol(max(kh, kw))
    assert sc.relative_error(fast, ref64) <= 1e-5 * max(1, kh * kw / 64)


@pytest.mark.parametrize("kh,kw", [(51, 51), (64, 64), (2, 64), (64, 3), (21, 13), (37, 29)])
@pytest.mark.parametrize("n,h,w", [(1, 200, 300), (3, 70, 133), (40, 64, 64)])
def test_runtime_k_register_blocked_kernel(kh, kw, n, h, w):
    # conv2d_big.cu: the paper's large-filter sweep (11..51) and up to 64 x 64,
    # 4- and 8-warp tiles (small and large grids), exact and fast modes
    if kh > h or kw > w:
        pytest.skip("filter larger than input")
    x = rand(kh * 1000 + kw + n, (n, h, w))
    f = rand(kh + 77 * kw, (kh, kw))
    xd = torch.from_numpy(x).cuda()
    got = sc.conv2d_reference(xd, f, exact=True).cpu().numpy()
    assert np.array_equal(got, O.conv2d_batched(x, f))
    fast = sc.conv2d_reference(xd, f, exact=False).cpu().numpy()
    ref64 = np.stack([O.oracle_conv2d(img, f) for img in x])
    assert O.normwise_error(fast, ref64) <= O.north_star_tol(max(kh, kw))


@pytest.mark.parametrize("k", [5, 7])
@pytest.mark.parametrize("n,h,w", [(64, 261, 1031), (64, 261, 1030), (40, 300, 1100),
                                   (2, 3001, 2060)])
def test_four_column_kernels_on_large_grids(k, n, h, w):
    # conv2d_cols4_kernel<5 / 7>: grids of >= 2 waves of 512-column CTAs; odd
    # output pitch (per-column stores), even pitch with whole warps (STG.64
    # pairs) and with a partial last warp; tall images (the 7x7 segment
    # length search), partial last row segments
    x = rand(k + 700 + w, (n, h, w))
    f = rand(k + 701, (k, k))
    xd = torch.from_numpy(x).cuda()
    got = sc.conv2d_reference(xd, f, exact=True).cpu().numpy()
    assert np.array_equal(got, O.conv2d_batched(x, f))
    fast = sc.conv2d_reference(xd, f, exact=False).cpu().numpy()
    ref64 = np.stack([O.oracle_conv2d(img, f) for img in x[:2]])
    assert O.normwise_error(fast[:2], ref64) <= O.north_star_tol(k)


@pytest.mark.parametrize("k", [9, 11, 13, 15, 17, 21])
def test_rotating_4col_kernels(k):
    # conv2d_rot4_kernel<K>: large batches of images (>= one wave of 512-col CTAs)
    x = rand(k + 900, (24, 256, 600))
    f = rand(k + 901, (k, k))
    xd = torch.from_numpy(x).cuda()
    got = sc.conv2d_reference(xd, f, exact=True).cpu().numpy()
    assert np.array_equal(got, O.conv2d_batched(x, f))
    fast = sc.conv2d_reference(xd, f, exact=False).cpu().numpy()
    ref64 = np.stack([O.oracle_conv2d(img, f) for img in x[:3]])
    assert O.normwise_error(fast[:3], ref64) <= O.north_star_tol(k)


@pytest.mark.parametrize("exact", [True, False])
def test_runtime_k_nonfinite_inputs_match_reference(exact):
    # a zero-padded tap must never multiply an inf beyond the filter width
    x = rand(5, (1, 90, 140))
    x[0, 10, 60] = np.inf
    x[0, 50, 20] = np.nan
    f = rand(6, (19, 23))
    got = sc.conv2d_reference(torch.from_numpy(x).cuda(), f, exact=exact).cpu().numpy()
    want = O.conv2d_batched(x, f)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(np.isinf(got), np.isinf(want))
    m = np.isfinite(want)
    if exact:
        assert np.array_equal(got[m], want[m])
    else:
        assert np.allclose(got[m], want[m], rtol=1e-4, atol=1e-4)


def test_config3_one_image_full_size_both_filters():
    rng = np.random.default_rng([0x5EED, 3])
    img = rng.uniform(0, 1, (1, 4096, 4096)).astype(np.float32)
    for k, fn in ((3, sc.conv2d_custom3), (5, sc.conv2d_custom5)):
        f = (rng.standard_normal((k, k), dtype=np.float32) / np.float32(k)).astype(np.float32)
        want = O.conv2d_batched(img, f)
        got, c = fn(torch.from_numpy(img).cuda(), f, VM, exact=True)
        assert np.array_equal(got.cpu().numpy(), want)
        assert c.macs == 4096 * 0 + (4097 - k) ** 2 * k * k
        fast, _ = fn(img, f, VM)                   # host pipeline
        assert O.normwise_error(fast, want) <= O.north_star_tol(k)


def test_config1_full_size():
    rng = np.random.default_rng([0x5EED, 1])
    x = rng.uniform(-1, 1, (64, 1048576)).astype(np.float32)
    w = rng.standard_normal((1, 7), dtype=np.float32)
    want = O.conv2d(x, w)
    got, c = sc.conv2d_slide_generic(torch.from_numpy(x).cuda(), w, VM, exact=True)
    assert np.array_equal(got.cpu().numpy(), want)
    fast, _ = sc.conv2d_slide_generic(x, w, VM)
    assert O.normwise_error(fast, want) <= O.north_star_tol(7)
    # one signal through conv1d_slide == the batched row, bit for bit
    y1, _ = sc.conv1d_slide(x[5], w[0], VM, exact=True)
    assert np.array_equal(y1[0], want[5])


def test_config5_band_and_properties():
    # a 1030-row band of the 65536-wide image: oracle-checkable
    rng = np.random.default_rng([0x5EED, 5])
    x = rng.uniform(-1, 1, (1030, 65536)).astype(np.float32)
    f = (rng.standard_normal((7, 7), dtype=np.float32) / np.float32(7)).astype(np.float32)
    want = O.conv2d(x, f)
    xd = torch.from_numpy(x).cuda()
    got = sc.conv2d_reference(xd, f, exact=True).cpu().numpy()
    assert np.array_equal(got, want)
    fast = sc.conv2d_reference(xd, f, exact=False).cpu().numpy()
    assert O.normwise_error(fast, want) <= O.north_star_tol(7)
    # banded on the GPU == whole on the GPU (exact), 4 virtual bands
    plans = sc.plan_row_bands(1030, 7, 4)
    parts = [sc.conv2d_reference(xd[p.in_start:min(1030, p.in_stop + p.halo)], f, exact=True)
             for p in plans]
    assert np.array_equal(torch.cat(parts).cpu().numpy(), want)


def test_linearity_in_the_filter():
    rng = np.random.default_rng(12)
    x = torch.from_numpy(rng.uniform(-1, 1, (3, 200, 300)).astype(np.float32)).cuda()
    f = rng.uniform(-1, 1, (5, 5)).astype(np.float32)
    g = rng.uniform(-1, 1, (5, 5)).astype(np.float32)
    a, b = np.float32(0.75), np.float32(-1.5)
    lhs = sc.conv2d_reference(x, a * f + b * g).double()
    rhs = a * sc.oracle_conv2d(x.double(), f) + b * sc.oracle_conv2d(x.double(), g)
    assert sc.relative_error(lhs, rhs) < 1e-5 * 2.25


def test_unit_filter_identity_and_impulse():
    x = rand(0, (7, 9))
    assert np.array_equal(sc.conv2d_reference(x, np.array([[1.0]], np.float32)), x)
    for p in range(3, 13):
        xi = np.zeros(16, np.float32)
        xi[p] = 1.0
        y = sc.conv1d_reference(xi, [1.0, 2.0, 3.0]).ravel()
        for i in range(len(y)):
            assert y[i] == ([1.0, 2.0, 3.0][p - i] if 0 <= p - i < 3 else 0.0)


def test_oracle_conv2d_float64_on_gpu():
    x = rand(42, (64, 64))
    f = rand(43, (5, 5))
    got = sc.oracle_conv2d(x, f)
    assert got.dtype == np.float64
    assert np.array_equal(got, O.oracle_conv2d(x, f))


def test_host_pipeline_band_path_large_image():
    x = rand(77, (1, 5000, 4096))                     # 82 MB single image -> row bands
    f = rand(78, (7, 7))
    got = sc.conv2d_reference(x, f, exact=True)
    assert np.array_equal(got, O.conv2d_batched(x, f))


def test_host_pipeline_tall_filter_on_wide_rows(monkeypatch):
    """kh - 1 >= the rows one host chunk holds: bands carry >= 3 (kh - 1)
    output rows (host_stream.cu) and stay bit-identical to the whole image."""
    monkeypatch.setenv("SC_HOST_CHUNK_MB", "1")        # 1 MiB chunks = one 262,144-wide row
    x = rand(79, (1, 64, 262144))
    f = rand(80, (9, 9))
    got = sc.conv2d_reference(x, f, exact=True)
    assert np.array_equal(got, O.conv2d_batched(x, f))


def test_unaligned_device_pointer_uses_generic_path():
    x = torch.from_numpy(rand(3, (1, 200 * 400 + 1))).cuda()
    view = x[0, 1:].reshape(200, 400)                 # 4-byte aligned only
    f = rand(4, (3, 3))
    got = sc.conv2d_reference(view, f, exact=True).cpu().numpy()
    assert np.array_equal(got, O.conv2d(view.cpu().numpy(), f))
