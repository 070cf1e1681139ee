"""Row bands across GPUs through the C ABI (sc_rowband_create / _conv2d_f32
/ _destroy, NCCL communicators from ncclCommInitAll, one host thread):
bit-identical to the oracle on the whole image (reference.py:15-23: output
row r reads input rows r .. r+kh-1 only).  One GPU: a single band (the
context, comm stream and completion polling run; no exchange).  Two or more
GPUs: real NCCL halos over NVLink (skipped on a one-GPU box)."""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu


def _run(devices, h, w, kh, kw, exact):
    rng = np.random.default_rng([h, w, kh, kw, len(devices)])
    x = rng.uniform(-1, 1, (h, w)).astype(np.float32)
    f = (rng.standard_normal((kh, kw), dtype=np.float32) / np.float32(kh)).astype(np.float32)
    plans = sc.plan_row_bands(h, kh, len(devices))
    bufs = []
    for p, d in zip(plans, devices):
        rows = p.in_stop - p.in_start
        b = sc.alloc_band(rows, w, kh, device=f"cuda:{d}")
        b[rows:] = float("nan")          # spare rows: overwritten by the halo (or unused)
        b[:rows] = torch.from_numpy(x[p.in_start:p.in_stop]).to(b.device)
        bufs.append(b)
    with sc.RowBandGroup(devices) as grp:
        ys = grp.conv2d(bufs, f, exact=exact)
        ys2 = grp.conv2d(bufs, f, exact=exact)           # the context is reusable
    got = np.concatenate([y.cpu().numpy() for y in ys])
    assert np.array_equal(got, np.concatenate([y.cpu().numpy() for y in ys2]))
    want = O.conv2d(x, f)
    if exact:
        assert np.array_equal(got, want)
    else:
        assert O.normwise_error(got, want) <= O.north_star_tol(kw)


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("h,w,kh,kw", [(300, 1024, 7, 7), (64, 4096, 3, 3), (50, 333, 5, 9)])
def test_rowband_abi_single_device(h, w, kh, kw, exact):
    _run([0], h, w, kh, kw, exact)


@pytest.mark.parametrize("exact", [True, False])
def test_rowband_abi_multi_device(exact):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (one band per GPU)")
    g = min(8, n)
    _run(list(range(g)), 1024 * g + 13, 8192, 7, 7, exact)


def test_rowband_abi_rejects_bad_bands():
    with sc.RowBandGroup([0]) as grp:
        with pytest.raises(ValueError):
            grp.conv2d([torch.zeros((10, 10))], np.ones((3, 3), np.float32))   # host tensor
        with pytest.raises(sc.ShapeError):
            grp.conv2d([torch.zeros((4, 64), device="cuda")], np.ones((7, 7), np.float32))
