"""BASELINE config 5 at full size: one 65,536 x 65,536 image, 7x7, valid --
the exact launch the bench times, plus the G = 2 / 4 / 8 row-band launches a
rank issues (its rows + the kh - 1 = 6 halo rows).

The whole 16 GiB image is too large for the float32 oracle in one piece, but
output row r depends only on input rows r .. r+6 and columns c .. c+6
(reference.py:15-23), so any (rows x cols) window of the output is checked
exactly by running the oracle on the matching input window.  Windows sampled:
the first and last rows, every G = 2 / 4 / 8 band edge (g * 8192 +- 515),
and windows straddling row-segment boundaries of the tiling the launch picked
(sc_conv2d_segment_rows; the 4-column kernel's wave model, conv2d.cu
cols4_rows).  Columns: the first and last 4,102 and one interior range.
Exact mode must be bit-identical; fast mode within 1e-5 * 7 normwise.
The band launches must reproduce the whole-image output bit for bit.
"""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from paper_2310_05218_b200 import _lib, _ops
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu

H = W = 65536
K = 7
OH = H - K + 1
WIN_R, WIN_C = 1024, 4096


@pytest.fixture(scope="module")
def cfg5():
    free, _ = torch.cuda.mem_get_info()
    if free < 70 * (1 << 30):
        pytest.skip("needs ~70 GiB of free device memory")
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    x = torch.empty((H, W), device=dev)
    for r0 in range(0, H, 8192):
        x[r0:r0 + 8192].uniform_(-1, 1, generator=gen)
    f = (np.random.default_rng([0x5EED, 5, 0xFFFF]).standard_normal((K, K), dtype=np.float32)
         / np.float32(K)).astype(np.float32)
    ye = torch.empty((OH, OH), device=dev)
    yf = torch.empty((OH, OH), device=dev)
    _ops.conv2d_into(x, f, ye, exact=True)
    _ops.conv2d_into(x, f, yf, exact=False)
    torch.cuda.synchronize()
    yield x, f, ye, yf
    del x, ye, yf
    torch.cuda.empty_cache()


def _row_windows():
    lib = _lib.load()
    starts = {0, OH - WIN_R}
    for g in range(1, 8):                       # G = 8 band edges (G = 2 / 4 are a subset)
        starts.add(g * (H // 8) - WIN_R // 2)
    for exact in (0, 1):
        seg = int(lib.sc_conv2d_segment_rows(1, H, W, K, K, exact))
        assert seg > 0, "config 5 should run the 4-column kernel"
        for m in (1, (OH // seg) // 2, OH // seg - 1):
            if 0 < m * seg < OH:
                starts.add(min(OH - WIN_R, max(0, m * seg - WIN_R // 2)))
    return sorted(starts)


def _check_window(x, f, ye, yf, r0, c0):
    xin = x[r0:r0 + WIN_R + K - 1, c0:c0 + WIN_C + K - 1].cpu().numpy()
    want = O.conv2d(xin, f)
    got_e = ye[r0:r0 + WIN_R, c0:c0 + WIN_C].cpu().numpy()
    got_f = yf[r0:r0 + WIN_R, c0:c0 + WIN_C].cpu().numpy()
    assert np.array_equal(got_e, want), ("exact", r0, c0)
    assert O.normwise_error(got_f, want) <= O.north_star_tol(K), ("fast", r0, c0)


def test_config5_full_image_sampled_windows(cfg5):
    x, f, ye, yf = cfg5
    rng = np.random.default_rng(55)
    for r0 in _row_windows():
        for c0 in (0, OH - WIN_C, int(rng.integers(1, OH - WIN_C))):
            _check_window(x, f, ye, yf, r0, c0)


@pytest.mark.parametrize("g", [2, 4, 8])
def test_config5_band_launches_equal_whole(cfg5, g):
    x, f, ye, yf = cfg5
    rows = H // g
    for exact, whole in ((True, ye), (False, yf)):
        yb = torch.empty_like(whole)
        for b in range(g):                       # exactly one rank's launch per band
            a = b * rows
            if b < g - 1:
                _ops.conv2d_into(x[a:a + rows + K - 1], f, yb[a:a + rows], exact=exact)
            else:
                _ops.conv2d_into(x[a:], f, yb[a:], exact=exact)
        torch.cuda.synchronize()
        assert torch.equal(yb, whole), (g, exact)
        del yb
    # oracle at the band edges of the band launches themselves (same data)
    for b in range(1, g):
        _check_window(x, f, ye, yf, b * rows - WIN_R // 2, OH - WIN_C)
