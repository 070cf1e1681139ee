"""Pin the CPU oracle (oracle/slideconv_oracle.py) to the REAL reference's outputs.

The golden vectors were produced by tests/golden/make_golden.py importing the
reference package; here the restated oracle must reproduce every one of them
bit-for-bit (same float32 operation order), plus the reference's integer
tables (analytic counters, pooling stage counts, kernel selection).
"""

import json
import os

import numpy as np
import pytest

from oracle import slideconv_oracle as O
from tests.golden.recipes import RECIPES, make_inputs
from tests.golden.golden_io import GOLD, SMALL, sha, oracle_eval


@pytest.mark.parametrize("name", sorted(RECIPES))
def test_oracle_matches_reference_golden(name):
    r = RECIPES[name]
    x, f = make_inputs(r)
    y, extra = oracle_eval(r, x, f)
    g = GOLD[name]
    assert list(y.shape) == g["shape"]
    assert y.dtype.str == g["dtype"]
    if name in SMALL:
        assert np.array_equal(y, SMALL[name], equal_nan=True)
    assert sha(y) == g["sha256"], name
    if "stages" in g:
        assert extra == g["stages"]
    if "counters" in g:
        assert list(extra) == g["counters"]


def test_counter_table():
    for lanes, h, w, kh, kw, variant, macs, slides, loads, im2col in GOLD["__counters__"]:
        assert O.analytic_counters(variant, h, w, kh, kw, lanes) == (macs, slides, loads, im2col)


def test_pool_stage_table():
    for k, s_sum, s_max in GOLD["__pool_stages__"]:
        assert O.pool_sum_stages(k) == s_sum
        assert O.pool_max_stages(k) == s_max
        assert O.sliding_window_sum(np.zeros(300, np.float32), k)[1] == s_sum
        assert O.sliding_window_max(np.zeros(300, np.float32), k)[1] == s_max


def test_nchw_composition_close_to_f64():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 8, 12, 13), dtype=np.float32)
    w = (rng.standard_normal((5, 8, 3, 3), dtype=np.float32) / np.float32(np.sqrt(72))).astype(np.float32)
    a = O.conv2d_nchw(x, w, 1)
    b = O.conv2d_nchw_f64(x, w, 1)
    assert a.shape == (2, 5, 12, 13)
    assert O.normwise_error(a, b) < 1e-6


def test_rowband_equals_whole_bitwise():
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (203, 150)).astype(np.float32)
    f = rng.standard_normal((7, 7), dtype=np.float32)
    whole = O.conv2d(x, f)
    for g in (1, 2, 3, 4, 8):
        assert np.array_equal(O.rowband_conv2d(x, f, g), whole)


def test_im2col_equals_direct_bitwise():
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (33, 47)).astype(np.float32)
    f = rng.uniform(-1, 1, (5, 4)).astype(np.float32)
    assert np.array_equal(O.conv2d_im2col(x, f), O.conv2d(x, f))
