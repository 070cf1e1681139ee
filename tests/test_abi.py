"""The C-ABI library loads here (no GPU) and exports every symbol that
include/slideconv_b200.h declares, with host-only behaviour checked."""

import ctypes
import os
import re

import pytest

from oracle import slideconv_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "slideconv_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2310_05218_b200 import _lib
    return _lib.load()


def test_header_declares_the_expected_entry_points():
    syms = declared_symbols()
    for s in ("sc_pool1d_f32", "sc_conv1d_f32", "sc_conv2d_f32", "sc_conv2d_f64",
              "sc_conv2d_nchw_f32", "sc_im2col_f32", "sc_gemm_f32", "sc_pool1d_f32_host",
              "sc_conv2d_f32_host", "sc_version", "sc_last_error", "sc_pool1d_pair_f32",
              "sc_pool1d_pair_f32_host"):
        assert s in syms


def test_every_declared_symbol_is_exported(lib):
    from paper_2310_05218_b200 import _lib
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(raw, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_version_and_stage_counts(lib):
    assert lib.sc_version() == 10000
    for k in range(1, 300):
        assert lib.sc_pool1d_stages(0, k) == O.pool_sum_stages(k)
        assert lib.sc_pool1d_stages(2, k) == O.pool_max_stages(k)


def test_validation_happens_before_any_device_work(lib):
    from paper_2310_05218_b200 import _lib
    # window out of range -> SC_ERR_SHAPE with the reference's message
    rc = lib.sc_pool1d_f32(0, None, 1, 2, 3, 0, None, None)
    assert rc == _lib.SC_ERR_SHAPE
    assert "window 3 out of range for length 2" in _lib.last_error()
    assert lib.sc_pool1d_f32(7, None, 1, 8, 3, 0, None, None) == _lib.SC_ERR_ARG
    assert lib.sc_conv2d_f32(None, 1, 3, 3, None, 4, 2, 0, None, None) == _lib.SC_ERR_SHAPE
    assert "exceeds input" in _lib.last_error()
    assert lib.sc_conv2d_nchw_f32(None, 1, 1, 1, 1, None, 1, 5, 5, 1, 0, None, None) == \
        _lib.SC_ERR_SHAPE
    assert lib.sc_im2col_f32(None, 3, 3, 4, 1, 0, 0, None, None) == _lib.SC_ERR_SHAPE
    # empty batches are a no-op
    assert lib.sc_pool1d_f32(0, None, 0, 8, 3, 0, None, None) == 0


def test_rowband_abi_validates_before_touching_devices(lib):
    import ctypes

    from paper_2310_05218_b200 import _lib
    h = ctypes.c_void_p()
    devs = (ctypes.c_int * 1)(0)
    assert lib.sc_rowband_create(0, devs, ctypes.byref(h)) == _lib.SC_ERR_ARG
    assert h.value is None
    assert lib.sc_rowband_create(1, devs, None) == _lib.SC_ERR_ARG
    assert lib.sc_rowband_conv2d_f32(None, None, None, 8, None, 3, 3, 0, None, None, 0) == \
        _lib.SC_ERR_ARG
    assert lib.sc_rowband_destroy(None) == 0
