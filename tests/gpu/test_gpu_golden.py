"""Replay every reference golden vector through the GPU drop-in (C-ABI path).

EXACT mode must reproduce the reference's float32 outputs bit for bit (the
sha256 / arrays were produced by the reference itself); FAST mode must stay
within the north-star tolerance (1e-5 * k normwise) and the reference tests'
elementwise bound 1e-5 * max(1, k^2/64) against the float64 oracle."""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O
from tests.golden.golden_io import GOLD, SMALL, sha
from tests.golden.recipes import RECIPES, accept1_lanes, make_inputs

pytestmark = pytest.mark.gpu


def gpu_eval(r, x, f, exact):
    op = r["op"]
    vm = sc.VectorModel(r.get("lanes", 16), "fast")
    if op == "conv2d_reference":
        return sc.conv2d_reference(x, f, exact=exact), None
    if op == "oracle_conv2d":
        return sc.oracle_conv2d(x, f), None
    if op == "conv1d_reference":
        return sc.conv1d_reference(x, f, exact=exact), None
    if op == "conv1d_slide":
        return sc.conv1d_slide(x, f, vm, exact=exact)
    if op == "variant":
        return sc.run_variant(sc.KernelVariant(r["variant"]), x, f, vm, exact=exact)
    if op == "conv1d_batch":
        return sc.conv2d_slide_generic(x, np.asarray(f).reshape(1, -1), vm, exact=exact)[0], None
    if op == "conv2d_batch":
        kh, kw = f.shape
        return sc.run_variant(sc.select_kernel(kh, kw, vm), x, f, vm, exact=exact)[0], None
    if op in ("pool_sum", "pool_max", "pool_avg"):
        fn = {"pool_sum": sc.sliding_window_sum, "pool_max": sc.sliding_window_max,
              "pool_avg": sc.sliding_window_mean}[op]
        y, st = fn(np.atleast_2d(x), r["k"], exact=exact)
        return y, st
    if op == "im2col":
        return sc.conv2d_im2col(x, f), None
    if op == "accept1":
        v = accept1_lanes(r["t"])
        vm = sc.VectorModel(v, "fast")
        outs = [sc.run_variant(var, x, f, vm, exact=exact)
                for var in sc.applicable_variants(f.shape[0], f.shape[1], vm)
                if var is not sc.KernelVariant.IM2COL_GEMM]
        macs = O.mac_count(x.shape[0], x.shape[1], f.shape[0], f.shape[1])
        for y, c in outs:
            assert c.macs == macs
            assert np.array_equal(y, outs[0][0])
        return outs[0][0], None
    raise ValueError(op)


NAMES = sorted(RECIPES)


@pytest.mark.parametrize("name", NAMES)
def test_exact_mode_bit_identical_to_reference(name):
    r = RECIPES[name]
    x, f = make_inputs(r)
    y, extra = gpu_eval(r, x, f, exact=True)
    g = GOLD[name]
    y = np.asarray(y).reshape(g["shape"])
    if r["op"] == "im2col":           # cuBLAS accumulation order differs: tolerance only
        want = SMALL[name] if name in SMALL else None
        if want is not None:
            assert sc.relative_error(y, want) < 1e-5
        return
    if name in SMALL:
        assert np.array_equal(y, SMALL[name], equal_nan=True)
    assert sha(y) == g["sha256"]
    if "stages" in g:
        assert extra == g["stages"]
    if "counters" in g:
        assert [extra.macs, extra.slides, extra.loads, extra.im2col_elems] == g["counters"]


@pytest.mark.parametrize("name", [n for n in NAMES if RECIPES[n]["op"] not in ("oracle_conv2d",)])
def test_fast_mode_within_tolerance(name):
    r = RECIPES[name]
    x, f = make_inputs(r)
    y, _ = gpu_eval(r, x, f, exact=False)
    g = GOLD[name]
    y = np.asarray(y, dtype=np.float64).reshape(g["shape"])
    op = r["op"]
    if op in ("pool_sum", "pool_max", "pool_avg"):
        k = r["k"]
        want = O.pool_batched(np.atleast_2d(x), k, op[5:])
        if op == "pool_max":
            assert np.array_equal(y.astype(np.float32), want)    # max: always exact
        else:
            assert O.normwise_error(y, want) <= O.north_star_tol(k)
        return
    xx = np.asarray(x, np.float32)
    ff = np.atleast_2d(np.asarray(f, np.float32))
    if op == "conv1d_batch":
        want = O.oracle_conv2d(xx, ff)
    elif op == "conv2d_batch":
        want = np.stack([O.oracle_conv2d(img, ff) for img in xx])
    else:
        want = O.oracle_conv2d(np.atleast_2d(xx), ff)
    want = want.reshape(g["shape"])
    k = max(ff.shape)
    assert O.normwise_error(y, want) <= O.north_star_tol(k)
    if float(np.max(np.abs(xx), initial=0)) <= 1.0 and float(np.max(np.abs(ff))) <= 1.0:
        assert sc.relative_error(y, want) <= 1e-5 * max(1.0, ff.shape[0] * ff.shape[1] / 64.0)
