"""Host-side behaviour of the drop-in API that needs no GPU: validation order
and exception classes (the reference's pytest.raises sites), kernel
selection, analytic counters, row-band planning."""

import numpy as np
import pytest

import paper_2310_05218_b200 as sc
from paper_2310_05218_b200.kernels import analytic_counters
from tests.golden.golden_io import GOLD


def test_select_kernel_table_matches_reference():
    for lanes, kh, kw, want in GOLD["__select__"]:
        assert sc.select_kernel(kh, kw, sc.VectorModel(lanes)).value == want


def test_counter_table_matches_reference():
    for lanes, h, w, kh, kw, variant, macs, slides, loads, im2col in GOLD["__counters__"]:
        c = analytic_counters(sc.KernelVariant(variant), sc.ConvShape(h, w, kh, kw),
                              sc.VectorModel(lanes))
        assert (c.macs, c.slides, c.loads, c.im2col_elems) == (macs, slides, loads, im2col)


def test_vector_model_validation():
    with pytest.raises(ValueError):
        sc.VectorModel(5)
    with pytest.raises(ValueError):
        sc.VectorModel(16, "gpu")
    assert sc.VectorModel(8).generic_max_kw == 9


def test_mac_count_reference_cases():
    # test_reference.py:89-94
    assert sc.mac_count(sc.ConvShape(10, 1, 3, 1)) == 24
    assert sc.mac_count(sc.ConvShape(512, 512, 3, 3)) == 2_340_900


# --- error classes raised before any device work (reference raise sites) ----

def test_filter_larger_than_input_raises():           # test_reference.py:37-42
    x = np.zeros((3, 3), dtype=np.float32)
    with pytest.raises(sc.ShapeError):
        sc.conv2d_reference(x, np.zeros((4, 2), dtype=np.float32))
    with pytest.raises(sc.ShapeError):
        sc.conv2d_reference(x, np.zeros((2, 4), dtype=np.float32))


def test_conv1d_too_wide_directs_to_compound():        # test_slide_kernels.py:93-94
    with pytest.raises(sc.FilterWidthError, match="compound"):
        sc.conv1d_slide(np.zeros(64), np.zeros(6), sc.VectorModel(4))


def test_conv1d_requires_height_one():
    with pytest.raises(sc.ShapeError):
        sc.conv1d_slide(np.zeros((2, 8)), np.ones(3), sc.VectorModel(4))
    with pytest.raises(sc.ShapeError):
        sc.conv1d_reference(np.zeros((2, 8)), np.ones(3))


def test_generic_rejects_wide_filters():               # test_slide_kernels.py:120-121
    with pytest.raises(sc.FilterWidthError):
        sc.conv2d_slide_generic(np.zeros((8, 8)), np.zeros((2, 6)), sc.VectorModel(4))


def test_compound_rejects_width_one():                 # test_slide_kernels.py:137-138
    with pytest.raises(sc.ShapeError):
        sc.conv2d_slide_compound(np.zeros((4, 4)), np.ones((1, 1)), sc.VectorModel(4))


@pytest.mark.parametrize("k,fn", [(3, sc.conv2d_custom3), (5, sc.conv2d_custom5)])
def test_custom_wrong_size_raises(k, fn):              # test_slide_kernels.py:145-146
    with pytest.raises(sc.FilterSizeError):
        fn(np.zeros((10, 10)), np.ones((k + 1, k + 1)), sc.VectorModel(8))


def test_width_error_precedes_shape_error():
    # kernels.py:239-244: the generic width check runs before ConvShape
    with pytest.raises(sc.FilterWidthError):
        sc.conv2d_slide_generic(np.zeros((2, 2)), np.zeros((3, 30)), sc.VectorModel(4))


def test_run_variant_not_applicable():
    with pytest.raises(sc.ShapeError):
        sc.run_variant(sc.KernelVariant.CUSTOM3, np.zeros((8, 8)), np.ones((5, 5)),
                       sc.VectorModel(8))


def test_pool_window_out_of_range():                   # test_pooling.py:62-66
    with pytest.raises(sc.ShapeError):
        sc.sliding_window_sum([1.0, 2.0], 3)
    with pytest.raises(sc.ShapeError):
        sc.sliding_window_max([1.0, 2.0], 0)
    with pytest.raises(sc.ShapeError):
        sc.sliding_window_mean(np.zeros((2, 5)), 6)
    # the fused pair validates like the single-op calls (pooling.py:32-33), before any CUDA call
    with pytest.raises(sc.ShapeError):
        sc.sliding_window_sum_max([1.0, 2.0], 3)
    with pytest.raises(sc.ShapeError):
        sc.sliding_window_mean_max(np.zeros((2, 5)), 0)


def test_tensor_coercion_errors():
    with pytest.raises(sc.ShapeError):
        sc.conv2d_reference(np.zeros((0, 3)), np.ones((1, 1)))
    with pytest.raises(sc.ShapeError):
        sc.conv2d_reference(np.zeros((3, 3)), np.ones((2, 2, 2)))


def test_nchw_validation():
    with pytest.raises(sc.ShapeError):
        sc.conv2d_nchw(np.zeros((1, 3, 8, 8)), np.zeros((4, 2, 3, 3)))
    with pytest.raises(sc.ShapeError):
        sc.conv2d_nchw(np.zeros((3, 8, 8)), np.zeros((4, 3, 3, 3)))


def test_gemm_validation():
    with pytest.raises(sc.ShapeError):
        sc.gemm(np.zeros((2, 3)), np.zeros((4, 2)))
    with pytest.raises(sc.ShapeError):
        sc.gemm(np.zeros(3), np.zeros((3, 1)))


def test_bloat_ratio():                                # test_gemm.py / acceptance criterion 3
    r = sc.bloat_ratio(sc.ConvShape(512, 512, 3, 3))
    assert abs(r - 260100 * 9 / 512 / 512) < 1e-12


@pytest.mark.parametrize("h,kh,world", [(65536, 7, 1), (65536, 7, 2), (65536, 7, 8),
                                        (1000, 7, 3), (203, 5, 4), (50, 1, 7)])
def test_row_band_plan_covers_every_output_row_once(h, kh, world):
    plans = sc.plan_row_bands(h, kh, world)
    assert len(plans) == world
    covered = []
    for p in plans:
        covered.extend(range(p.out_start, p.out_stop))
        assert p.out_stop - p.out_start == p.interior_rows + (p.halo if p.rank < world - 1 else 0)
    assert covered == list(range(h - kh + 1))
    assert sum(p.in_stop - p.in_start for p in plans) == h


def test_row_band_plan_rejects_thin_bands():
    with pytest.raises(sc.ShapeError):
        sc.plan_row_bands(20, 7, 8)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sc.conv2d_reference(np.ones((4, 4), np.float32), np.ones((2, 2), np.float32))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sc.sliding_window_sum(np.ones(8, np.float32), 3)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sc.sliding_window_mean_max(np.ones(8, np.float32), 3)


def test_verify_suite_rejects_zero_trials():
    import paper_2310_05218_b200 as sc
    with pytest.raises(ValueError):
        sc.verify_suite(trials=0)


@pytest.mark.parametrize("kw", [dict(reps=2), dict(warmup=-1), dict(filter_sizes=()),
                                dict(filter_sizes=(512,)), dict(in_n=0)])
def test_harness_config_validation(kw):
    from paper_2310_05218_b200 import harness
    with pytest.raises(ValueError):
        harness.BenchConfig(**kw).validate()
