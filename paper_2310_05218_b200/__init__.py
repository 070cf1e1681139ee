"""B200-native (sm_100a) Sliding Window Sum convolution and pooling primitives
(arXiv 2310.05218), a drop-in for the hot path of the reference ``slideconv``
package: same function names, argument order, shapes, dtypes, errors and
returned cost counters; every primitive is a hand-written CUDA kernel reached
through the C ABI in include/slideconv_b200.h.  No CPU fallback exists.
"""

from ._device import pinned_empty, set_default_mode
from .gemm import bloat_ratio, conv2d_im2col, gemm, im2col_2d
from .kernels import (KernelVariant, analytic_counters, applicable_variants, compound_width,
                      conv1d_slide, conv2d_custom3, conv2d_custom5, conv2d_slide_compound,
                      conv2d_slide_generic, counted_offsets, run_variant, select_kernel,
                      variant_applicable)
from .lanes import VectorModel, slide
from .nchw import conv2d_nchw
from .pooling import (sliding_window_max, sliding_window_mean, sliding_window_mean_max,
                      sliding_window_sum, sliding_window_sum_max)
from .reference import conv1d_reference, conv2d_reference, oracle_conv2d, relative_error
from .rowband import RowBandGroup, RowBandPlan, alloc_band, conv2d_rowband, plan_row_bands
from .verify import PropertyResult, VerifyReport, verify_suite
from .tensor import (ConvShape, CostCounters, FilterSizeError, FilterWidthError, ShapeError,
                     mac_count)

__version__ = "0.1.0"

__all__ = [
    # reference hot-path subset (slideconv/__init__.py:39-49)
    "ConvShape", "CostCounters", "FilterSizeError", "FilterWidthError", "KernelVariant",
    "ShapeError", "VectorModel", "slide", "applicable_variants", "bloat_ratio", "conv1d_reference",
    "conv1d_slide", "conv2d_custom3", "conv2d_custom5", "conv2d_im2col", "conv2d_reference",
    "conv2d_slide_compound", "conv2d_slide_generic", "gemm", "im2col_2d", "mac_count",
    "oracle_conv2d", "run_variant", "select_kernel", "sliding_window_max", "sliding_window_sum",
    # helpers the reference keeps in submodules
    "analytic_counters", "compound_width", "counted_offsets", "variant_applicable",
    "relative_error", "verify_suite", "VerifyReport", "PropertyResult",
    # B200 extensions (BASELINE configs)
    "sliding_window_mean", "sliding_window_sum_max", "sliding_window_mean_max", "conv2d_nchw",
    "conv2d_rowband", "plan_row_bands", "RowBandPlan", "alloc_band", "RowBandGroup",
    "pinned_empty", "set_default_mode",
]
