"""The randomized property suite (reference verify.py:64-215) on the GPU kernels:
every property passes, and fault injection flips exactly the targeted one."""

import pytest

import paper_2310_05218_b200 as sc

pytestmark = pytest.mark.gpu

PROPERTIES = ["cross_variant_oracle", "flop_parity", "delta_filter", "slide_count_formulas",
              "custom_fewer_slides", "pooling_sum", "pooling_max", "boundary_shapes",
              "backend_equivalence"]


@pytest.mark.parametrize("seed", [0, 7])
def test_suite_passes(seed):
    report = sc.verify_suite(seed=seed, trials=24)
    assert [r.name for r in report.results] == PROPERTIES
    assert report.passed, report.summary()


@pytest.mark.parametrize("lanes", [4, 8, 32])
def test_suite_other_lane_widths(lanes):
    report = sc.verify_suite(seed=3, trials=6, vm=sc.VectorModel(lanes))
    assert report.passed, report.summary()


@pytest.mark.parametrize("target", PROPERTIES)
def test_fault_injection_is_detected(target):
    report = sc.verify_suite(seed=1, trials=3, corrupt=target)
    failed = [r.name for r in report.results if not r.passed]
    assert failed == [target], report.summary()
