"""The GPU benchmark harness keeps the reference's CSV / plot-data contract
(reference bench.py:22-185) and produces correct outputs for every cell."""

import csv

import numpy as np
import pytest

from paper_2310_05218_b200 import harness
from paper_2310_05218_b200.kernels import KernelVariant

pytestmark = pytest.mark.gpu


def test_small_run_csv_and_plot_data(tmp_path):
    cfg = harness.BenchConfig(filter_sizes=(3, 5, 17), input_h=64, input_w=72, reps=3, warmup=1)
    recs = harness.run_benchmark(cfg)
    # every applicable variant plus the im2col baseline, per size, in enum order
    assert {r.kw for r in recs} == {3, 5, 17}
    for k in (3, 5, 17):
        names = [r.variant for r in recs if r.kw == k]
        assert KernelVariant.IM2COL_GEMM in names
        base = next(r for r in recs if r.kw == k and r.variant is KernelVariant.IM2COL_GEMM)
        assert base.speedup_vs_baseline == 1.0
        # all variants compute the same function: checksums agree
        sums = [r.checksum for r in recs if r.kw == k]
        assert np.allclose(sums, sums[0], rtol=1e-4, atol=1e-3)
    out = tmp_path / "b.csv"
    harness.emit_csv(recs, out)
    rows = list(csv.reader(open(out)))
    assert tuple(rows[0]) == harness.CSV_FIELDS and len(rows) == len(recs) + 1
    assert all(int(r[5]) > 0 for r in rows[1:])
    sp, tp = harness.emit_plot_data(recs, cfg, tmp_path / "plots")
    assert sp.read_text().startswith("# ") and "im2col" in tp.read_text().lower()


def test_batched_images_scale_macs():
    one = harness.run_benchmark(harness.BenchConfig(filter_sizes=(3,), input_h=40, input_w=40,
                                                    reps=3, warmup=0))
    four = harness.run_benchmark(harness.BenchConfig(filter_sizes=(3,), input_h=40, input_w=40,
                                                     reps=3, warmup=0, in_n=4))
    assert [4 * r.macs for r in one] == [r.macs for r in four]
