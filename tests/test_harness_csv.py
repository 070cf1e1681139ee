"""The GPU harness's CSV / plot-data contract without a GPU (reference
bench.py:132-185 and its acceptance criterion 9: CSV round-trip)."""

import csv
import math

import pytest

from paper_2310_05218_b200 import harness
from paper_2310_05218_b200.kernels import KernelVariant


def _records():
    out = []
    for k in (3, 11):
        for v, ns in ((KernelVariant.SLIDE_GENERIC, 1200), (KernelVariant.IM2COL_GEMM, 9000)):
            out.append(harness.BenchRecord(variant=v, kh=k, kw=k, in_h=512, in_w=512, median_ns=ns * k,
                                           min_ns=ns * k - 5, macs=510 * 510 * k * k, slides=k,
                                           im2col_elems=0 if v is KernelVariant.SLIDE_GENERIC else 7,
                                           gflops=1.0 / 3.0 * k, speedup_vs_baseline=9000 / ns,
                                           checksum=0.25))
    return out


def test_csv_round_trip(tmp_path):
    recs = _records()
    path = tmp_path / "b.csv"
    harness.emit_csv(recs, path)
    rows = list(csv.DictReader(open(path)))
    assert tuple(rows[0].keys()) == harness.CSV_FIELDS
    assert len(rows) == len(recs)
    for r, rec in zip(rows, recs):
        assert r["variant"] == str(rec.variant)
        assert int(r["median_ns"]) == rec.median_ns and int(r["macs"]) == rec.macs
        assert float(r["gflops"]) == rec.gflops            # repr() round-trips exactly
        assert float(r["speedup"]) == rec.speedup_vs_baseline


def test_plot_data_blocks(tmp_path):
    sp, tp = harness.emit_plot_data(_records(), harness.BenchConfig(roofline_gflops=74450.0),
                                    tmp_path / "plots")
    speed = sp.read_text().split("\n\n")
    assert speed[0].startswith(f"# {KernelVariant.IM2COL_GEMM}") or speed[0].startswith("# ")
    thr = tp.read_text()
    assert "# roofline" in thr and "74450.0" in thr
    for line in thr.splitlines():
        if line and not line.startswith("#"):
            k, v = line.split()
            assert int(k) in (3, 11) and math.isfinite(float(v))


def test_emit_errors(tmp_path):
    with pytest.raises(ValueError):
        harness.emit_csv([], tmp_path / "x.csv")
    one = [r for r in _records() if r.kw == 3]
    with pytest.raises(ValueError):
        harness.emit_plot_data(one, harness.BenchConfig(), tmp_path / "p")
    with pytest.raises(OSError):
        harness.emit_csv(_records(), tmp_path / "missing_dir" / "x.csv")
