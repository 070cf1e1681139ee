"""bench.py's multi-rank plumbing on CPU: `--gpus 2 --dry-run` re-launches
itself under torch.distributed.run (one rank per "GPU"), runs the real halo
exchange of rowband.py over gloo, reduces over ranks and prints ONE JSON line
with n_gpus = 2; plus the helpers both arms share."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("n", [2, 3])
def test_dry_run_launches_n_ranks(n):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                          "--dry-run", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == n and rec["dry_run"] is True
    assert rec["rowband_cfg5"]["ranks"] == n
    assert rec["rowband_cfg5"]["halo_ok"] is True
    assert rec["config"] == bench.bench_config(n)


def test_both_arms_share_the_config_dict():
    assert bench.bench_config(1) == bench.bench_config(1)
    src = open(os.path.join(ROOT, "bench.py")).read()
    # both JSON lines take their config from bench_config (same_config check)
    assert src.count('"config": bench_config(world)') >= 2


def test_compact_per_config_is_short():
    detail = {
        "cfg1_conv1d_k7": {"ms": 0.08, "gbs": 6400.0, "gflops": 1, "bound": "hbm",
                           "frac_of_bound": 0.97, "hbm_frac": 0.97, "im2col_cublas_ms": 4.0},
        **{f"cfg2_pool_k{k}": {op: {"ms": 0.08, "gbs": 6400.0, "frac_of_bound": 0.97}
                               for op in ("avg", "max", "sum")} | {"torch_pool_ms": {"avg": 1,
                                                                                     "max": 2}}
           for k in (3, 16, 64, 255)},
        "cfg5_7x7_65536": {"ms": 6.7, "gbs": 5100.0, "bound": "fp32", "frac_of_bound": 0.84,
                           "im2col_cublas_ms": 1100.0, "clocks": {"sm_mhz": 1700}},
        "rowband_cfg5_projection": {"whole_ms": 7.0, "G2": {"proj_eff": 0.99},
                                    "G4": {"proj_eff": 0.98}, "G8": {"proj_eff": 0.95}},
    }
    c = bench.compact_per_config(detail)
    assert set(detail) <= set(c)
    assert len(json.dumps(c)) < 1500
