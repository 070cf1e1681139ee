"""pytest plugin: make `import slideconv` (the reference package) resolve to
this drop-in, so the reference's own test files run unchanged against the
sm_100a kernels.  Loaded with `-p tests.ref_replay.slideconv_alias`.

Module map (reference pkg/src/slideconv/ -> paper_2310_05218_b200/):
  slideconv            -> the package (+ the harness names the reference
                          __init__ re-exports: BenchConfig, emit_csv, ...)
  slideconv.reference / kernels / pooling / tensor / gemm / lanes / verify
                       -> the same-named modules
  slideconv.bench      -> harness (the reference's CSV / plot-data contract)
"""

import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2310_05218_b200 as _pkg  # noqa: E402
from paper_2310_05218_b200 import (gemm, harness, kernels, lanes, pooling,  # noqa: E402
                                   reference, tensor, verify)


def _install():
    alias = types.ModuleType("slideconv")
    alias.__dict__.update({k: v for k, v in vars(_pkg).items() if not k.startswith("__")})
    for name in ("BenchConfig", "BenchRecord", "emit_csv", "emit_plot_data",
                 "load_reference_series", "run_benchmark"):
        if hasattr(harness, name):
            setattr(alias, name, getattr(harness, name))
    if hasattr(lanes, "slide"):
        alias.slide = lanes.slide
    alias.__path__ = []  # a package, so `slideconv.x` submodule imports resolve
    sys.modules["slideconv"] = alias
    for sub, mod in (("reference", reference), ("kernels", kernels), ("pooling", pooling),
                     ("tensor", tensor), ("gemm", gemm), ("lanes", lanes), ("verify", verify),
                     ("bench", harness)):
        sys.modules[f"slideconv.{sub}"] = mod
        setattr(alias, sub, mod)


_install()
