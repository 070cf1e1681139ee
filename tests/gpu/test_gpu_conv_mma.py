"""The opt-in tensor-core slide-MMA conv (csrc/conv2d_mma.cu, SC_CONV_MMA=1)
vs the oracle: fast-mode tolerance 1e-5*k (north star), the non-finite
fallback (tiles recomputed with FMAs reproduce the reference's inf / NaN
pattern), ragged row segments and batches.  The switch is read once per
process, so the checks run in a child process."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r'''
import json, sys
import numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O
out = []
rng = np.random.default_rng(11)
for shape, (kh, kw) in [((2, 2048, 4096), (7, 7)), ((1, 1500, 10240), (7, 7)),
                        ((3, 700, 8192), (9, 9)), ((2, 1029, 8448), (6, 8)),
                        ((1, 1200, 9216), (8, 5))]:
    x = rng.uniform(-1, 1, shape).astype(np.float32)
    f = (rng.standard_normal((kh, kw)) / np.sqrt(kh * kw)).astype(np.float32)
    got = sc.conv2d_slide_compound(torch.from_numpy(x).cuda(), f, sc.VectorModel(16))[0]
    want = O.conv2d_batched(x, f)
    out.append({"case": [list(shape), kh, kw],
                "err": O.normwise_error(got.cpu().numpy(), want),
                "tol": O.north_star_tol(max(kh, kw))})
x = rng.uniform(-1, 1, (2, 2048, 4096)).astype(np.float32)
x[0, 100, 200] = np.inf
x[1, 1500, 1030] = np.nan
x[1, 10, 4000] = -np.inf
x[0, 900, 77] = 1e30
f = (rng.standard_normal((7, 7)) / 7).astype(np.float32)
got = sc.conv2d_slide_compound(torch.from_numpy(x).cuda(), f, sc.VectorModel(16))[0].cpu().numpy()
want = O.conv2d_batched(x, f)
fin = np.isfinite(want)
out.append({"nonfinite": True,
            "mask_equal": bool(np.array_equal(np.isnan(got), np.isnan(want)) and
                               np.array_equal(np.isinf(got), np.isinf(want))),
            "err": O.normwise_error(got[fin], want[fin]), "tol": O.north_star_tol(7)})
lib = sc._lib.load()
out.append({"launch_rows": int(lib.sc_conv2d_segment_rows(1, 2048, 4096, 7, 7, 0))})
print(json.dumps(out))
'''


def test_slide_mma_parity():
    env = {**os.environ, "SC_CONV_MMA": "1"}
    r = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + CHILD], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for case in res[:-1]:
        assert case["err"] <= case["tol"], case
    assert res[-2]["mask_equal"], res[-2]
