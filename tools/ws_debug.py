"""Weights-stationary NCHW kernel debug: single-tap filters with bf16-exact data."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402
from oracle import slideconv_oracle as O  # noqa: E402


def bf16_exact(a):
    t = torch.from_numpy(a).to(torch.bfloat16).to(torch.float32)
    return t.numpy()


rng = np.random.default_rng(0)
n, cin, cout, h, w = 1, 32, 64, 8, 16
x = bf16_exact(rng.standard_normal((n, cin, h, w), dtype=np.float32))
for tap in [(1, 1), (0, 0), (0, 1), (1, 0), (2, 2), None]:
    wt = np.zeros((cout, cin, 3, 3), np.float32)
    if tap is None:
        wt = bf16_exact(rng.standard_normal((cout, cin, 3, 3), dtype=np.float32))
    else:
        wt[:, :, tap[0], tap[1]] = bf16_exact(rng.standard_normal((cout, cin), dtype=np.float32))
    y = sc.conv2d_nchw(x, wt, 1)
    ref = O.conv2d_nchw_f64(x, wt, 1)
    err = np.abs(y - ref)
    print(f"tap {tap}: normwise {O.normwise_error(y, ref):.3e}  max {err.max():.3e}")
    if err.max() > 1e-3:
        bad = np.argwhere(err > 1e-3)
        print("  first bad (n, co, r, c):", bad[:6].tolist(), "count", len(bad), "of", err.size)
        co, r = 0, 3
        print("  got ", np.round(y[0, co, r, :8], 3))
        print("  want", np.round(ref[0, co, r, :8], 3))
        # is it a shifted version?  correlate against shifted refs
        for dr in (-1, 0, 1):
            for dc in (-2, -1, 0, 1, 2):
                sh = np.roll(np.roll(ref, dr, axis=2), dc, axis=3)
                e = np.abs(y - sh)[:, :, 2:-2, 3:-3].max()
                if e < 1e-3:
                    print(f"  matches ref shifted by rows {dr} cols {dc}")
        # channel permutation?
        for co2 in range(cout):
            if np.abs(y[0, 0, 2:-2, 3:-3] - ref[0, co2, 2:-2, 3:-3]).max() < 1e-3:
                print(f"  out channel 0 == ref channel {co2}")
