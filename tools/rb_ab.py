"""A/B on one GPU: a row-band rank's work as two launches (interior +
boundary strip with torch.cat) vs one launch over the band + in-place halo."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2310_05218_b200 import _ops  # noqa: E402

H = W = 65536
f7 = np.random.default_rng(1).standard_normal((7, 7), dtype=np.float32) / 7


def timed(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for g in (8, 4):
    rows = H // g
    buf = torch.rand((rows + 6, W), device="cuda")
    y = torch.empty((rows, W - 6), device="cuda")
    band, halo = buf[:rows], buf[rows:].clone()

    def two():
        _ops.conv2d_into(band, f7, y[:rows - 6])
        _ops.conv2d_into(torch.cat([band[rows - 6:], halo]), f7, y[rows - 6:])

    def one():
        _ops.conv2d_into(buf, f7, y)
    res = {"two": [], "one": []}
    for _ in range(4):
        res["two"].append(timed(two))
        res["one"].append(timed(one))
    print(g, {k: [round(v, 3) for v in vs] for k, vs in res.items()}, flush=True)
    del buf, y, band, halo
