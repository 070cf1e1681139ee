"""Device time of the large-filter 2-D conv kernels (the paper's 11..51 sweep)
on a few image batches: TFLOP/s (2 * MACs / t) per filter size."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

ks = [int(v) for v in os.environ.get("KS", "11,17,21,29,33,37,51").split(",")]
shapes = [tuple(int(d) for d in s.split("x")) for s in os.environ.get("SHAPES", "32x512x512,4x2048x2048").split(",")]
exact = os.environ.get("EXACT", "0") == "1"


def bench(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n * 1e-3


for shp in shapes:
    x = torch.rand(shp, device="cuda") * 2 - 1
    row = []
    for k in ks:
        f = np.random.default_rng(k).standard_normal((k, k), dtype=np.float32) / k
        t = bench(lambda: sc.conv2d_reference(x, f, exact=exact))
        oh, ow = shp[-2] - k + 1, shp[-1] - k + 1
        fl = 2 * k * k * oh * ow * (shp[0] if len(shp) == 3 else 1)
        row.append(f"k={k}: {t * 1e3:.3f}ms {fl / t / 1e12:.1f}TF")
    print("x".join(map(str, shp)), " | ".join(row), flush=True)
