"""Device time of exact-mode (bit-identical to the reference) pooling and
convolution on the BASELINE shapes, next to the default fast mode."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402


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
    return a.elapsed_time(b) / n * 1e3


x = torch.randn((256, 262144), device="cuda")
for k in (3, 16, 64, 100, 255):
    row = []
    for name, fn in (("sum", sc.sliding_window_sum), ("avg", sc.sliding_window_mean),
                     ("max", sc.sliding_window_max)):
        te = bench(lambda: fn(x, k, exact=True))
        tf = bench(lambda: fn(x, k, exact=False))
        row.append(f"{name} exact {te:7.1f}us fast {tf:6.1f}us")
    print(f"k={k}: " + " | ".join(row), flush=True)
del x
x = torch.rand((32, 4096, 4096), device="cuda")
for k in (3, 5):
    f = np.random.default_rng(k).standard_normal((k, k), dtype=np.float32) / k
    te = bench(lambda: sc.conv2d_reference(x, f, exact=True), 5)
    tf = bench(lambda: sc.conv2d_reference(x, f, exact=False), 5)
    print(f"conv {k}x{k}: exact {te:8.1f}us fast {tf:8.1f}us", flush=True)
