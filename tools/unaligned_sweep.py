"""Pooling on signals whose length is not a multiple of 32 (the TMA kernels
need L % 32 == 0): device time against the aligned length."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402


def bench(fn, n=20):
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


for L in (262144, 262143, 262140):
    x = torch.randn((256, L), device="cuda")
    row = []
    for k in (3, 16, 64, 255):
        for name, fn in (("sum", sc.sliding_window_sum), ("max", sc.sliding_window_max)):
            t = bench(lambda: fn(x, k))
            row.append(f"{name}{k} {t:6.1f}")
    print(f"L={L}: " + " | ".join(row), flush=True)
