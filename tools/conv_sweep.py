"""Back-to-back timing of the conv kernels for BASELINE configs 1 / 3 / 5."""
import os
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


tag = f"ROWS={os.environ.get('SC_CONV_ROWS', 'auto')}"
which = os.environ.get("WHICH", "c1,c3,c5,c7").split(",")
out = []
if "c1" in which:
    x = torch.rand((64, 1 << 20), device="cuda")
    f = np.random.default_rng(1).standard_normal((1, 7), dtype=np.float32)
    t = bench(lambda: sc.conv2d_reference(x, f, exact=False), 20)
    out.append(f"1x7 {t:7.1f}us {4 * (2 * x.numel()) / t / 1e3:5.0f}GB/s")
    del x
if "c3" in which or "c5" in which:
    x = torch.rand((32, 4096, 4096), device="cuda")
    for k in (3, 5):
        if f"c{k}" not in which:
            continue
        f = np.random.default_rng(k).standard_normal((k, k), dtype=np.float32) / k
        t = bench(lambda: sc.conv2d_reference(x, f, exact=False))
        out.append(f"{k}x{k} {t:7.1f}us {4 * (x.numel() + 32 * (4097 - k) ** 2) / t / 1e3:5.0f}GB/s")
    del x
if "c7" in which:
    x = torch.rand((65536, 65536), device="cuda")
    f = np.random.default_rng(7).standard_normal((7, 7), dtype=np.float32) / 7
    t = bench(lambda: sc.conv2d_reference(x, f, exact=False), 3)
    out.append(f"7x7 {t:7.1f}us {2 * 49 * 65530 ** 2 / t / 1e6:6.0f}GFLOP/s")
print(tag, " | ".join(out), flush=True)
