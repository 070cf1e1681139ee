"""Back-to-back timing of the pooling kernels vs a device copy of the same bytes."""
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

x = torch.randn((256, 262144), device="cuda")
y = torch.empty_like(x)
ks = [int(v) for v in os.environ.get("KS", "16,3,64").split(",")]
ops = os.environ.get("OPS", "avg,max,sum").split(",")


def bench(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n * 1e3


tag = f"NBUF={os.environ.get('SC_POOL_NBUF', '-')} TPC={os.environ.get('SC_POOL_TPC', '-')}"
if os.environ.get("COPY", "0") == "1":
    t = bench(lambda: y.copy_(x))
    print(f"copy 268MB: {t:.1f} us  {4 * x.numel() * 2 / t / 1e3:.0f} GB/s")
fns = {"avg": sc.sliding_window_mean, "max": sc.sliding_window_max, "sum": sc.sliding_window_sum}
for k in ks:
    row = []
    for name in ops:
        t = bench(lambda: fns[name](x, k))
        row.append(f"{name} {t:6.1f}us {4 * (x.numel() + 256 * (262144 - k + 1)) / t / 1e3:5.0f}GB/s")
    print(f"{tag} k={k}: " + " | ".join(row))
