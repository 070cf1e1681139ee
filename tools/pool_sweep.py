"""Back-to-back timing of the pooling kernels vs a torch copy of the same bytes."""
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

x = torch.randn((256, 262144), device="cuda")
y = torch.empty_like(x)


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


nb = 4 * (x.numel() * 2)
t = bench(lambda: y.copy_(x))
print(f"torch copy 268MB: {t:.1f} us  {nb / t / 1e3:.0f} GB/s")
big = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
big2 = torch.empty_like(big)
t = bench(lambda: big2.copy_(big), 20)
print(f"torch copy 2GiB: {t:.1f} us  {4 * (1 << 30) / t / 1e3:.0f} GB/s")
for k in (16, 3, 64):
    for name, fn in (("avg", sc.sliding_window_mean), ("max", sc.sliding_window_max),
                     ("sum", sc.sliding_window_sum)):
        t = bench(lambda: fn(x, k))
        print(f"NBUF={os.environ.get('SC_POOL_NBUF', '3')} k={k} {name}: {t:.1f} us  "
              f"{4 * (x.numel() + 256 * (262144 - k + 1)) / t / 1e3:.0f} GB/s")
