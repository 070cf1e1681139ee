"""Host<->device bandwidth vs the host-buffer pooling pipeline."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

B, L = 256, 262144
xh = sc.pinned_empty((B, L))
xh[...] = np.random.default_rng(0).standard_normal((B, L), dtype=np.float32)
xd = torch.empty((B, L), device="cuda")
yh = torch.empty((B, L), pin_memory=True)


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


xt = torch.from_numpy(xh)
h2d = t(lambda: xd.copy_(xt, non_blocking=True))
d2h = t(lambda: yh.copy_(xd, non_blocking=True))
s1 = torch.cuda.Stream()
s2 = torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        xd.copy_(xt, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(xd, non_blocking=True)


bd = t(both)
nb = 4 * B * L
print(f"H2D {nb / h2d / 1e9:.1f} GB/s, D2H {nb / d2h / 1e9:.1f} GB/s, both-overlapped {2 * nb / bd / 1e9:.1f} GB/s total")
for op in (sc.sliding_window_mean, sc.sliding_window_max):
    tt = t(lambda: op(xh, 16))
    print(f"{op.__name__} host path: {tt * 1e3:.2f} ms -> {2 * nb / tt / 1e9:.1f} GB/s (in+out)")
xp = np.ascontiguousarray(xh.copy())
tt = t(lambda: sc.sliding_window_mean(xp, 16), 3)
print(f"pageable input: {tt * 1e3:.2f} ms -> {2 * nb / tt / 1e9:.1f} GB/s")
import os
print("cpus", os.cpu_count())
