"""Fused host path (sliding_window_mean_max on pinned numpy) against the
link's ceilings for its 1 : 2 H2D : D2H pattern (268 MB up, 537 MB down)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_05218_b200 as sc  # noqa: E402

B, L, K = 256, 262144, 16
nb = 4 * B * L
xh = sc.pinned_empty((B, L))
xh[...] = np.random.default_rng(0).standard_normal((B, L), dtype=np.float32)
xt = torch.from_numpy(xh)
xd = torch.empty((B, L), device="cuda")
y1 = torch.empty((B, L), pin_memory=True)
y2 = torch.empty((B, L), pin_memory=True)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, n=8):
    fn(); fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


d2h = t(lambda: y1.copy_(xd, non_blocking=True))
h2d = t(lambda: xd.copy_(xt, non_blocking=True))
print(f"H2D alone {nb / h2d / 1e9:.1f} GB/s, D2H alone {nb / d2h / 1e9:.1f} GB/s")


def pattern():  # whole-buffer copies: 1 up, 2 down, all concurrent
    with torch.cuda.stream(s1):
        xd.copy_(xt, non_blocking=True)
    with torch.cuda.stream(s2):
        y1.copy_(xd, non_blocking=True)
        y2.copy_(xd, non_blocking=True)


tp = t(pattern)
print(f"1 up + 2 down concurrent (whole buffers): {tp * 1e3:.2f} ms -> D2H {2 * nb / tp / 1e9:.1f} GB/s")


def pattern2():  # the two downloads on two streams
    with torch.cuda.stream(s1):
        xd.copy_(xt, non_blocking=True)
    with torch.cuda.stream(s2):
        y1.copy_(xd, non_blocking=True)
    with torch.cuda.stream(s3):
        y2.copy_(xd, non_blocking=True)


tp = t(pattern2)
print(f"1 up + 2 down on 3 streams: {tp * 1e3:.2f} ms -> D2H {2 * nb / tp / 1e9:.1f} GB/s")
tt = t(lambda: sc.sliding_window_mean_max(xh, K))
print(f"fused host call (chunk {os.environ.get('SC_HOST_CHUNK_MB', 'dflt')} MB): {tt * 1e3:.2f} ms")
tt = t(lambda: (sc.sliding_window_mean(xh, K), sc.sliding_window_max(xh, K)))
print(f"two host calls: {tt * 1e3:.2f} ms")
