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

# the pipeline's own pattern with plain copies: chunk i = 16 MB up, then two
# 16 MB downloads, on slot stream i % 3 (device buffers reused per slot)
for cmb in (16, 64):
    cn = (cmb << 20) // 4
    nchunk = (B * L) // cn
    streams = [torch.cuda.Stream() for _ in range(3)]
    din = [torch.empty(cn, device="cuda") for _ in range(3)]
    xf, y1f, y2f = xt.view(-1), y1.view(-1), y2.view(-1)

    def chunked():
        for i in range(nchunk):
            s = streams[i % 3]
            with torch.cuda.stream(s):
                din[i % 3].copy_(xf[i * cn:(i + 1) * cn], non_blocking=True)
                y1f[i * cn:(i + 1) * cn].copy_(din[i % 3], non_blocking=True)
                y2f[i * cn:(i + 1) * cn].copy_(din[i % 3], non_blocking=True)

    tc = t(chunked)
    print(f"plain copies, {nchunk} x {cmb} MB chunks (1 up, 2 down) on 3 slot streams: {tc * 1e3:.2f} ms")

    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    dall = torch.empty(B * L, device="cuda")

    def roles():  # upload runs ahead on its own stream; downloads follow by events
        evs = []
        for i in range(nchunk):
            with torch.cuda.stream(up):
                dall[i * cn:(i + 1) * cn].copy_(xf[i * cn:(i + 1) * cn], non_blocking=True)
                e = torch.cuda.Event()
                e.record(up)
            with torch.cuda.stream(down):
                down.wait_event(e)
                y1f[i * cn:(i + 1) * cn].copy_(dall[i * cn:(i + 1) * cn], non_blocking=True)
                y2f[i * cn:(i + 1) * cn].copy_(dall[i * cn:(i + 1) * cn], non_blocking=True)

    tr = t(roles)
    print(f"plain copies, {nchunk} x {cmb} MB chunks, upload-ahead role streams: {tr * 1e3:.2f} ms")

# the C entry point alone, outputs preallocated (what the Python wrapper adds on top)
from paper_2310_05218_b200 import _lib
lib = _lib.load()
ya = sc.pinned_empty((B, L - K + 1)); ym = sc.pinned_empty((B, L - K + 1))
tc_ = t(lambda: lib.sc_pool1d_pair_f32_host(_lib.POOL_AVG, xh.ctypes.data, B, L, K, 0, ya.ctypes.data, ym.ctypes.data, 0))
print(f"sc_pool1d_pair_f32_host alone (preallocated pinned outputs): {tc_ * 1e3:.2f} ms")
