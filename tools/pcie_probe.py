"""PCIe ceilings on the box: pinned H2D alone, D2H alone, and both at once on
two streams (the host pipeline's best case), 256 MB transfers."""
import time

import torch

n = 64 << 20  # floats = 256 MB
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, device="cuda")
d_b = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


nb = 4 * n
t = timed(h2d)
print(f"H2D alone: {nb / t / 1e9:.1f} GB/s")
t = timed(d2h)
print(f"D2H alone: {nb / t / 1e9:.1f} GB/s")
t = timed(both)
print(f"H2D + D2H concurrent: {nb / t / 1e9:.1f} GB/s each direction, {2 * nb / t / 1e9:.1f} total")

# chunked, the host pipeline's pattern: 16 x 16 MB, each chunk H2D then D2H
# on one of 3 streams (chunk i+3 reuses chunk i's device buffer)
streams = [torch.cuda.Stream() for _ in range(3)]
cn = n // 16
dev_in = [torch.empty(cn, device="cuda") for _ in range(3)]
dev_out = [torch.empty(cn, device="cuda") for _ in range(3)]


def chunked():
    for i in range(16):
        s = streams[i % 3]
        with torch.cuda.stream(s):
            dev_in[i % 3].copy_(h_in[i * cn:(i + 1) * cn], non_blocking=True)
            dev_out[i % 3].copy_(dev_in[i % 3])
            h_out[i * cn:(i + 1) * cn].copy_(dev_out[i % 3], non_blocking=True)


t = timed(chunked)
print(f"chunked 16 x 16 MB, 3 streams: {nb / t / 1e9:.1f} GB/s each direction")
