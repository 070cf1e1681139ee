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
