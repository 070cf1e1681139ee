"""Host-side cost per drop-in call (device tensors): wall time per enqueue and a
cProfile breakdown of the Python wrapper."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

x = torch.randn((256, 262144), device="cuda")
xn = torch.randn((16, 64, 112, 112), device="cuda")
wn = torch.randn((64, 64, 3, 3), device="cuda")
for fn, name in ((lambda: sc.sliding_window_mean(x, 16), "mean"),
                 (lambda: sc.sliding_window_max(x, 16), "max"),
                 (lambda: sc.conv2d_nchw(xn, wn, 1), "nchw")):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(4e8))  # keep the GPU busy so enqueue never blocks
    t0 = time.perf_counter()
    for _ in range(200):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: {1e6 * (t1 - t0) / 200:.1f} us host per call", flush=True)
torch.cuda._sleep(int(4e8))
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    sc.sliding_window_mean(x, 16)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)

# raw C-ABI call cost (no Python wrapper): pooling and conv on device pointers
import ctypes  # noqa: E402
from paper_2310_05218_b200 import _lib  # noqa: E402

lib = _lib.load()
y = torch.empty((256, 262144 - 15), device="cuda")
stream = torch.cuda.current_stream().cuda_stream
for name, call in (("sc_pool1d_f32 avg", lambda: lib.sc_pool1d_f32(1, x.data_ptr(), 256, 262144, 16, 0, y.data_ptr(), stream)),
                   ("sc_pool1d_stages", lambda: lib.sc_pool1d_stages(1, 16)),
                   ("sc_version", lambda: lib.sc_version())):
    call()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(4e8))
    t0 = time.perf_counter()
    for _ in range(200):
        call()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: {1e6 * (t1 - t0) / 200:.2f} us per raw call", flush=True)
