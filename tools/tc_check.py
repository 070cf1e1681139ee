"""Quick correctness + timing check of the tcgen05 NCHW path vs float64."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402
from oracle import slideconv_oracle as O  # noqa: E402

rng = np.random.default_rng(4)
for_shapes = not os.environ.get("TC_ONLY_TIME")
for (n, cin, cout, h, w) in [(1, 32, 64, 8, 16), (1, 64, 64, 16, 32), (2, 64, 64, 112, 112),
                             (1, 32, 128, 20, 24), (3, 64, 128, 13, 48), (1, 128, 64, 9, 32), (1, 64, 64, 112, 112), (2, 32, 64, 30, 224),
                             (2, 32, 192, 17, 160)]:
    x = rng.standard_normal((n, cin, h, w), dtype=np.float32)
    wt = (rng.standard_normal((cout, cin, 3, 3), dtype=np.float32) / np.float32(np.sqrt(9 * cin))).astype(np.float32)
    t0 = time.time()
    y = sc.conv2d_nchw(x, wt, 1)
    torch.cuda.synchronize()
    ref = O.conv2d_nchw_f64(x, wt, 1)
    err = O.normwise_error(y, ref)
    print(f"{(n, cin, cout, h, w)} normwise {err:.3e} tol {O.north_star_tol(3, cin):.1e} "
          f"maxabs {np.max(np.abs(y - ref)):.3e} ({time.time() - t0:.2f}s)", flush=True)

xd = torch.randn((16, 64, 112, 112), device="cuda")
wd = torch.randn((64, 64, 3, 3), device="cuda") / 24
for _ in range(30):
    sc.conv2d_nchw(xd, wd, 1)
torch.cuda.synchronize()
ts = []
for rep in range(5):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    a.record()
    for _ in range(100):
        sc.conv2d_nchw(xd, wd, 1)
    w1 = time.perf_counter()
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b) / 100)
    print(f"  host issue {1e4 * (w1 - w0):.1f} us/call, device {ts[-1] * 1e3:.1f} us/call")
t = sorted(ts)[2]
print(f"config 4 TC: {t * 1e3:.1f} us (min {min(ts)*1e3:.1f} max {max(ts)*1e3:.1f})  {2 * 16 * 64 * 112 * 112 * 64 * 9 / t / 1e9:.1f} TFLOP/s")
