"""Config-5-like band (7x7 on 8192 x 65536) through the large-filter
slide-MMA kernel (forced) vs the default FFMA kernel."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_05218_b200 as sc
from paper_2310_05218_b200 import _ops
H = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
x = torch.empty((H, 65536), device="cuda").uniform_(-1, 1)
f = (np.random.default_rng(7).standard_normal((7, 7)) / 7).astype(np.float32)
y = torch.empty((H - 6, 65530), device="cuda")


def timed(mode, reps=5):
    os.environ["SC_CONV_MMA_BIG"] = mode
    for _ in range(2):
        _ops.conv2d_into(x, f, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        _ops.conv2d_into(x, f, y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t0 = timed("0")
y0 = y.clone()
t2 = timed("2")
err = float((y.double() - y0.double()).norm() / y0.double().norm())
print(f"{H} x 65536 7x7: ffma {t0:.3f} ms, mma_big {t2:.3f} ms (x{t0 / t2:.2f}), normwise diff {err:.2e}; "
      f"scaled to 65536 rows: {t0 * 65536 / H:.2f} vs {t2 * 65536 / H:.2f} ms")
