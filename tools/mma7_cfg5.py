"""Config 5 (7x7 on H x 65,536) through the opt-in 7x7 slide-MMA kernel
(SC_CONV_MMA=1) vs the default FFMA kernel, sustained: python tools/mma7_cfg5.py [H]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_05218_b200 as sc
from paper_2310_05218_b200 import _ops
H = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
x = torch.empty((H, 65536), device="cuda").uniform_(-1, 1)
f = (np.random.default_rng(7).standard_normal((7, 7)) / 7).astype(np.float32)
y = torch.empty((H - 6, 65530), device="cuda")
os.environ["SC_CONV_MMA_BIG"] = "0"


def timed(mode, reps=8, hot=1.0):
    os.environ["SC_CONV_MMA"] = mode
    t_end = time.time() + hot
    while time.time() < t_end:
        _ops.conv2d_into(x, f, y)
        torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); _ops.conv2d_into(x, f, y); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for rnd in range(2):
    t0 = timed("0"); y0 = y[:64].clone()
    t1 = timed("1")
    err = float((y[:64].double() - y0.double()).norm() / y0.double().norm())
    print(f"{H} x 65536 7x7, after 1 s of load: ffma {t0:.3f} ms, slide-MMA {t1:.3f} ms (x{t0 / t1:.3f}), normwise diff {err:.1e}", flush=True)
