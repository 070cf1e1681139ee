"""Config 5 with the FFMA kernel and the tensor-core slide-MMA kernel running
concurrently on two streams, each on its own row band (rows split by a
fraction): python tools/hetero_cfg5.py 0.0 0.3 0.45 0.6 1.0"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2310_05218_b200 import _ops  # noqa: E402

H = W = 65536
K = 7
g = torch.Generator(device="cuda")
g.manual_seed(5)
x = torch.empty((H, W), device="cuda")
x.uniform_(-1, 1, generator=g)
f = (np.random.default_rng(5).standard_normal((K, K)) / K).astype(np.float32)
y = torch.empty((H - K + 1, W - K + 1), device="cuda")
ref = torch.empty_like(y)
os.environ["SC_CONV_MMA"] = "0"
_ops.conv2d_into(x, f, ref)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
oh = H - K + 1


def run(frac):
    r1 = int(oh * frac) // 8 * 8
    ev = torch.cuda.Event()
    ev.record()
    if r1 > 0:
        with torch.cuda.stream(sa):
            sa.wait_event(ev)
            os.environ["SC_CONV_MMA"] = "1"
            _ops.conv2d_into(x[: r1 + K - 1], f, y[:r1])
    if r1 < oh:
        with torch.cuda.stream(sb):
            sb.wait_event(ev)
            os.environ["SC_CONV_MMA"] = "0"
            _ops.conv2d_into(x[r1:], f, y[r1:])
    torch.cuda.current_stream().wait_stream(sa)
    torch.cuda.current_stream().wait_stream(sb)


for frac in [float(v) for v in sys.argv[1:]]:
    for _ in range(2):
        run(frac)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(5):
        e0.record()
        run(frac)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    d = float((y - ref).abs().max())
    print(f"frac {frac:.2f}: {sorted(ts)[2]:.3f} ms  max|diff vs FFMA| {d:.2e}", flush=True)
