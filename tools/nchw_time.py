"""Config 4 (N16 Cin64 Cout64 112^2, 3x3 pad 1) per-call time, L2 flushed
between calls (median of 30), fast mode; prints ms and the executed bf16
TFLOP/s of the 3-product split."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(4)
x = torch.randn((16, 64, 112, 112), generator=g, device="cuda")
w = torch.randn((64, 64, 3, 3), generator=g, device="cuda") / 24
flush = torch.empty(64 << 20, device="cuda")
for _ in range(5):
    sc.conv2d_nchw(x, w, 1)
ts = []
for _ in range(30):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sc.conv2d_nchw(x, w, 1)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
fl = 2 * 16 * 64 * 64 * 9 * 112 * 112
print(json.dumps({"cfg4_ms": round(ms, 4), "executed_bf16_tflops": round(3 * fl / ms / 1e9, 1),
                  "frac_of_1664": round(3 * fl / ms / 1e9 / 1664.6, 3)}))
