"""Exact sums / averages for 32 < k <= 64 (pool_exact.cu, B = 64 tiles) on the
config-2 input: device ms per call."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

x = torch.randn((256, 262144), device="cuda")
res = {}
for k in (37, 48, 63, 100, 255):
    for name, fn in (("sum", sc.sliding_window_sum), ("avg", sc.sliding_window_mean)):
        for _ in range(3):
            fn(x, k, exact=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn(x, k, exact=True)
        b.record()
        b.synchronize()
        res[f"{name}{k}"] = round(a.elapsed_time(b) / 10, 4)
print(json.dumps(res))
