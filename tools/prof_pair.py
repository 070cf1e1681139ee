"""k=16 and k=64 window sums back to back (for ncu --cache-control none)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

x = torch.randn((256, 262144), device="cuda")
for k in (16, 64):
    for _ in range(6):
        sc.sliding_window_sum(x, k)
torch.cuda.synchronize()
print("ok")
