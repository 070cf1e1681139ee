"""Per-k-block timeline of CTA 0 of the NCHW tensor-core kernel (library built with
make EXTRA=-DSC_TC_TRACE; the stamps overwrite y)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

xd = torch.randn((16, 64, 112, 112), device="cuda")
wd = torch.randn((64, 64, 3, 3), device="cuda") / 24
for _ in range(3):
    y = sc.conv2d_nchw(xd, wd, 1)
torch.cuda.synchronize()
t = y.reshape(-1)[:8 * 64].view(torch.int32).cpu().numpy().astype(np.int64).reshape(8, 64)
t0 = t[0, 0]
t = (t - t0) & 0xffffffff
t[t > 2**31] -= 2**32
names = ["mma:split_ok", "mma:b_ok", "mma:committed", "split:free_ok", "split:st_issued", "prod:b_empty_ok", "split:arrive", "split:st_done"]
print("kc " + " ".join(f"{n:>15}" for n in names))
for kc in range(45):
    print(f"{kc:2d} " + " ".join(f"{t[r, kc]:15d}" for r in range(8)))
