"""Per-k-block timeline of CTA 0 of the NCHW tensor-core kernel plus per-CTA
globaltimer stamps (library built with make EXTRA=-DSC_TC_TRACE; the stamps
overwrite y)."""
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
flat = y.reshape(-1)
t = flat[:9 * 128].view(torch.int32).cpu().numpy().astype(np.int64).reshape(9, 128)
t0 = t[0, 0]
t = (t - t0) & 0xffffffff
t[t > 2**31] -= 2**32
names = ["mma:full_ok", "-", "mma:committed", "split:free_ok", "split:st_issued", "prod:free_ok",
         "split:arrive", "split:st_done", "mma:issued"]
print("kc " + " ".join(f"{n:>15}" for n in names))
for kc in range(0, 99):
    print(f"{kc:2d} " + " ".join(f"{t[r, kc]:15d}" for r in range(9)))
g = flat[2048:2048 + 148 * 8].view(torch.int64).cpu().numpy().reshape(148, 4)
base = g[:, 0].min()
g = g - base
print("per-CTA globaltimer (ns): start, setup done, loop done, teardown")
for b in range(0, 148, 8):
    print(b, g[b])
print("max loop end", g[:, 2].max(), "min", g[:, 2].min(), "mean setup", g[:, 1].mean())
