"""Device-side A/B of the slide-MMA conv (SC_CONV_MMA=1) against the FFMA
kernel on a 7x7 image: max difference, wrong rows / columns.
python tools/pair_diag.py H W"""
import os, sys, torch, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2310_05218_b200 as sc
from paper_2310_05218_b200 import _ops
h, w = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda"); g.manual_seed(5)
x = torch.empty((h, w), device="cuda"); x.uniform_(-1, 1, generator=g)
f = (np.random.default_rng(5).standard_normal((7, 7)) / 7).astype(np.float32)
y0 = torch.empty((h - 6, w - 6), device="cuda"); y1 = torch.empty_like(y0)
os.environ["SC_CONV_MMA"] = "0"; _ops.conv2d_into(x, f, y0)
os.environ["SC_CONV_MMA"] = "1"; _ops.conv2d_into(x, f, y1)
torch.cuda.synchronize()
d = (y1 - y0).abs()
bad = d > 1e-3
print("shape", h, w, "max diff", float(d.max()), "bad frac", float(bad.float().mean()))
if bad.any():
    rows = bad.any(dim=1).nonzero().flatten()
    cols = bad.any(dim=0).nonzero().flatten()
    print("bad rows", rows.numel(), rows[:20].tolist(), "... last", rows[-5:].tolist())
    print("bad cols", cols.numel(), cols[:20].tolist(), "... last", cols[-5:].tolist())
    rs = sc._lib.load().sc_conv2d_segment_rows(1, h, w, 7, 7, 0)
    print("seg rows (ffma)", rs)
