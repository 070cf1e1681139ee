"""One shape through the large-filter slide-MMA kernel (for ncu):
python tools/mma_big_one.py B H W K [reps]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_05218_b200 as sc
os.environ["SC_CONV_MMA_BIG"] = "2"
b, h, w, k = (int(v) for v in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
x = torch.rand((b, h, w), device="cuda") * 2 - 1
f = (np.random.default_rng(k).standard_normal((k, k)) / k).astype(np.float32)
for _ in range(reps):
    sc.conv2d_reference(x, f, exact=False)
torch.cuda.synchronize()
