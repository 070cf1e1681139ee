import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402
from oracle import slideconv_oracle as O  # noqa: E402
n, cin, cout, h, w = 1, 32, 64, 8, 16
x = np.ones((n, cin, h, w), np.float32)
wt = np.zeros((cout, cin, 3, 3), np.float32)
wt[:, :, 1, 1] = 1.0          # center tap only -> out = cin everywhere
y = sc.conv2d_nchw(x, wt, 1)
print("center-only: y[0,0,:3,:5]", y[0, 0, :3, :5], "y[0,5,2,:5]", y[0, 5, 2, :5])
wt2 = np.zeros_like(wt); wt2[3, 0, 1, 1] = 2.0   # co=3 gets 2*x[ci=0]
x2 = np.arange(n * cin * h * w, dtype=np.float32).reshape(n, cin, h, w) % 7
y2 = sc.conv2d_nchw(x2, wt2, 1)
print("single weight: y2[0,3,:2,:6]", y2[0, 3, :2, :6], "want", 2 * x2[0, 0, :2, :6], "other ch max", np.abs(y2[0, :3]).max())
wt3 = np.zeros_like(wt); wt3[0, 0, 1, 0] = 1.0   # left tap: out[w] = x[w-1]
y3 = sc.conv2d_nchw(x2, wt3, 1)
print("left tap: y3[0,0,0,:6]", y3[0, 0, 0, :6], "x row", x2[0, 0, 0, :6])
ref = O.conv2d_nchw_f64(x2, wt3, 1)
print("left tap err", np.abs(y3 - ref).max())
