"""Small invocations of every kernel family, for compute-sanitizer runs."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((3, 4096), dtype=np.float32)).cuda()
for k in (3, 16, 64, 100, 255, 300):
    for fn in (sc.sliding_window_sum, sc.sliding_window_max, sc.sliding_window_mean):
        fn(x, k)
        fn(x, k, exact=True)
xr = torch.from_numpy(rng.standard_normal((2, 1000), dtype=np.float32)).cuda()
for k in (5, 40, 300):
    sc.sliding_window_max(xr, k)
    sc.sliding_window_sum(xr, k, exact=True)
img = torch.from_numpy(rng.uniform(0, 1, (2, 64, 256)).astype(np.float32)).cuda()
for k in (1, 3, 5, 7, 11):
    f = rng.standard_normal((k, k), dtype=np.float32)
    sc.conv2d_reference(img, f)
    sc.conv2d_reference(img, f, exact=True)
sc.conv2d_reference(img, rng.standard_normal((1, 7), dtype=np.float32))
sc.oracle_conv2d(img.double(), rng.standard_normal((3, 3)))
xn = torch.from_numpy(rng.standard_normal((1, 32, 16, 32), dtype=np.float32)).cuda()
wn = torch.from_numpy(rng.standard_normal((64, 32, 3, 3), dtype=np.float32)).cuda()
sc.conv2d_nchw(xn, wn, 1)
sc.conv2d_nchw(xn, wn, 1, exact=True)
sc.conv2d_im2col(img[0, :40, :50].contiguous(), rng.standard_normal((3, 3), dtype=np.float32))
h = np.ascontiguousarray(rng.standard_normal((3, 4096), dtype=np.float32))
sc.sliding_window_mean(h, 16)
sc.conv2d_reference(np.ascontiguousarray(img.cpu().numpy()), rng.standard_normal((5, 5), dtype=np.float32))
torch.cuda.synchronize()
print("sanitize cases done")
