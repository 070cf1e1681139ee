"""Small fixed workloads for ncu captures (one launch family per name)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "pool16"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda")
g = torch.Generator(device=dev)
g.manual_seed(1)
vm = sc.VectorModel(16)
if which.startswith("psum") or which.startswith("pavg") or which.startswith("pmax"):
    k = int(which[4:])
    fn = {"psum": sc.sliding_window_sum, "pavg": sc.sliding_window_mean,
          "pmax": sc.sliding_window_max}[which[:4]]
    x = torch.randn((256, 262144), generator=g, device=dev)
    for _ in range(reps):
        fn(x, k)
elif which.startswith("pair"):
    k = int(which[4:])
    x = torch.randn((256, 262144), generator=g, device=dev)
    for _ in range(reps):
        sc.sliding_window_mean_max(x, k)
elif which.startswith("pool"):
    k = int(which[4:])
    x = torch.randn((256, 262144), generator=g, device=dev)
    for _ in range(reps):
        sc.sliding_window_mean(x, k)
        sc.sliding_window_max(x, k)
        sc.sliding_window_sum(x, k)
elif which in ("conv3", "conv5"):
    k = int(which[4:])
    x = torch.rand((32, 4096, 4096), generator=g, device=dev)
    f = np.random.default_rng(k).standard_normal((k, k), dtype=np.float32) / k
    for _ in range(reps):
        sc.conv2d_reference(x, f, exact=False)
elif which == "conv1d":
    x = torch.rand((64, 1 << 20), generator=g, device=dev)
    f = np.random.default_rng(1).standard_normal((1, 7), dtype=np.float32)
    for _ in range(reps):
        sc.conv2d_reference(x, f, exact=False)
elif which == "conv7full":
    # config 5 itself: one 65,536^2 image (16 GiB in + 16 GiB out)
    x = torch.empty((65536, 65536), device=dev)
    x.uniform_(-1, 1, generator=g)
    f = np.random.default_rng(7).standard_normal((7, 7), dtype=np.float32) / 7
    y = torch.empty((65530, 65530), device=dev)
    from paper_2310_05218_b200 import _ops
    for _ in range(reps):
        _ops.conv2d_into(x, f, y)
elif which == "conv7":
    x = torch.rand((16384, 65536), generator=g, device=dev)
    f = np.random.default_rng(7).standard_normal((7, 7), dtype=np.float32) / 7
    for _ in range(reps):
        sc.conv2d_reference(x, f, exact=False)
elif which.startswith("big"):
    k = int(which[3:])
    x = torch.rand((32, 512, 512), generator=g, device=dev)
    f = np.random.default_rng(k).standard_normal((k, k), dtype=np.float32) / k
    for _ in range(reps):
        sc.conv2d_reference(x, f, exact=False)
elif which == "nchw":
    x = torch.randn((16, 64, 112, 112), generator=g, device=dev)
    w = torch.randn((64, 64, 3, 3), generator=g, device=dev) / 24
    for _ in range(reps):
        sc.conv2d_nchw(x, w, 1)
torch.cuda.synchronize()
print("done", which)
