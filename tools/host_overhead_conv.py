"""Host cost per conv call on a device-resident 512x512 image, with a cProfile
breakdown (the harness showed ~50 us per call at k = 3)."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

x = torch.rand((512, 512), device="cuda")
vm = sc.VectorModel(16)
for k in (3, 11, 51):
    f = np.random.default_rng(k).uniform(-1, 1, (k, k)).astype(np.float32)
    fn = (lambda: sc.conv2d_custom3(x, f, vm)) if k == 3 else (lambda: sc.conv2d_slide_compound(x, f, vm))
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1e9))
    t0 = time.perf_counter()
    for _ in range(100):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"k={k}: host {1e6 * (t1 - t0) / 100:.1f} us/call, total incl. drain {1e6 * (t2 - t0) / 100:.1f}", flush=True)
f = np.random.default_rng(3).uniform(-1, 1, (3, 3)).astype(np.float32)
torch.cuda._sleep(int(1e9))
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    sc.conv2d_custom3(x, f, vm)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
