"""Pooling (k=16 avg / max) and a same-size device copy timed under sustained
load (2 s of back-to-back launches first, so the clocks sit at the power cap)."""
import subprocess
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

x = torch.randn((256, 262144), device="cuda")
y = torch.empty_like(x)
tag = sys.argv[1] if len(sys.argv) > 1 else ""


def sustained(fn, n=100):
    t_end = time.time() + 2.0
    while time.time() < t_end:
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
    torch.cuda._sleep(int(2e9 * n * 40e-6))
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    return a.elapsed_time(b) / n * 1e3, clk


bytes_op = 4 * (x.numel() + 256 * (262144 - 15))
for name, fn in (("copy", lambda: y.copy_(x)), ("avg", lambda: sc.sliding_window_mean(x, 16)),
                 ("max", lambda: sc.sliding_window_max(x, 16))):
    t, clk = sustained(fn)
    nb = 8 * x.numel() if name == "copy" else bytes_op
    print(f"{tag} {name}: {t:.1f} us  {nb / t / 1e3:.0f} GB/s  (sm clock after: {clk} MHz)", flush=True)
