"""Device time of conv2d_nchw (3x3, pad 1, fast mode) over CNN-like shapes."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402


def bench(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n * 1e3


for nb, cin, cout, hw in [(16, 64, 64, 112), (32, 64, 64, 56), (16, 128, 128, 56), (32, 128, 128, 28),
                          (16, 256, 256, 28), (64, 64, 64, 56), (8, 32, 64, 112)]:
    x = torch.randn((nb, cin, hw, hw), device="cuda")
    w = torch.randn((cout, cin, 3, 3), device="cuda") / (3 * cin ** 0.5)
    t = bench(lambda: sc.conv2d_nchw(x, w, 1))
    tc = bench(lambda: torch.nn.functional.conv2d(x, w, padding=1))
    fl = 2 * nb * cout * cin * 9 * hw * hw
    print(f"N{nb} C{cin}->{cout} {hw}x{hw}: {t:7.1f}us {fl / t / 1e6:5.0f} TF(fp32-eq) | "
          f"torch(cuDNN, TF32 {torch.backends.cudnn.allow_tf32}) {tc:7.1f}us", flush=True)
