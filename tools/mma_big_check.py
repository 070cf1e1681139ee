"""Large-filter slide-MMA kernel (SC_CONV_MMA_BIG=1) against the float64
oracle and the FFMA kernels: python tools/mma_big_check.py [time]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_05218_b200 as sc

dev = torch.device("cuda")
do_time = len(sys.argv) > 1 and sys.argv[1] == "time"


def run(x, f, on):
    os.environ["SC_CONV_MMA_BIG"] = "2" if on else "0"
    y = sc.conv2d_reference(x, f, exact=False)
    torch.cuda.synchronize()
    return y


def timed(x, f, on, reps=10):
    os.environ["SC_CONV_MMA_BIG"] = "2" if on else "0"
    for _ in range(2):
        sc.conv2d_reference(x, f, exact=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        sc.conv2d_reference(x, f, exact=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


shapes = [((2, 200, 1300), 11, 11), ((1, 300, 2100), 17, 17), ((3, 256, 512), 25, 25),
          ((1, 130, 1024), 51, 51), ((1, 400, 1100), 53, 57), ((2, 90, 3000), 13, 31),
          ((1, 700, 777), 33, 10)]
if len(sys.argv) > 2 and sys.argv[2] == "sweep":
    shapes = [((32, 512, 512), k, k) for k in (13, 15, 19, 21, 23)] + \
             [((8, 1024, 1024), k, k) for k in (13, 15, 17, 19, 21, 25, 51)] + \
             [((4, 2048, 2048), k, k) for k in (13, 15, 19, 21)] + \
             [((1, 4096, 4096), 33, 3), ((1, 4096, 4096), 51, 5), ((1, 4096, 4096), 5, 51),
              ((1, 4096, 4096), 3, 33), ((1, 4096, 4096), 25, 9), ((1, 4096, 4096), 9, 25)]
elif do_time:
    shapes = [((32, 512, 512), k, k) for k in (11, 17, 25, 33, 51)] + \
             [((4, 2048, 2048), k, k) for k in (11, 17, 25, 33, 51)] + \
             [((1, 4096, 4096), k, k) for k in (17, 51)]
for shp, kh, kw in shapes:
    g = torch.Generator(device=dev); g.manual_seed(kh * 100 + kw)
    x = torch.rand(shp, generator=g, device=dev) * 2 - 1
    f = (np.random.default_rng(kh * kw).standard_normal((kh, kw)) / np.sqrt(kh * kw)).astype(np.float32)
    if do_time:
        t1 = timed(x, f, True); t0 = timed(x, f, False)
        macs = shp[0] * (shp[1] - kh + 1) * (shp[2] - kw + 1) * kh * kw
        print(f"{shp} {kh}x{kw}: mma {t1:.3f} ms ({2 * macs / t1 / 1e9:.0f} TFLOP/s useful)  ffma {t0:.3f} ms  x{t0 / t1:.2f}", flush=True)
        continue
    y1 = run(x, f, True).double().cpu()
    y0 = run(x, f, False).double().cpu()
    ref = torch.nn.functional.conv2d(x.double().cpu()[:, None], torch.from_numpy(f).double()[None, None])[:, 0]
    e1 = float((y1 - ref).norm() / ref.norm()); e0 = float((y0 - ref).norm() / ref.norm())
    print(f"{shp} {kh}x{kw}: mma normwise {e1:.2e} (tol {1e-5 * kw:.1e})  ffma {e0:.2e}  maxabs {float((y1-ref).abs().max()):.2e}", flush=True)
