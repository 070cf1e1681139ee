"""GPU check + timing of the slide-MMA conv kernel (csrc/conv2d_mma.cu).

python tools/mma_check.py [--big]   (needs a GPU; SC_CONV_MMA=0 selects the
FFMA kernels for the comparison run, which this script does in a subprocess)
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def conv(x, f, exact=False):
    import paper_2310_05218_b200 as sc
    y, _ = sc.conv2d_slide_compound(x, f, sc.VectorModel(16), exact=exact)
    return y


def check_shapes():
    import torch
    from oracle import slideconv_oracle as O
    rng = np.random.default_rng(7)
    cases = [((2, 4096, 4096), (7, 7)), ((1, 3000, 10240), (7, 7)), ((2, 2048, 8192), (9, 9)),
             ((2, 2048, 8192), (6, 8)), ((1, 2048, 12288), (9, 9)), ((3, 1500, 8448), (7, 7)),
             ((2, 2048, 8192), (8, 5))]
    out = []
    os.environ.setdefault("SC_CONV_MMA", "1")
    for shape, (kh, kw) in cases:
        x = rng.uniform(-1, 1, shape).astype(np.float32)
        f = (rng.standard_normal((kh, kw)) / np.sqrt(kh * kw)).astype(np.float32)
        got = conv(torch.from_numpy(x).cuda(), f).cpu().numpy()
        want = O.conv2d_batched(x, f)
        err = O.normwise_error(got, want)
        tol = O.north_star_tol(kw)
        out.append({"shape": shape, "k": (kh, kw), "err": err, "tol": tol, "ok": err <= tol})
        print(json.dumps(out[-1]), flush=True)
    # non-finite inputs: tiles recomputed with FMAs
    x = rng.uniform(-1, 1, (2, 4096, 4096)).astype(np.float32)
    x[0, 100, 200] = np.inf
    x[1, 3000, 1030] = np.nan
    x[1, 10, 4000] = -np.inf
    f = (rng.standard_normal((7, 7)) / 7).astype(np.float32)
    got = conv(torch.from_numpy(x).cuda(), f).cpu().numpy()
    want = O.conv2d_batched(x, f)
    fin = np.isfinite(want)
    same_mask = bool(np.array_equal(np.isnan(got), np.isnan(want)) and
                     np.array_equal(np.isposinf(got), np.isposinf(want)) and
                     np.array_equal(np.isneginf(got), np.isneginf(want)))
    err = O.normwise_error(got[fin], want[fin])
    print(json.dumps({"nonfinite": True, "mask_equal": same_mask, "err_finite": err}), flush=True)
    return out


def time_cfg5(reps=10, sustain_s=0.0):
    import torch
    import paper_2310_05218_b200 as sc
    h = w = 65536
    x = torch.empty((h, w), device="cuda", dtype=torch.float32)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x.uniform_(-1, 1, generator=g)
    f = (np.random.default_rng(5).standard_normal((7, 7)) / 7).astype(np.float32)
    y = torch.empty((h - 6, w - 6), device="cuda", dtype=torch.float32)
    from paper_2310_05218_b200 import _ops
    for _ in range(2):
        _ops.conv2d_into(x, f, y)
    torch.cuda.synchronize()
    import time
    t_end = time.time() + sustain_s
    while time.time() < t_end:
        for _ in range(20):
            _ops.conv2d_into(x, f, y)
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        _ops.conv2d_into(x, f, y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    byts = 4 * (h * w + (h - 6) * (w - 6) + 49)
    # oracle bands: first / last / a segment boundary
    from oracle import slideconv_oracle as O
    rows = int(sc._lib.load().sc_conv2d_segment_rows(1, h, w, 7, 7, 0))
    errs = []
    for r in (0, h - 6 - 64, max(0, rows - 32) if rows > 0 else 5000, 32768 - 30):
        band = x[r:r + 70].cpu().numpy()
        want = O.conv2d(band, f)
        got = y[r:r + 64].cpu().numpy()
        errs.append(O.normwise_error(got, want))
    print(json.dumps({"sustain_s": sustain_s, "cfg5_ms": round(ms, 3), "gbs": round(byts / ms / 1e6, 1),
                      "mma": os.environ.get("SC_CONV_MMA", "1"), "band_errs": errs,
                      "seg_rows": rows}), flush=True)


if __name__ == "__main__":
    if "--time" in sys.argv:
        time_cfg5(reps=20, sustain_s=float(os.environ.get("SUSTAIN", "0")))
        sys.exit(0)
    if "--sustained" in sys.argv:
        for env in ("1", "0", "1", "0"):
            subprocess.run([sys.executable, __file__, "--time"],
                           env={**os.environ, "SC_CONV_MMA": env, "SUSTAIN": "3"}, check=False)
        sys.exit(0)
    check_shapes()
    if "--big" in sys.argv:
        for env in ("1", "0"):
            subprocess.run([sys.executable, __file__, "--time"],
                           env={**os.environ, "SC_CONV_MMA": env}, check=False)
