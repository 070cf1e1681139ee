"""Randomised parity soak on the GPU (evidence for profiles/): the reference's
property suite over many seeds, plus random shapes / windows / filters for
every kernel family against the CPU oracle -- exact mode bit-identical, fast
mode within the north-star tolerance, max pooling always bit-exact.

usage: python tools/soak.py [seconds]   (prints one summary line per family)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402
from oracle import slideconv_oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
t_end = time.time() + budget
rng = np.random.default_rng(20261020)
stats = {}


def note(fam, ok, detail=""):
    s = stats.setdefault(fam, [0, 0, []])
    s[0] += 1
    if not ok:
        s[1] += 1
        if len(s[2]) < 5:
            s[2].append(detail)


# 1. the reference's property suite, many seeds
for seed in range(12):
    rep = sc.verify_suite(seed=seed, trials=40)
    note("verify_suite", rep.passed, f"seed {seed}: {rep.summary()}")

FNS = {"sum": sc.sliding_window_sum, "avg": sc.sliding_window_mean, "max": sc.sliding_window_max}
while time.time() < t_end:
    # 2. pooling: random lengths (aligned and ragged), windows 1..5000, batch 1..4
    aligned = rng.random() < 0.6
    n = int(rng.integers(1024, 40000))
    n = n // 32 * 32 if aligned else n
    k = int(min(n, rng.choice([rng.integers(1, 34), rng.integers(34, 300), rng.integers(300, 700),
                                rng.integers(700, 5000)])))
    b = int(rng.integers(1, 5))
    x = rng.standard_normal((b, n), dtype=np.float32) * np.float32(rng.choice([1e-3, 1.0, 1e3]))
    if rng.random() < 0.2:
        x[0, rng.integers(0, n)] = rng.choice([np.inf, -np.inf, np.nan])
    if rng.random() < 0.3:
        x[:, ::int(rng.integers(2, 50))] = np.float32(rng.choice([0.0, -0.0]))
    xd = torch.from_numpy(x).cuda()
    for op, fn in FNS.items():
        want = O.pool_batched(x, k, op)
        got_e = fn(xd, k, exact=True)[0].cpu().numpy()
        same = np.array_equal(np.isnan(got_e), np.isnan(want)) and np.array_equal(
            got_e[~np.isnan(want)].view(np.uint32), want[~np.isnan(want)].view(np.uint32))
        note(f"pool {op} exact", same, f"n={n} k={k} b={b}")
        got_f = fn(xd, k)[0].cpu().numpy()
        if op == "max":
            note("pool max fast", np.array_equal(np.isnan(got_f), np.isnan(want)) and np.array_equal(
                got_f[~np.isnan(want)].view(np.uint32), want[~np.isnan(want)].view(np.uint32)),
                f"n={n} k={k}")
        elif np.isfinite(x).all():
            note(f"pool {op} fast", O.normwise_error(got_f, want) <= O.north_star_tol(k),
                 f"n={n} k={k}")
    # 2b. the fused pair: bit-identical to the single-op calls, both modes
    for mean in (False, True):
        pair = sc.sliding_window_mean_max if mean else sc.sliding_window_sum_max
        one = sc.sliding_window_mean if mean else sc.sliding_window_sum
        for ex in (False, True):
            (ya, _), (ym, _) = pair(xd, k, exact=ex)
            ra = one(xd, k, exact=ex)[0]
            rm = sc.sliding_window_max(xd, k, exact=ex)[0]
            same = all(np.array_equal(np.isnan(a_), np.isnan(b_)) and np.array_equal(
                a_[~np.isnan(b_)].view(np.uint32), b_[~np.isnan(b_)].view(np.uint32))
                for a_, b_ in ((ya.cpu().numpy(), ra.cpu().numpy()),
                               (ym.cpu().numpy(), rm.cpu().numpy())))
            note("pool pair", same, f"n={n} k={k} b={b} mean={mean} exact={ex}")
    # 3. 2-D conv: random shapes and filters (square and not, 1..64)
    kh = int(rng.choice([1, 3, 5, 7, rng.integers(1, 65)]))
    kw = int(rng.choice([kh, rng.integers(1, 65)]))
    h = int(rng.integers(kh, kh + 300))
    w = int(rng.integers(kw, kw + 700))
    b = int(rng.integers(1, 4))
    x = rng.uniform(-1, 1, (b, h, w)).astype(np.float32)
    f = rng.standard_normal((kh, kw), dtype=np.float32)
    xd = torch.from_numpy(x).cuda()
    want = O.conv2d_batched(x, f)
    note("conv2d exact", np.array_equal(sc.conv2d_reference(xd, f, exact=True).cpu().numpy(), want),
         f"{b}x{h}x{w} f{kh}x{kw}")
    fast = sc.conv2d_reference(xd, f).cpu().numpy()
    ref64 = np.stack([O.oracle_conv2d(img, f) for img in x])
    note("conv2d fast", O.normwise_error(fast, ref64) <= O.north_star_tol(max(kh, kw)),
         f"{b}x{h}x{w} f{kh}x{kw}")
    # 3b. the large-filter tensor-core kernel, forced (kh <= 53, kw <= 57):
    # tolerance, and the FFMA kernels' inf / NaN pattern
    if 2 <= kh <= 53 and 2 <= kw <= 57:
        xs = x.copy()
        if rng.random() < 0.3:
            xs[0, rng.integers(0, h), rng.integers(0, w)] = rng.choice([np.inf, np.nan, 1e35, -np.inf])
        xs *= np.float32(rng.choice([1e-6, 1.0, 1e5]))
        xsd = torch.from_numpy(xs).cuda()
        if rng.random() < 0.5:
            os.environ["SC_MMA_BIG_ROWS"] = str(int(rng.integers(1, 80)))
        os.environ["SC_CONV_MMA_BIG"] = "2"
        got = sc.conv2d_reference(xsd, f).cpu().numpy()
        os.environ["SC_CONV_MMA_BIG"] = "0"
        os.environ.pop("SC_MMA_BIG_ROWS", None)
        ref = sc.conv2d_reference(xsd, f).cpu().numpy()
        os.environ.pop("SC_CONV_MMA_BIG", None)
        fin = np.isfinite(ref)
        ok = (np.array_equal(np.isnan(got), np.isnan(ref)) and np.array_equal(np.isinf(got), np.isinf(ref))
              and O.normwise_error(got[fin], ref[fin]) <= O.north_star_tol(max(kh, kw)))
        note("conv2d mma_big", ok, f"{b}x{h}x{w} f{kh}x{kw}")
    # 4. NCHW 3x3 pad 1 (tensor-core and CUDA-core paths)
    if rng.random() < 0.25:
        cin = int(rng.choice([32, 64, 128, 3, 17]))
        cout = int(rng.choice([64, 128, 8]))
        hh, ww = int(rng.integers(4, 40)), int(rng.choice([16, 32, 48, 23]))
        nb = int(rng.integers(1, 3))
        xn = rng.standard_normal((nb, cin, hh, ww), dtype=np.float32)
        wn = (rng.standard_normal((cout, cin, 3, 3), dtype=np.float32) / np.float32(3 * cin ** 0.5))
        got = sc.conv2d_nchw(torch.from_numpy(xn).cuda(), torch.from_numpy(wn).cuda(), 1)
        got = got.cpu().numpy()
        want64 = O.conv2d_nchw_f64(xn, wn, 1)
        note("nchw fast", O.normwise_error(got, want64) <= O.north_star_tol(3, cin),
             f"{nb}x{cin}x{hh}x{ww} -> {cout}")
        got_e = sc.conv2d_nchw(torch.from_numpy(xn).cuda(), torch.from_numpy(wn).cuda(), 1,
                               exact=True).cpu().numpy()
        note("nchw exact", np.array_equal(got_e, O.conv2d_nchw(xn, wn, 1)),
             f"{nb}x{cin}x{hh}x{ww} -> {cout}")

for fam, (n, bad, ex) in stats.items():
    print(f"{fam:18s} cases {n:6d}  failures {bad}" + (f"  e.g. {ex}" if bad else ""), flush=True)
print("ALL PASS" if all(v[1] == 0 for v in stats.values()) else "FAILURES", flush=True)
