"""Fused mean+max pooling vs the two single-op launches on config 2
(256 x 262,144), back-to-back launches between two events with the stream
parked: python tools/pair_time.py 16 3 64   (SC_POOL_TPC=n sweeps tiles/CTA)"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_05218_b200 as sc
B, L = 256, 262144
x = torch.randn((B, L), device="cuda")
reps = int(os.environ.get('REPS', 40))


def timed(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    if os.environ.get("SUSTAIN"):  # ~1 s of the same work first: power-capped clocks
        import time
        t_end = time.time() + float(os.environ["SUSTAIN"])
        while time.time() < t_end:
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda._sleep(int(2e9 * (reps * 150e-6 + 1e-3)))
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for k in [int(v) for v in sys.argv[1:]] or [16]:
    o = B * (L - k + 1)
    two = timed(lambda: (sc.sliding_window_mean(x, k), sc.sliding_window_max(x, k)))
    one = timed(lambda: sc.sliding_window_mean_max(x, k))
    cp = torch.empty_like(x)
    cpt = timed(lambda: cp.copy_(x))
    print(f"k={k} tpc={os.environ.get('SC_POOL_TPC', 'dflt')}: two launches {two:.1f} us "
          f"({2 * 4 * (B * L + o) / two / 1e3:.0f} GB/s), fused {one:.1f} us "
          f"({4 * (B * L + 2 * o) / one / 1e3:.0f} GB/s of its 3 streams), copy {cpt:.1f} us "
          f"({8 * B * L / cpt / 1e3:.0f} GB/s)", flush=True)
