"""Interleaved A/B of tiles-per-CTA for the fused mean+max kernel under
sustained load (config 2): python tools/pair_tpc_ab.py 16 2,3,4,6"""
import os, sys, time, statistics, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_05218_b200 as sc
B, L = 256, 262144
k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
tpcs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "2,3,4").split(",")]
x = torch.randn((B, L), device="cuda")
fn = lambda: sc.sliding_window_mean_max(x, k)
t_end = time.time() + 1.5
while time.time() < t_end:
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
res = {t: [] for t in tpcs}
for rnd in range(12):
    for t in tpcs:
        os.environ["SC_POOL_TPC"] = str(t)
        t_hot = time.time() + float(os.environ.get("HOT", "0"))  # sustained load first
        while True:
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
            if time.time() >= t_hot:
                break
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda._sleep(int(2e9 * (50 * 100e-6 + 1e-3)))
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[t].append(e0.elapsed_time(e1) / 50 * 1e3)
for t in tpcs:
    v = res[t]
    print(f"k={k} tpc={t}: median {statistics.median(v):.1f} us  min {min(v):.1f}  max {max(v):.1f}")
