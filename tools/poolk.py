"""Per-launch device time of sum / avg / max pooling on config 2 (256 x 262,144)
for the given windows: python tools/poolk.py 64 255"""
import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2310_05218_b200 as sc
x = torch.randn((256, 262144), device="cuda")
for k in [int(v) for v in sys.argv[1:]]:
    for op in ("max", "sum", "avg"):
        fn = {"max": sc.sliding_window_max, "sum": sc.sliding_window_sum, "avg": sc.sliding_window_mean}[op]
        for _ in range(3): fn(x, k)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda._sleep(200000)   # park the stream so the events time device work only
            e0.record(); fn(x, k); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ts.sort(); ms = ts[10]
        print(f"k={k} {op}: {ms*1e3:.1f} us  {4*(x.numel()*2)/ms/1e6:.0f} GB/s")
