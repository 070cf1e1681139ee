"""Time the wide-window pooling kernels (pool_wide.cu) per op and window."""
import sys, torch
sys.path.insert(0, '.')
import paper_2310_05218_b200 as sc
x = torch.randn((256, 262144), device='cuda')
fns = {"sum": sc.sliding_window_sum, "avg": sc.sliding_window_mean, "max": sc.sliding_window_max}
if len(sys.argv) > 1:          # one launch per (op, k) for ncu
    for op in sys.argv[1].split(','):
        for k in [int(v) for v in sys.argv[2].split(',')]:
            fns[op](x, k)
    torch.cuda.synchronize()
    sys.exit()
for k in (100, 200, 255, 300, 1000, 2049):
    row = []
    for op, fn in fns.items():
        for _ in range(3): fn(x, k)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(20): fn(x, k)
        b.record(); b.synchronize()
        row.append(f"{op} {a.elapsed_time(b)/20*1e3:.1f}us")
    print(k, *row, flush=True)
