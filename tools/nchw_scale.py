import sys, torch
sys.path.insert(0, '.')
import paper_2310_05218_b200 as sc
def bench(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a=torch.cuda.Event(True); b=torch.cuda.Event(True); a.record()
    for _ in range(n): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b)/n*1e3
for nb in (4, 8, 16, 32, 64):
    x = torch.randn((nb, 64, 112, 112), device='cuda'); w = torch.randn((64, 64, 3, 3), device='cuda') / 24
    t = bench(lambda: sc.conv2d_nchw(x, w, 1))
    print(nb, f"{t:.1f}us", f"{2*nb*64*64*9*112*112/t/1e6:.0f} TFLOP/s(fp32-equiv)")
