import sys, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc
dev = torch.device("cuda")
gen = torch.Generator(device=dev); gen.manual_seed(2)
xp = torch.randn((256, 262144), generator=gen, device=dev)
x2 = torch.randn((256, 262144), device=dev)
def t(fn, n=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / n * 1e3
for k in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else '3,16,64,255').split(',')]:
    print(k, "gen", round(t(lambda: sc.sliding_window_max(xp, k)), 1), "plain", round(t(lambda: sc.sliding_window_max(x2, k)), 1))
print("zeros in xp:", int((xp == 0).sum()))
