import sys, torch, json
sys.path.insert(0,'.')
import bench
import paper_2310_05218_b200 as sc
import torch.nn.functional as F
x = torch.randn((256, 262144), device='cuda')
for k in (3,16,64,255):
    a = bench.time_launches(torch, lambda: F.avg_pool1d(x.unsqueeze(1), k, stride=1), 20, 3)
    m = bench.time_launches(torch, lambda: F.max_pool1d(x.unsqueeze(1), k, stride=1), 20, 3)
    o = bench.time_launches(torch, lambda: sc.sliding_window_mean(x, k), 20, 3)
    print(k, f"torch avg {a*1e6:.1f}us max {m*1e6:.1f}us | ours avg {o*1e6:.1f}us")
