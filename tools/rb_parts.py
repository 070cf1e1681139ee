import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2310_05218_b200 as sc
from paper_2310_05218_b200 import _ops
H=W=65536; rows=H//8
x=torch.rand((rows+6, W), device='cuda')
f7=np.random.default_rng(1).standard_normal((7,7),dtype=np.float32)/7
y=torch.empty((rows, W-6), device='cuda')
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize(); a=torch.cuda.Event(True); b=torch.cuda.Event(True); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/n
band=x[:rows]; halo=x[rows:rows+6].clone()
print('interior', t(lambda: _ops.conv2d_into(band, f7, y[:rows-6])))
edge=torch.cat([band[rows-6:], halo]); print('edge conv', t(lambda: _ops.conv2d_into(edge, f7, y[rows-6:])))
print('cat', t(lambda: torch.cat([band[rows-6:], halo])))
print('one launch rows+6', t(lambda: _ops.conv2d_into(x, f7, y)))
