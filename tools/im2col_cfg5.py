import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2310_05218_b200 as sc
from paper_2310_05218_b200 import _lib as L_
lib = L_.load()
dev = torch.device('cuda')
xb = torch.empty((65536, 65536), device=dev)
for r0 in range(0, 65536, 8192): xb[r0:r0+8192].uniform_(-1, 1)
f7 = (np.random.default_rng(5).standard_normal((7, 7), dtype=np.float32) / 7).astype(np.float32)
o = 65530
yc = torch.empty((o, o), device=dev); cols = torch.empty(256 * o * 49, device=dev)
fdk = torch.from_numpy(f7.reshape(-1)).to(dev)
st = torch.cuda.current_stream()
for _ in range(2):
    a=torch.cuda.Event(True); b=torch.cuda.Event(True); a.record()
    rc = lib.sc_conv2d_im2col_f32(xb.data_ptr(), 65536, 65536, fdk.data_ptr(), 7, 7, cols.data_ptr(), 256, yc.data_ptr(), st.cuda_stream)
    b.record(); b.synchronize(); print('rc', rc, 'ms', a.elapsed_time(b))
del cols
y = sc.conv2d_reference(xb, f7)
for r in (0, 1000, 40000, 65529):
    d = (y[r] - yc[r]).abs().max().item(); print(r, d)
