import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O
from tests.gpu.test_gpu_pool_robust import _spiky, _window_abs_sum, EPS32
for (k, n) in [(34, 32*1061), (255, 32*1061), (100, 9001)]:
    b = 32 if n % 32 else 6
    x = _spiky(b, n, 4242 + k + n)
    xd = torch.from_numpy(x).cuda()
    want = O.pool_batched(x, k, "sum")
    got = sc.sliding_window_sum(xd, k)[0].cpu().numpy()
    fin = np.isfinite(want)
    A = _window_abs_sum(x, k)
    err = np.where(fin, np.abs(got.astype(np.float64) - want), 0)
    rel = err / np.maximum(A, 1e-30)
    idx = np.unravel_index(np.argmax(rel), rel.shape)
    print(k, n, "worst rel", rel[idx], idx, got[idx], want[idx], A[idx])
    bad = np.argwhere(rel > 2 * k * EPS32)
    print(" n bad", len(bad), bad[:10].tolist())
    r, c = idx
    print(" x window", x[r, c:c+k].tolist()[:40])
