"""Per-role clock64 timeline of CTA (0,0,0) of the large-filter slide-MMA
kernel: python tools/mma_big_trace.py B H W K"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_05218_b200 as sc
b, h, w, k = (int(v) for v in sys.argv[1:5])
x = torch.rand((b, h, w), device="cuda") * 2 - 1
f = (np.random.default_rng(k).standard_normal((k, k)) / k).astype(np.float32)
tr = torch.zeros(8 * 1024 + 5 * 2048 + 64, dtype=torch.int64, device="cuda")
os.environ["SC_CONV_MMA_BIG"] = "2"
for _ in range(2):
    sc.conv2d_reference(x, f, exact=False)
os.environ["SC_MMA_BIG_TRACE"] = hex(tr.data_ptr())
sc.conv2d_reference(x, f, exact=False)
torch.cuda.synchronize()
raw = tr.cpu().numpy()
t = raw[:8 * 1024].reshape(8, 1024)
g = raw[8 * 1024:8 * 1024 + 4 * 2048].reshape(-1, 4)
mid = raw[8 * 1024 + 4 * 2048:8 * 1024 + 5 * 2048]
life = (g[:, 1] - g[:, 0]) / 1e3
order = np.argsort(-life)[:10]
print("slowest CTAs (linear index: lifetime us, of which range scan us):",
      [(int(i), round(float(life[i]), 1), round(float(g[i, 2] - g[i, 0]) / 1e3, 1),
        "issuer mid/last us", round(float(mid[i] - g[i, 0]) / 1e3, 1), round(float(g[i, 3] - g[i, 0]) / 1e3, 1))
       for i in order if g[i, 0] > 0])
print("range scan us min/median/max", [round(float(v) / 1e3, 1) for v in np.percentile((g[:, 2] - g[:, 0])[g[:, 0] > 0], [0, 50, 100])])
g = g[g[:, 0] > 0]
print("CTAs", len(g), "entry spread us", (g[:, 0].max() - g[:, 0].min()) / 1e3, "lifetime us min/median/max",
      (g[:, 1] - g[:, 0]).min() / 1e3, float(np.median(g[:, 1] - g[:, 0])) / 1e3, (g[:, 1] - g[:, 0]).max() / 1e3,
      "kernel span us", (g[:, 1].max() - g[:, 0].min()) / 1e3)
t0 = t[7, 0]
print("kernel entry -> set-up done", t0 - t[7, 3], "; range scan + filter image copy", t[7, 1] - t0,
      "; all roles done", t[7, 2] - t0)
names = ["split_wait_done", "split_publish", "iss_begin", "iss_split_ready", "iss_commit", "epi_begin", "epi_end"]
n = int((t[4] > 0).sum())
print("batches", n)
print("b  " + " ".join(f"{s:>16}" for s in names))
for i in list(range(0, min(n, 12))) + list(range(max(12, n - 4), n)):
    print(f"{i:<3}" + " ".join(f"{(t[r, i] - t0) if t[r, i] else -1:>16}" for r in range(7)))
d = np.diff(t[4, :n])
print("issuer period per batch: median", np.median(d), "mean", d.mean())
print("issue time per batch (commit - split_ready): median", np.median(t[4, :n] - t[3, :n]))
print("split: publish - wait_done median", np.median(t[1, :n] - t[0, :n]))
m = t[6] > 0   # the traced warp drains every other batch (two epilogue groups)
print("epilogue body median", np.median((t[6] - t[5])[m]), "batches", int(m.sum()))
print("last commit", t[4, n - 1] - t0, "last traced epilogue end", t[6][m].max() - t0)
