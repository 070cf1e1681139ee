import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2310_05218_b200 as sc
g = torch.Generator(device="cuda"); g.manual_seed(4)
x = torch.randn((16, 64, 112, 112), generator=g, device="cuda")
w = torch.randn((64, 64, 3, 3), generator=g, device="cuda") / 24
for _ in range(5): sc.conv2d_nchw(x, w, 1)
torch.cuda.synchronize()
def run(flush_elems, use_graph, sleep=0):
    flush = torch.empty(flush_elems, device="cuda")
    gr = None
    if use_graph:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            sc.conv2d_nchw(x, w, 1)
    ts = []
    for _ in range(30):
        flush.zero_()
        if sleep: torch.cuda._sleep(sleep)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        if gr is not None: gr.replay()
        else: sc.conv2d_nchw(x, w, 1)
        b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[15]
for fe, gph, sl in [(64 << 20, False, 0), (64 << 20, True, 0), (256 << 20, False, 0), (64 << 20, False, 1000000), (64 << 20, True, 1000000)]:
    try:
        print(f"flush {fe*4>>20} MB graph {gph} sleep {sl}: {run(fe, gph, sl)*1e3:.1f} us", flush=True)
    except Exception as e:
        print("fail", gph, repr(e)[:200])
