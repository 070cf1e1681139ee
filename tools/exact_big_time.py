"""Exact sums for k > 512 on the config-2 input (256 x 262,144, and the
unaligned 256 x 262,143 as one flat signal): the tile +
pass composite (pool1d.cu launch_exact_big) vs the reference-structured global
passes (SC_POOL_NO_EXACT_BLOCK=1, run in a subprocess)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    if "--child" in sys.argv:
        import torch
        import paper_2310_05218_b200 as sc
        g = torch.Generator(device="cuda")
        g.manual_seed(2)
        res = {}
        for L, k in [(262144, 600), (262144, 1000), (262144, 2048), (262144, 3000), (262144, 4095),
                     (262144, 8191), (262143, 1000), (262143, 2048)]:
            x = torch.randn((256, L), device="cuda", generator=g)
            for _ in range(2):
                sc.sliding_window_sum(x, k, exact=True)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                sc.sliding_window_sum(x, k, exact=True)
            b.record()
            b.synchronize()
            res[f"L{L}_k{k}"] = round(a.elapsed_time(b) / 5, 3)
        print(json.dumps({"passes_only": os.environ.get("SC_POOL_NO_EXACT_BLOCK") is not None,
                          "ms": res}), flush=True)
        sys.exit(0)
    for env in ({}, {"SC_POOL_NO_EXACT_BLOCK": "1"}):
        subprocess.run([sys.executable, __file__, "--child"], env={**os.environ, **env}, check=False)
