"""Alternating avg / max pooling launches: device time per launch with and
without CUDA events between the launches (host run-ahead in both cases)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2310_05218_b200 as sc  # noqa: E402

x = torch.randn((256, 262144), device="cuda")
n = 50


def run(events: bool):
    t_end = time.time() + 1.0
    while time.time() < t_end:
        sc.sliding_window_mean(x, 16)
        sc.sliding_window_max(x, 16)
    torch.cuda.synchronize()
    torch.cuda._sleep(int(2e9 * n * 2 * 40e-6))
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    ev = [torch.cuda.Event(True) for _ in range(2 * n)] if events else None
    a.record()
    for i in range(n):
        if events:
            ev[2 * i].record()
        sc.sliding_window_mean(x, 16)
        if events:
            ev[2 * i + 1].record()
        sc.sliding_window_max(x, 16)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (2 * n) * 1e3


for events in (False, True, False, True):
    print(f"events={events}: {run(events):.1f} us per launch", flush=True)
