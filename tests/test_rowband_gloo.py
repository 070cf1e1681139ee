"""Row-band partitioner with a real halo exchange: world_size 2 and 3 `gloo`
process groups on CPU.  The band compute is the CPU oracle (injected `conv`);
the exchange, planning and assembly are the product code."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import slideconv_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, h, w, kh, kw, q, in_place=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_05218_b200 as sc
        rng = np.random.default_rng(11)
        x = rng.uniform(-1, 1, (h, w)).astype(np.float32)
        f = rng.standard_normal((kh, kw), dtype=np.float32)
        plan = sc.plan_row_bands(h, kh, world)[rank]
        rows = plan.in_stop - plan.in_start
        if in_place:
            band = sc.alloc_band(rows, w, kh)
            band[rows:] = float("nan")              # spare rows: must be overwritten
            band[:rows] = torch.from_numpy(x[plan.in_start:plan.in_stop])
        else:
            band = torch.from_numpy(x[plan.in_start:plan.in_stop].copy())

        def conv(a, b):
            return torch.from_numpy(O.conv2d(a.numpy(), b))

        y, c = sc.conv2d_rowband(band, f, conv=conv, halo_in_place=in_place)
        q.put((rank, plan.out_start, plan.out_stop, y.numpy(), c.macs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("in_place", [False, True])
@pytest.mark.parametrize("world,h,w,kh,kw", [(2, 64, 40, 7, 7), (3, 50, 33, 5, 3),
                                              (2, 31, 17, 1, 4)])
def test_rowband_gloo_matches_whole_image(world, h, w, kh, kw, in_place):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, w, kh, kw, q, in_place))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (h, w)).astype(np.float32)
    f = rng.standard_normal((kh, kw), dtype=np.float32)
    whole = O.conv2d(x, f)
    got = np.concatenate([r[3] for r in results], axis=0)
    assert got.shape == whole.shape
    assert np.array_equal(got, whole)          # banded == whole, bit for bit
    for rank, o0, o1, y, _ in results:
        assert y.shape[0] == o1 - o0
    assert sum(r[4] for r in results) == O.mac_count(h, w, kh, kw)
