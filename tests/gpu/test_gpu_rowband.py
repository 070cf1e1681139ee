"""Row-band path on the GPU through a real NCCL process group (world 1 here:
this run has one GPU; the multi-rank exchange is covered by the gloo tests
and by the virtual-band test in test_gpu_conv.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_rowband_single_rank_equals_whole(nccl_world1):
    rng = np.random.default_rng(55)
    x = rng.uniform(-1, 1, (1030, 4096)).astype(np.float32)
    f = rng.standard_normal((7, 7), dtype=np.float32)
    y, c = sc.conv2d_rowband(torch.from_numpy(x).cuda(), f, exact=True)
    assert np.array_equal(y.cpu().numpy(), O.conv2d(x, f))
    assert c.macs == O.mac_count(1030, 4096, 7, 7)


def test_rowband_single_rank_halo_in_place(nccl_world1):
    rng = np.random.default_rng(56)
    x = rng.uniform(-1, 1, (777, 2048)).astype(np.float32)
    f = rng.standard_normal((7, 7), dtype=np.float32)
    buf = sc.alloc_band(777, 2048, 7, device="cuda")
    buf[777:] = float("nan")                     # the last rank never reads the spare rows
    buf[:777] = torch.from_numpy(x).cuda()
    y, c = sc.conv2d_rowband(buf, f, exact=True, halo_in_place=True)
    assert np.array_equal(y.cpu().numpy(), O.conv2d(x, f))
    assert c.macs == O.mac_count(777, 2048, 7, 7)


def test_rowband_plan_band_sizes():
    for g in (1, 2, 4, 8):
        plans = sc.plan_row_bands(65536, 7, g)
        assert sum(p.out_rows for p in plans) == 65530
        assert all(p.in_stop - p.in_start == 65536 // g for p in plans)
