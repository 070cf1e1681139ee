"""Row bands across several ranks with the real sm_100a kernel on halos
received from another rank (reference.py:15-23: output row r reads input rows
r .. r+kh-1 only, so band g plus the first kh-1 rows of band g+1 is exact).

* NCCL, one rank per GPU (min(8, device_count) ranks; skipped below 2 GPUs):
  the product path -- NCCL P2P over NVLink, halo received in place or as a
  separate boundary strip.
* gloo, 2 and 3 ranks sharing cuda:0: the exchange goes through host memory
  (rowband._exchange_halo_staged), the band convolution is still the CUDA
  kernel, run by each rank on its own band.  No rank's kernel waits on
  another's: the exchange completes on the host before the launch that reads
  it, so one GPU can host the ranks.
Exact mode must be bit-identical to the oracle on the whole image; fast mode
within the north-star tolerance and, for the fixed-size (<= 7x7) kernels,
bit-identical to the single-launch whole-image fast result (every output's
FFMA chain runs the taps in the same order in a band and in the whole image).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _image(h, w, kh, kw):
    rng = np.random.default_rng([0x5EED, 5, h, w, kh, kw])
    x = rng.uniform(-1, 1, (h, w)).astype(np.float32)
    f = (rng.standard_normal((kh, kw), dtype=np.float32) / np.float32(kh)).astype(np.float32)
    return x, f


def _worker(rank, world, port, backend, h, w, kh, kw, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_05218_b200 as sc
        x, f = _image(h, w, kh, kw)
        plan = sc.plan_row_bands(h, kh, world)[rank]
        rows = plan.in_stop - plan.in_start
        for exact in (True, False):
            for in_place in (False, True):
                if in_place:
                    band = sc.alloc_band(rows, w, kh, device=dev)
                    band[rows:] = float("nan")       # must be overwritten by the halo
                    band[:rows] = torch.from_numpy(x[plan.in_start:plan.in_stop]).to(dev)
                else:
                    band = torch.from_numpy(x[plan.in_start:plan.in_stop].copy()).to(dev)
                y, c = sc.conv2d_rowband(band, f, exact=exact, halo_in_place=in_place)
                assert y.is_cuda and y.shape[0] == plan.out_rows
                np.save(os.path.join(out_dir, f"r{rank}_e{int(exact)}_p{int(in_place)}.npy"),
                        y.cpu().numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, backend, h, w, kh, kw, tmp_path):
    import paper_2310_05218_b200 as sc
    port = _free_port()
    mp.spawn(_worker, args=(world, port, backend, h, w, kh, kw, str(tmp_path)), nprocs=world,
             join=True)
    x, f = _image(h, w, kh, kw)
    want = O.conv2d(x, f)
    whole_fast = sc.conv2d_reference(torch.from_numpy(x).cuda(), f, exact=False).cpu().numpy()
    for exact in (1, 0):
        for in_place in (0, 1):
            parts = [np.load(tmp_path / f"r{r}_e{exact}_p{in_place}.npy") for r in range(world)]
            got = np.concatenate(parts, axis=0)
            assert got.shape == want.shape
            if exact:
                assert np.array_equal(got, want), (world, backend, in_place)
            else:
                assert O.normwise_error(got, want) <= O.north_star_tol(kw)
                if kh <= 7:   # fixed-size kernels: same FFMA chain per output
                    assert np.array_equal(got, whole_fast), (world, backend, in_place)


@pytest.mark.parametrize("world,h,w,kh,kw", [(2, 515, 2048, 7, 7), (3, 301, 1030, 7, 7),
                                              (2, 200, 4096, 3, 3), (3, 180, 777, 11, 11),
                                              (2, 96, 1000, 5, 5)])
def test_rowband_gloo_ranks_cuda_kernel(world, h, w, kh, kw, tmp_path):
    _run(world, "gloo", h, w, kh, kw, tmp_path)


def test_rowband_nccl_ranks(tmp_path):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs for NCCL ranks (one rank per GPU)")
    world = min(8, n)
    _run(world, "nccl", 1024 + 7 * world, 8192, 7, 7, tmp_path)
