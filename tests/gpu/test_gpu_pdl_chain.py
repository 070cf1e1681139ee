"""Back-to-back pooling launches on one stream with programmatic dependent
launch: each kernel may start while its predecessor drains, so a chain whose
every step reads the previous step's output (and overwrites a buffer the
step before read) checks that griddepcontrol.wait orders the memory."""

import numpy as np
import pytest
import torch

import paper_2310_05218_b200 as sc
from oracle import slideconv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [3, 16, 33])
def test_dependent_chain(k):
    rng = np.random.default_rng(k)
    x = rng.standard_normal((64, 65536), dtype=np.float32)
    cur = torch.from_numpy(x).cuda()
    want = x
    for step in range(6):
        fn, op = [(sc.sliding_window_sum, "sum"), (sc.sliding_window_max, "max"),
                  (sc.sliding_window_mean, "avg")][step % 3]
        cur = fn(cur, k, exact=True)[0] if op != "max" else fn(cur, k)[0]
        want = O.pool_batched(want, k, op)
    torch.cuda.synchronize()
    assert np.array_equal(cur.cpu().numpy(), want)


def test_buffer_reuse_war():
    # launch 1 reads `a`; launch 2 (queued right behind it) writes its output
    # into `a`'s storage: launch 1 must still see the original `a`
    rng = np.random.default_rng(7)
    n, L, k = 128, 131072, 16
    a_np = rng.standard_normal((n, L), dtype=np.float32)
    b_np = rng.standard_normal((n, L), dtype=np.float32)
    lib = sc._lib.load()
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(10):
        a = torch.from_numpy(a_np).cuda()
        b = torch.from_numpy(b_np).cuda()
        ya = torch.empty((n, L - k + 1), device="cuda")
        torch.cuda.synchronize()
        assert lib.sc_pool1d_f32(2, a.data_ptr(), n, L, k, 0, ya.data_ptr(), st) == 0
        assert lib.sc_pool1d_f32(2, b.data_ptr(), n, L, k, 0, a.data_ptr(), st) == 0
        torch.cuda.synchronize()
        assert np.array_equal(ya.cpu().numpy(), O.pool_batched(a_np, k, "max"))
        got_b = a.cpu().numpy().reshape(-1)[: n * (L - k + 1)].reshape(n, L - k + 1)
        assert np.array_equal(got_b, O.pool_batched(b_np, k, "max"))
