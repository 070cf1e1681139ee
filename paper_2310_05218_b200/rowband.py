"""Row-band partitioner for very large single-image convolutions (new;
BASELINE config 5: one 65,536^2 image, 7x7, split across 1/2/4/8 GPUs).

A valid conv output row r reads input rows r .. r+kh-1 only
(reference.py:19-22), so an image split into row bands is exact when every
band also sees the first kh-1 rows of the next band (banded evaluation is
bit-identical to the whole image).  One process per GPU:

  rank g owns input rows [start_g, stop_g) on its device;
  1. post the halo exchange (torch.distributed P2P over NCCL -> NVLink):
     send my first kh-1 rows to g-1, receive the next band's first kh-1 rows
     from g+1 -- 6 x W floats per neighbour pair for 7x7;
  2. meanwhile run the conv on the rows that need no halo (output rows
     [start_g, stop_g - kh + 1)), on the compute stream;
  3. wait for the halo, then run the (kh-1)-row boundary strip.
The last rank has no successor and produces stop - kh + 1 rows.  Batches
(configs 1-3) shard with no communication at all; see bench.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .tensor import ConvShape, CostCounters, ShapeError, as_filter2d, mac_count


@dataclass(frozen=True)
class RowBandPlan:
    """Band g: input rows [in_start, in_stop) owned, output rows
    [out_start, out_stop) produced, halo rows received from g+1."""

    rank: int
    world: int
    in_start: int
    in_stop: int
    out_start: int
    out_stop: int
    halo: int

    @property
    def out_rows(self) -> int:
        return self.out_stop - self.out_start

    @property
    def interior_rows(self) -> int:
        """Output rows computable from owned rows alone."""
        return max(0, min(self.out_stop, self.in_stop - self.halo) - self.out_start)


def plan_row_bands(h: int, kh: int, world: int) -> list[RowBandPlan]:
    """Equal row bands (the last takes the remainder); every band but the last
    receives kh-1 halo rows from its successor."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if kh < 1 or h < kh:
        raise ShapeError(f"filter height {kh} exceeds image height {h}")
    rows = h // world
    halo = kh - 1
    if world > 1 and rows < max(1, halo):
        raise ShapeError(f"{world} bands of {rows} rows cannot carry a {halo}-row halo")
    oh = h - kh + 1
    plans = []
    for g in range(world):
        a = g * rows
        b = (g + 1) * rows if g < world - 1 else h
        o1 = min(b, oh)
        plans.append(RowBandPlan(g, world, a, b, a, max(a, o1), halo if g < world - 1 else 0))
    return plans


def exchange_halo(x_local, halo: int, group=None, recv=None):
    """Post the halo exchange for this rank's band; returns (recv_buf, works).

    Sends x_local[:halo] to rank-1 and receives `halo` rows from rank+1 with
    one batched NCCL (or gloo) P2P group -- into `recv` when given (e.g. the
    spare rows after the band), else into a new buffer.  Caller waits on
    `works` before touching recv_buf."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if x_local.is_cuda and dist.get_backend(group) != "nccl":
        return _exchange_halo_staged(x_local, halo, group, recv)
    ops = []
    if halo > 0 and world > 1:
        if rank > 0:
            send = x_local[:halo].contiguous()
            ops.append(dist.P2POp(dist.isend, send, dist.get_global_rank(group, rank - 1)
                                  if group is not None else rank - 1, group))
        if rank < world - 1:
            if recv is None:
                recv = torch.empty((halo,) + tuple(x_local.shape[1:]), dtype=x_local.dtype,
                                   device=x_local.device)
            ops.append(dist.P2POp(dist.irecv, recv, dist.get_global_rank(group, rank + 1)
                                  if group is not None else rank + 1, group))
        else:
            recv = None
    else:
        recv = None
    works = dist.batch_isend_irecv(ops) if ops else []
    return recv, works


class _StagedWork:
    """Completion handle of a host-staged exchange: wait() finishes the CPU
    P2P ops, then copies the received rows into the caller's device buffer."""

    def __init__(self, works, host_recv, recv):
        self._works, self._host_recv, self._recv = works, host_recv, recv

    def wait(self):
        for wk in self._works:
            wk.wait()
        if self._recv is not None:
            self._recv.copy_(self._host_recv)
            self._recv = None
        return True


def _exchange_halo_staged(x_local, halo, group, recv):
    """The same exchange for backends without device P2P (gloo): the halo
    rows travel through host memory; the band compute stays on the GPU."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if halo <= 0 or world <= 1:
        return None, []
    peer = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    ops, host_recv = [], None
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, x_local[:halo].to("cpu").contiguous(), peer(rank - 1),
                              group))
    if rank < world - 1:
        if recv is None:
            recv = torch.empty((halo,) + tuple(x_local.shape[1:]), dtype=x_local.dtype,
                               device=x_local.device)
        host_recv = torch.empty(tuple(recv.shape), dtype=recv.dtype)
        ops.append(dist.P2POp(dist.irecv, host_recv, peer(rank + 1), group))
    else:
        recv = None
    works = dist.batch_isend_irecv(ops) if ops else []
    return recv, [_StagedWork(works, host_recv, recv)]


def alloc_band(rows: int, w: int, kh: int, device=None):
    """A (rows + kh - 1, w) float32 buffer for one rank's band: fill
    [:rows] with the band, pass the whole buffer to
    conv2d_rowband(..., halo_in_place=True); the received halo lands in the
    spare rows, so the band is convolved by ONE launch (no boundary-strip
    launch and no concatenation)."""
    import torch
    return torch.empty((rows + kh - 1, w), dtype=torch.float32, device=device)


def conv2d_rowband(x_local, f, *, group=None, exact=None, conv=None, halo_in_place=False):
    """Distributed valid conv of a row-banded image: this rank's band in,
    this rank's output rows out (concatenating ranks gives the whole output).

    x_local: (rows_g, W) tensor on this rank's device, or with
    halo_in_place=True an alloc_band() buffer of rows_g + kh - 1 rows whose
    last kh - 1 rows are spare.  `conv` (x2d, f) -> y2d defaults to the
    sm_100a kernel; the CPU gloo tests inject the oracle.

    Default path: the interior rows are convolved while the halo is in flight
    (two launches: interior, then the 2(kh-1)-row boundary strip).  In-place
    path: the halo is received into the spare rows and the whole band is one
    launch after the wait -- the exchange (1.5 MiB per pair for config 5) is
    shorter than the boundary-strip launch and concatenation it replaces
    (~40 us per rank measured on B200)."""
    import torch
    f = as_filter2d(f)
    kh, kw = f.shape
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    halo = kh - 1
    last = rank == world - 1
    if halo_in_place:
        rows = int(x_local.shape[0]) - halo
        band = x_local[:rows]
    else:
        rows = int(x_local.shape[0])
        band = x_local
    w = int(x_local.shape[1])
    if rows < halo or (last and rows < kh) or rows < 1:
        raise ShapeError(f"band of {rows} rows too small for a {kh}x{kw} filter")
    n_out = rows if not last else rows - kh + 1
    s = ConvShape(rows + (0 if last else halo), w, kh, kw)
    if halo_in_place:
        recv, works = exchange_halo(band, halo, group, recv=x_local[rows:] if not last else None)
        for wk in works:
            wk.wait()
        src = x_local if not last else band
        if conv is None:
            from . import _ops
            y = torch.empty((n_out, w - kw + 1), dtype=torch.float32, device=x_local.device)
            _ops.conv2d_into(src, f, y, exact)
        else:
            y = conv(src, f)
        return y, CostCounters(macs=mac_count(s))
    recv, works = exchange_halo(band, halo, group)
    n_int = rows - kh + 1 if rows >= kh else 0   # interior output rows
    if conv is None:
        from . import _ops
        y = torch.empty((n_out, w - kw + 1), dtype=torch.float32, device=x_local.device)
        if n_int > 0:
            _ops.conv2d_into(band, f, y[:n_int], exact)      # overlaps the exchange
        for wk in works:
            wk.wait()
        if not last and halo > 0:
            edge = torch.cat([band[rows - halo:], recv], dim=0)
            _ops.conv2d_into(edge, f, y[n_int:], exact)
    else:
        parts = [conv(band, f)] if n_int > 0 else []
        for wk in works:
            wk.wait()
        if not last and halo > 0:
            edge = torch.cat([band[rows - halo:], recv], dim=0)  # 2*halo rows
            parts.append(conv(edge, f))
        y = torch.cat(parts, dim=0) if len(parts) > 1 else parts[0]
    return y, CostCounters(macs=mac_count(s))


class RowBandGroup:
    """Row bands on several GPUs of this process, one host thread, through
    the C ABI (include/slideconv_b200.h, sc_rowband_*): the context owns one
    NCCL communicator per device; each call exchanges the kh-1 halo rows with
    grouped ncclSend/ncclRecv on a comm stream while the interior rows are
    convolved, then runs the boundary rows (no copy, no concatenation).

        grp = RowBandGroup([0, 1, 2, 3])
        bufs = [alloc_band(rows, W, kh, device=f"cuda:{d}") ...]   # fill [:rows]
        ys = grp.conv2d(bufs, f)          # list of per-band outputs
    """

    def __init__(self, devices):
        import ctypes

        from . import _lib
        self._lib = _lib.load()
        self.devices = [int(d) for d in devices]
        arr = (ctypes.c_int * len(self.devices))(*self.devices)
        h = ctypes.c_void_p()
        _lib.check(self._lib.sc_rowband_create(len(self.devices), arr, ctypes.byref(h)))
        self._h = h

    def conv2d(self, bands, f, *, exact=None, timeout_ms: int = 120_000):
        """bands[g]: contiguous float32 CUDA tensor (rows_g + kh - 1, W) on
        devices[g], rows [:rows_g] filled; returns the per-band outputs
        (rows_g, W - kw + 1), the last band rows_g - kh + 1."""
        import ctypes

        import torch

        from . import _lib
        from ._device import mode_flag
        if self._h is None:
            raise RuntimeError("RowBandGroup is closed")
        f = as_filter2d(f)
        kh, kw = f.shape
        G = len(self.devices)
        if len(bands) != G:
            raise ValueError(f"expected {G} bands, got {len(bands)}")
        w = int(bands[0].shape[1])
        rows, ys = [], []
        for g, b in enumerate(bands):
            if (not b.is_cuda or b.device.index != self.devices[g] or b.dtype != torch.float32
                    or not b.is_contiguous() or int(b.shape[1]) != w):
                raise ValueError(f"band {g}: contiguous float32 CUDA tensor on cuda:"
                                 f"{self.devices[g]} with {w} columns required")
            r = int(b.shape[0]) - (kh - 1)
            rows.append(r)
            n_out = r if g < G - 1 else r - kh + 1
            ys.append(torch.empty((max(n_out, 0), w - kw + 1), dtype=torch.float32,
                                  device=b.device))
        vp = ctypes.c_void_p
        c_bands = (vp * G)(*[b.data_ptr() for b in bands])
        c_rows = (ctypes.c_int64 * G)(*rows)
        c_ys = (vp * G)(*[y.data_ptr() for y in ys])
        c_streams = (vp * G)(*[torch.cuda.current_stream(b.device).cuda_stream for b in bands])
        fc = np.ascontiguousarray(f, dtype=np.float32)
        _lib.check(self._lib.sc_rowband_conv2d_f32(self._h, c_bands, c_rows, w, fc.ctypes.data,
                                                   kh, kw, mode_flag(exact), c_ys, c_streams,
                                                   int(timeout_ms)))
        return ys

    def close(self):
        if self._h is not None:
            self._lib.sc_rowband_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover -- best effort
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
