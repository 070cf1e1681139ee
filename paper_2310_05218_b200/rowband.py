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


def exchange_halo(x_local, halo: int, group=None):
    """Post the halo exchange for this rank's band; returns (recv_buf, works).

    Sends x_local[:halo] to rank-1 and receives `halo` rows from rank+1 with
    one batched NCCL (or gloo) P2P group.  Caller waits on `works` before
    touching recv_buf."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ops = []
    recv = None
    if halo > 0 and world > 1:
        if rank > 0:
            send = x_local[:halo].contiguous()
            ops.append(dist.P2POp(dist.isend, send, dist.get_global_rank(group, rank - 1)
                                  if group is not None else rank - 1, group))
        if rank < world - 1:
            recv = torch.empty((halo,) + tuple(x_local.shape[1:]), dtype=x_local.dtype,
                               device=x_local.device)
            ops.append(dist.P2POp(dist.irecv, recv, dist.get_global_rank(group, rank + 1)
                                  if group is not None else rank + 1, group))
    works = dist.batch_isend_irecv(ops) if ops else []
    return recv, works


def conv2d_rowband(x_local, f, *, group=None, exact=None, conv=None):
    """Distributed valid conv of a row-banded image: this rank's band in,
    this rank's output rows out (concatenating ranks gives the whole output).

    x_local: (rows_g, W) tensor on this rank's device.  `conv` (x2d, f) -> y2d
    defaults to the sm_100a kernel; the CPU gloo tests inject the oracle."""
    import torch
    import torch.distributed as dist
    f = as_filter2d(f)
    kh, kw = f.shape
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    halo = kh - 1
    rows, w = int(x_local.shape[0]), int(x_local.shape[1])
    last = rank == world - 1
    if rows < halo or (last and rows < kh):
        raise ShapeError(f"band of {rows} rows too small for a {kh}x{kw} filter")
    recv, works = exchange_halo(x_local, halo, group)
    n_int = rows - kh + 1 if rows >= kh else 0   # interior output rows
    n_out = rows if not last else rows - kh + 1
    if conv is None:
        from . import _ops
        y = torch.empty((n_out, w - kw + 1), dtype=torch.float32, device=x_local.device)
        if n_int > 0:
            _ops.conv2d_into(x_local, f, y[:n_int], exact)      # overlaps the exchange
        for wk in works:
            wk.wait()
        if not last and halo > 0:
            edge = torch.cat([x_local[rows - halo:], recv], dim=0)
            _ops.conv2d_into(edge, f, y[n_int:], exact)
    else:
        parts = [conv(x_local, f)] if n_int > 0 else []
        for wk in works:
            wk.wait()
        if not last and halo > 0:
            edge = torch.cat([x_local[rows - halo:], recv], dim=0)  # 2*halo rows
            parts.append(conv(edge, f))
        y = torch.cat(parts, dim=0) if len(parts) > 1 else parts[0]
    s = ConvShape(rows + (0 if last else halo), w, kh, kw)
    return y, CostCounters(macs=mac_count(s))
