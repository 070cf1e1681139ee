"""Multi-core CPU timing of the oracle -- TEST / BENCH INFRASTRUCTURE ONLY.

Used by bench.py's cpu_baseline leg and its `--impl reference` arm: the
reference's own algorithm (restated in oracle/slideconv_oracle.py, which is
pinned bit-for-bit to the reference's outputs) timed on the host's cores.
Methodology follows the reference benchmark (pkg/src/slideconv/bench.py:71-78,
:105-112): one process per core, each pinned to its core (the reference pins
itself to a single core); work is sharded by unit (signal / image / band);
inputs are generated inside the workers BEFORE a barrier, so generation is
excluded from the timed region; wall time = last finish - first start.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from oracle import slideconv_oracle as O


def host_cores() -> list[int]:
    try:
        return sorted(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return list(range(os.cpu_count() or 1))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --------------------------------------------------------------------- tasks
# task = (kind, params); unit = integer index -> (inputs, bytes, flops)

def _gen(kind, p, unit):
    rng = np.random.default_rng([0x5EED, p["cfg"], unit])
    if kind == "pool":
        return (rng.standard_normal(p["n"], dtype=np.float32),)
    if kind == "conv1d":
        return (rng.uniform(-1, 1, (1, p["n"])).astype(np.float32),)
    if kind == "conv2d":
        lo = p.get("lo", 0.0)
        return (rng.uniform(lo, 1, (p["h"], p["w"])).astype(np.float32),)
    if kind == "nchw":
        return (rng.standard_normal((1, p["cin"], p["h"], p["w"]), dtype=np.float32),)
    raise ValueError(kind)


def _weights(kind, p):
    rng = np.random.default_rng([0x5EED, p["cfg"], 0xFFFF])
    if kind == "conv1d":
        return rng.standard_normal((1, p["k"]), dtype=np.float32)
    if kind == "conv2d":
        k = p["k"]
        return (rng.standard_normal((k, k), dtype=np.float32) / np.float32(k)).astype(np.float32)
    if kind == "nchw":
        return (rng.standard_normal((p["cout"], p["cin"], 3, 3), dtype=np.float32)
                / np.float32(np.sqrt(9 * p["cin"]))).astype(np.float32)
    return None


def _compute(kind, p, inputs, w):
    """One unit of the reference's work, as the reference would be called."""
    if kind == "pool":
        (x,) = inputs
        for op in p["ops"]:
            {"sum": O.sliding_window_sum, "max": O.sliding_window_max,
             "avg": O.sliding_window_mean}[op](x, p["k"])
        return
    if kind in ("conv1d", "conv2d"):
        O.conv2d(inputs[0], w)
        return
    if kind == "nchw":
        O.conv2d_nchw(inputs[0], w, 1)
        return


def _worker(core, kind, p, units, barrier, q):
    try:
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        pass
    w = _weights(kind, p)
    data = [_gen(kind, p, u) for u in units]
    barrier.wait()
    t0 = time.perf_counter()
    for inp in data:
        _compute(kind, p, inp, w)
    t1 = time.perf_counter()
    q.put((t0, t1, len(units)))


def time_units(kind: str, p: dict, n_units: int, workers: int | None = None) -> dict:
    """Run n_units of the task across `workers` pinned processes; return
    {'seconds': wall, 'units': n_units, 'cores': workers}."""
    cores = host_cores()
    workers = max(1, min(workers or len(cores), n_units))
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(workers)
    q = ctx.Queue()
    shards = [list(range(i, n_units, workers)) for i in range(workers)]
    procs = [ctx.Process(target=_worker, args=(cores[i % len(cores)], kind, p, shards[i], barrier, q))
             for i in range(workers)]
    for pr in procs:
        pr.start()
    res = [q.get() for _ in procs]
    for pr in procs:
        pr.join()
    t0 = min(r[0] for r in res)
    t1 = max(r[1] for r in res)
    return {"seconds": t1 - t0, "units": n_units, "cores": workers}


def time_one_core(kind: str, p: dict, n_units: int) -> float:
    """In-process single-core timing (the reference's own methodology)."""
    w = _weights(kind, p)
    data = [_gen(kind, p, u) for u in range(n_units)]
    t0 = time.perf_counter()
    for inp in data:
        _compute(kind, p, inp, w)
    return time.perf_counter() - t0
