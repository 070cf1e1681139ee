"""Multi-core CPU timing of the oracle -- TEST / BENCH INFRASTRUCTURE ONLY.

Used by bench.py's cpu_baseline leg and its `--impl reference` arm: the
reference's own algorithm (restated in oracle/slideconv_oracle.py, which is
pinned bit-for-bit to the reference's outputs) timed on the host's cores.
Methodology follows the reference benchmark (pkg/src/slideconv/bench.py:71-78,
:105-112): one process per core, each pinned to its core (the reference pins
itself to a single core); work is sharded by unit (signal / image / band);
inputs are generated inside the workers BEFORE a barrier, so generation is
excluded from the timed region; wall time = last finish - first start.

The worker processes are PERSISTENT (`CpuPool`): started once, pinned once,
inputs generated once per task and kept; every timed step is then a barrier
plus the compute, so consecutive steps measure the same thing (round 1 spawned
fresh processes every step, and two arms of the same run disagreed by 2x).
"""

from __future__ import annotations

import atexit
import multiprocessing as mp
import os
import statistics
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
# task = (kind, params); unit = integer index -> inputs

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


def _task_key(kind, p, units):
    return (kind, tuple(sorted((k, tuple(v) if isinstance(v, (list, tuple)) else v)
                               for k, v in p.items())), tuple(units))


def _pool_worker(core, conn, barrier):
    try:
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        pass
    cache = {}
    while True:
        msg = conn.recv()
        if msg[0] == "stop":
            return
        _, kind, p, units = msg
        key = _task_key(kind, p, units)
        if key not in cache:
            cache.clear()                      # one task's inputs resident at a time
            cache[key] = (_weights(kind, p), [_gen(kind, p, u) for u in units])
        w, data = cache[key]
        conn.send("ready")
        barrier.wait()
        t0 = time.perf_counter()
        for inp in data:
            _compute(kind, p, inp, w)
        t1 = time.perf_counter()
        conn.send((t0, t1, len(units)))


class CpuPool:
    """One pinned process per host core, started once."""

    def __init__(self, workers: int | None = None):
        cores = host_cores()
        self.workers = max(1, min(workers or len(cores), len(cores)))
        ctx = mp.get_context("spawn")
        self._barrier = ctx.Barrier(self.workers)
        self._conns, self._procs = [], []
        for i in range(self.workers):
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_pool_worker, args=(cores[i], b, self._barrier), daemon=True)
            pr.start()
            self._conns.append(a)
            self._procs.append(pr)

    def run(self, kind: str, p: dict, n_units: int) -> dict:
        """Time n_units of the task sharded over all workers (every worker
        joins the barrier, idle ones with no units)."""
        shards = [list(range(i, n_units, self.workers)) for i in range(self.workers)]
        for c, s in zip(self._conns, shards):
            c.send(("run", kind, p, s))
        for c in self._conns:
            assert c.recv() == "ready"
        res = [c.recv() for c in self._conns]
        busy = [r for r in res if r[2] > 0]
        t0 = min(r[0] for r in busy)
        t1 = max(r[1] for r in busy)
        return {"seconds": t1 - t0, "units": n_units, "cores": len(busy)}

    def close(self):
        for c in self._conns:
            try:
                c.send(("stop",))
            except (OSError, BrokenPipeError):
                pass
        for pr in self._procs:
            pr.join(timeout=10)


_POOL: CpuPool | None = None


def get_pool() -> CpuPool:
    global _POOL
    if _POOL is None:
        _POOL = CpuPool()
        atexit.register(_POOL.close)
    return _POOL


def time_units(kind: str, p: dict, n_units: int, workers: int | None = None) -> dict:
    """One timed run of n_units across the persistent pinned pool (`workers`
    is accepted for compatibility; the pool always uses every host core)."""
    return get_pool().run(kind, p, n_units)


def time_steps(kind: str, p: dict, n_units: int, steps: int, warmup: int = 1) -> dict:
    """The estimator both bench arms use: median over `steps` timed runs
    after `warmup` untimed ones, on the persistent pool."""
    pool = get_pool()
    for _ in range(warmup):
        pool.run(kind, p, n_units)
    secs = [pool.run(kind, p, n_units)["seconds"] for _ in range(steps)]
    return {"seconds": statistics.median(secs), "all": secs, "units": n_units,
            "cores": pool.workers}


def time_one_core(kind: str, p: dict, n_units: int) -> float:
    """In-process single-core timing (the reference's own methodology)."""
    w = _weights(kind, p)
    data = [_gen(kind, p, u) for u in range(n_units)]
    t0 = time.perf_counter()
    for inp in data:
        _compute(kind, p, inp, w)
    return time.perf_counter() - t0
