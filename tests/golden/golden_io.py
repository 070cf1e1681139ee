"""Load the committed golden fixtures and evaluate recipes with the CPU oracle."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle import slideconv_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden_hashes.json")) as _fh:
    GOLD = json.load(_fh)
_npz = np.load(os.path.join(HERE, "golden_small.npz"))
SMALL = {k: _npz[k] for k in _npz.files}


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def oracle_eval(r, x, f):
    """The oracle's answer for one recipe: (y, stages | counters | None)."""
    op = r["op"]
    lanes = r.get("lanes", 16)
    if op in ("conv2d_reference", "accept1"):
        return O.conv2d(x, f), None
    if op == "oracle_conv2d":
        return O.oracle_conv2d(x, f), None
    if op == "conv1d_reference":
        return O.conv2d(x, f), None
    if op in ("conv1d_slide", "variant"):
        xx = np.atleast_2d(np.asarray(x, np.float32))
        ff = np.atleast_2d(np.asarray(f, np.float32))
        variant = r.get("variant", "slide_generic")
        c = O.analytic_counters(variant, xx.shape[0], xx.shape[1], ff.shape[0], ff.shape[1], lanes)
        return O.conv2d(xx, ff), c
    if op == "conv1d_batch":
        return O.conv2d_batched(x[:, None, :], f)[:, 0, :], None
    if op == "conv2d_batch":
        return O.conv2d_batched(x, f), None
    if op in ("pool_sum", "pool_max", "pool_avg"):
        kind = op[5:]
        k = r["k"]
        y = O.pool_batched(np.atleast_2d(x), k, kind)
        st = O.pool_max_stages(k) if kind == "max" else O.pool_sum_stages(k)
        return y, st
    if op == "im2col":
        return O.conv2d_im2col(x, f), None
    raise ValueError(op)
