"""Generate golden vectors from the REAL reference package (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes
  tests/golden/golden_small.npz   -- full arrays of the reference's known-answer
                                     and small seeded cases
  tests/golden/golden_hashes.json -- sha256 of the reference's output bytes for
                                     larger seeded cases, with the recipe that
                                     regenerates the inputs (numpy default_rng)

The inputs follow the reference tests' own recipes (file:line in each entry).
Nothing here is imported at run time; /root/reference is not on the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import slideconv as ref  # noqa: E402
from slideconv.kernels import analytic_counters  # noqa: E402

sys.path.insert(0, os.path.join(HERE, "..", ".."))
from tests.golden.recipes import RECIPES, make_inputs  # noqa: E402


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def run_ref(r, x, f):
    """Evaluate one recipe with the reference's public API."""
    op = r["op"]
    vm = ref.VectorModel(r.get("lanes", 16), "fast")
    if op == "conv2d_reference":
        return ref.conv2d_reference(x, f), None
    if op == "oracle_conv2d":
        return ref.oracle_conv2d(x, f), None
    if op == "conv1d_reference":
        return ref.conv1d_reference(x, f), None
    if op == "conv1d_slide":
        y, c = ref.conv1d_slide(x, f, vm)
        return y, c
    if op == "variant":
        y, c = ref.run_variant(ref.KernelVariant(r["variant"]), x, f, vm)
        return y, c
    if op == "conv1d_batch":      # 64-signal config: one conv1d_slide per signal
        ys = [ref.conv1d_slide(row, f, vm)[0][0] for row in x]
        return np.stack(ys), None
    if op == "conv2d_batch":      # batched images: one custom/generic call per image
        ys = [ref.run_variant(ref.select_kernel(f.shape[0], f.shape[1], vm), img, f, vm)[0]
              for img in x]
        return np.stack(ys), None
    if op in ("pool_sum", "pool_max"):
        fn = ref.sliding_window_sum if op == "pool_sum" else ref.sliding_window_max
        ys, st = [], None
        for row in np.atleast_2d(x):
            y, st = fn(row, r["k"])
            ys.append(y)
        return np.stack(ys), st
    if op == "pool_avg":          # avg = reference sum / float32(k)
        ys, st = [], None
        for row in np.atleast_2d(x):
            y, st = ref.sliding_window_sum(row, r["k"])
            ys.append(y / np.float32(r["k"]))
        return np.stack(ys), st
    if op == "im2col":
        return ref.conv2d_im2col(x, f), None
    if op == "accept1":           # every applicable fast variant agrees bit-for-bit
        from tests.golden.recipes import accept1_lanes
        v = accept1_lanes(r["t"])
        vm = ref.VectorModel(v, "fast")
        outs = [ref.run_variant(var, x, f, vm)[0]
                for var in ref.applicable_variants(f.shape[0], f.shape[1], vm)]
        assert all(np.array_equal(outs[0], o) for o in outs), "variants disagree"
        return outs[0], None
    raise ValueError(op)


def main():
    small = {}
    hashes = {}
    for name, r in RECIPES.items():
        x, f = make_inputs(r)
        y, extra = run_ref(r, x, f)
        entry = {"recipe": r, "sha256": sha(y), "shape": list(y.shape), "dtype": y.dtype.str}
        if isinstance(extra, int):
            entry["stages"] = extra
        elif extra is not None:
            entry["counters"] = [extra.macs, extra.slides, extra.loads, extra.im2col_elems]
        hashes[name] = entry
        if y.size <= 70_000:
            small[name] = y
    # analytic counter table over many shapes (kernels.py:100-120)
    table = []
    for lanes in (4, 8, 16, 32):
        vm = ref.VectorModel(lanes)
        for (h, w) in ((9, 11), (17, 23), (20, 33), (64, 64), (512, 512), (4096, 4096), (1, 1048576)):
            for k in (1, 2, 3, 5, 6, 7, 9, 17, 33):
                kh = 1 if h == 1 else k
                if kh > h or k > w:
                    continue
                s = ref.ConvShape(h, w, kh, k)
                for v in ref.KernelVariant:
                    c = analytic_counters(v, s, vm)
                    table.append([lanes, h, w, kh, k, v.value, c.macs, c.slides, c.loads, c.im2col_elems])
    hashes["__counters__"] = table
    # pooling stage counts k = 1..299 (pooling.py)
    stages = []
    for k in range(1, 300):
        _, s_sum = ref.sliding_window_sum(np.zeros(300, np.float32), k)
        _, s_max = ref.sliding_window_max(np.zeros(300, np.float32), k)
        stages.append([k, s_sum, s_max])
    hashes["__pool_stages__"] = stages
    # select_kernel table (kernels.py:78-94)
    sel = []
    for lanes in (4, 8, 16, 32):
        for kh in (1, 3, 5, 7):
            for kw in range(1, 3 * lanes):
                sel.append([lanes, kh, kw, ref.select_kernel(kh, kw, ref.VectorModel(lanes)).value])
    hashes["__select__"] = sel
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **small)
    with open(os.path.join(HERE, "golden_hashes.json"), "w") as fh:
        json.dump(hashes, fh, indent=0, sort_keys=True)
    print(f"{len(RECIPES)} recipes, {len(small)} stored in full")


if __name__ == "__main__":
    main()
