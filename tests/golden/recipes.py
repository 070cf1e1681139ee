"""Input recipes for the golden vectors (shared by make_golden.py and the tests).

Each recipe regenerates its inputs with numpy's default_rng exactly the way the
reference's own tests draw them (cited per entry), so the fixtures only need to
hold the reference's OUTPUTS (full arrays when small, sha256 otherwise).
"""

from __future__ import annotations

import numpy as np

RECIPES: dict[str, dict] = {}


def _add(name, **r):
    RECIPES[name] = r


# -- known-answer tests ------------------------------------------------------
_K9 = [[1, 2, 3], [4, 5, 6], [7, 8, 9]]
# test_reference.py:17-20, test_slide_kernels.py:98-101, test_gemm.py:85-88
_add("kat_ones2x2_ref", op="conv2d_reference", x=_K9, f=[[1, 1], [1, 1]])
_add("kat_ones2x2_generic", op="variant", variant="slide_generic", lanes=4, x=_K9, f=[[1, 1], [1, 1]])
_add("kat_ones2x2_compound", op="variant", variant="slide_compound", lanes=4, x=_K9, f=[[1, 1], [1, 1]])
_add("kat_ones2x2_im2col", op="im2col", x=_K9, f=[[1, 1], [1, 1]])
_add("kat_oracle_ones2x2", op="oracle_conv2d", x=_K9, f=[[1, 1], [1, 1]])
# test_reference.py:45-47, test_slide_kernels.py:75-77
_add("kat_conv1d_ones", op="conv1d_reference", x=[1, 2, 3, 4, 5], f=[1, 1, 1])
_add("kat_conv1d_slide_ones", op="conv1d_slide", lanes=4, x=[1, 2, 3, 4, 5], f=[1, 1, 1])
# test_slide_kernels.py:79-82
_add("kat_conv1d_single_tap", op="conv1d_slide", lanes=4, x="arange10", f=[1.0])
# test_slide_kernels.py:103-108 / :157-162 / verify.py:104-115 (delta-filter crops)
_add("kat_delta3_8x8", op="variant", variant="slide_generic", lanes=4, x="arange64_8x8", f="delta3")
_add("kat_delta5_12x12", op="variant", variant="custom5", lanes=4, x="arange144_12x12", f="delta5")
_add("kat_delta3_12x13_custom3", op="variant", variant="custom3", lanes=16, x="arange156_12x13", f="delta3")
_add("kat_delta5_12x13_compound", op="variant", variant="slide_compound", lanes=16, x="arange156_12x13", f="delta5")
# test_pooling.py:15-25, :45-49
_add("kat_pool_sum_1to5_k3", op="pool_sum", k=3, x=[1, 2, 3, 4, 5])
_add("kat_pool_sum_k1", op="pool_sum", k=1, x="arange8")
_add("kat_pool_max_31415_k3", op="pool_max", k=3, x=[3, 1, 4, 1, 5])
_add("kat_pool_max_31415_k1", op="pool_max", k=1, x=[3, 1, 4, 1, 5])
_add("kat_pool_sum_row_k4", op="pool_sum", k=4, x="arange10")

# -- seeded reference-test instances ------------------------------------------
# test_reference.py:30-34
_add("ref_64x64_5x5_s42", op="conv2d_reference", seed=42, dist="u11", xs=(64, 64), fs=(5, 5))
_add("oracle_64x64_5x5_s42", op="oracle_conv2d", seed=42, dist="u11", xs=(64, 64), fs=(5, 5))
# test_reference.py:50-54
_add("conv1d_1024_k11_s7", op="conv1d_reference", seed=7, dist="u11", xs=(1024,), fs=(11,))
# test_slide_kernels.py:84-90
_add("conv1d_slide_4096_k11_s17", op="conv1d_slide", lanes=16, seed=17, dist="u11", xs=(4096,), fs=(11,))
# test_slide_kernels.py:110-117 (generic, 31x29, seed lanes*10+k)
for _lanes in (4, 8):
    for _k in (1, 2, 3, 5, 7):
        if _k <= _lanes + 1:
            _add(f"generic_31x29_k{_k}_v{_lanes}", op="variant", variant="slide_generic", lanes=_lanes,
                 seed=_lanes * 10 + _k, dist="u11", xs=(31, 29), fs=(_k, _k))
# test_slide_kernels.py:130-134 (compound 40x41, seed k)
for _k in (6, 9, 13):
    _add(f"compound_40x41_k{_k}", op="variant", variant="slide_compound", lanes=4,
         seed=_k, dist="u11", xs=(40, 41), fs=(_k, _k))
# test_slide_kernels.py:148-155 (custom 40x40, seed 100+k)
_add("custom3_40x40", op="variant", variant="custom3", lanes=8, seed=103, dist="u11", xs=(40, 40), fs=(3, 3))
_add("custom5_40x40", op="variant", variant="custom5", lanes=8, seed=105, dist="u11", xs=(40, 40), fs=(5, 5))
_add("im2col_40x40_k5", op="im2col", seed=105, dist="u11", xs=(40, 40), fs=(5, 5))
# paper filter sizes (bench.py:20) through compound, 64x64
for _k in (11, 17, 29, 33, 51):
    _add(f"compound_64x64_k{_k}", op="variant", variant="slide_compound", lanes=16,
         seed=1000 + _k, dist="u11", xs=(64, 64), fs=(_k, _k))
# test_pooling.py:28-33
_add("pool_sum_4096_k13_s13", op="pool_sum", k=13, seed=13, dist="u11", xs=(4096,))
# test_pooling.py:36-42 (length 300, seed k)
for _k in (1, 2, 3, 4, 7, 15, 16, 31, 33, 64):
    _add(f"pool_sum_300_k{_k}", op="pool_sum", k=_k, seed=_k, dist="u11", xs=(300,))
# test_pooling.py:52-59 (max exact, seed 100+k)
for _k in (2, 3, 7, 8, 20, 64):
    _add(f"pool_max_4096_k{_k}", op="pool_max", k=_k, seed=100 + _k, dist="u11", xs=(4096,))
# test_acceptance.py:134-152 (criterion 6: 4096, seed 6, k = 1..64)
for _k in range(1, 65):
    _add(f"accept6_sum_k{_k}", op="pool_sum", k=_k, seed=6, dist="u11", xs=(4096,))
    _add(f"accept6_max_k{_k}", op="pool_max", k=_k, seed=6, dist="u11", xs=(4096,))
# wide windows beyond the reference tests (doubling + combine of many bits)
for _k in (100, 127, 128, 129, 255, 256, 511, 1000):
    _add(f"pool_sum_8192_k{_k}", op="pool_sum", k=_k, seed=7000 + _k, dist="n01", xs=(8192,))
    _add(f"pool_max_8192_k{_k}", op="pool_max", k=_k, seed=7000 + _k, dist="n01", xs=(8192,))

# -- BASELINE.json config-shaped samples (reference applied per unit) ----------
# cfg2: 256 x 262,144 N(0,1), k = 16 (+3, 64, 255): a 4-signal sample
for _k in (3, 16, 64, 255):
    for _op in ("pool_sum", "pool_max", "pool_avg"):
        _add(f"cfg2_{_op}_k{_k}", op=_op, k=_k, seed=0x5EED2, dist="n01", xs=(4, 262144))
# cfg1: 64 x 1,048,576 U[-1,1], k = 7, w N(0,1): a 2-signal sample
_add("cfg1_conv1d_k7", op="conv1d_batch", lanes=16, seed=0x5EED1, dist="u11", fdist="n01",
     xs=(2, 1048576), fs=(1, 7))
# cfg3: 4096^2 U[0,1], 3x3 / 5x5 N(0,1/k^2): one image each
_add("cfg3_conv2d_3x3", op="conv2d_batch", lanes=16, seed=0x5EED3, dist="u01", fdist="n_k2",
     xs=(1, 4096, 4096), fs=(3, 3))
_add("cfg3_conv2d_5x5", op="conv2d_batch", lanes=16, seed=0x5EED35, dist="u01", fdist="n_k2",
     xs=(1, 4096, 4096), fs=(5, 5))
# cfg5: 65536^2 7x7 -> a 518-row x 8192-col band (band == whole image)
_add("cfg5_band_7x7", op="variant", variant="slide_generic", lanes=16, seed=0x5EED5, dist="u11",
     fdist="n_k2", xs=(518, 8192), fs=(7, 7))

# -- acceptance criterion 1 stream (test_acceptance.py:42-67), first 150 instances
for _t in range(150):
    _add(f"accept1_t{_t:03d}", op="accept1", t=_t)


_NAMED = {
    "arange10": lambda: np.arange(10, dtype=np.float32),
    "arange8": lambda: np.arange(8, dtype=np.float32),
    "arange64_8x8": lambda: np.arange(64, dtype=np.float32).reshape(8, 8),
    "arange144_12x12": lambda: np.arange(144, dtype=np.float32).reshape(12, 12),
    "arange156_12x13": lambda: np.arange(156, dtype=np.float32).reshape(12, 13),
}


def _delta(k):
    f = np.zeros((k, k), dtype=np.float32)
    f[k // 2, k // 2] = 1.0
    return f


def _draw(rng, dist, shape, k=None):
    if dist == "u11":
        return rng.uniform(-1, 1, shape).astype(np.float32)
    if dist == "u01":
        return rng.uniform(0, 1, shape).astype(np.float32)
    if dist == "n01":
        return rng.standard_normal(shape, dtype=np.float32)
    if dist == "n_k2":       # N(0, 1/k^2): std 1/k with k = filter width
        return (rng.standard_normal(shape, dtype=np.float32) / np.float32(shape[-1])).astype(np.float32)
    raise ValueError(dist)


_ACCEPT_CACHE: list = []


def _accept1(t):
    """Replay test_acceptance.py:43-55's stream up to instance t."""
    if not _ACCEPT_CACHE:
        rng = np.random.default_rng(2026)
        for i in range(150):
            v = (4, 8, 16)[i % 3]
            k = int(rng.integers(1, v + 10))
            h = int(rng.integers(k, 129))
            w = int(rng.integers(k, 129))
            x = rng.uniform(-1, 1, (h, w)).astype(np.float32)
            f = rng.uniform(-1, 1, (k, k)).astype(np.float32)
            _ACCEPT_CACHE.append((v, x, f))
    return _ACCEPT_CACHE[t]


def make_inputs(r):
    """Return (x, f) as float32 numpy arrays (f may be None for pooling)."""
    if r["op"] == "accept1":
        _, x, f = _accept1(r["t"])
        return x, f
    if "seed" not in r:
        x = r["x"]
        x = _NAMED[x]() if isinstance(x, str) else np.asarray(x, dtype=np.float32)
        f = r.get("f")
        if isinstance(f, str):
            f = _delta(int(f[-1]))
        elif f is not None:
            f = np.asarray(f, dtype=np.float32)
        return x, f
    rng = np.random.default_rng(r["seed"])
    x = _draw(rng, r["dist"], tuple(r["xs"]))
    f = None
    if "fs" in r:
        f = _draw(rng, r.get("fdist", r["dist"]), tuple(r["fs"]))
    return x, f


def accept1_lanes(t):
    return _accept1(t)[0]
