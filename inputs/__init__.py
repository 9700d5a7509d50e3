"""Seeded synthetic-input definitions shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no edge hash, no threshold
quantisation, no connectivity, no greedy).  It only states *what* input each
workload is: generator kind, sizes, the integer quadrant thresholds of the
R-MAT sampler, the probability model and the (R, k, hash_seed, alpha)
parameters taken from BASELINE.json `configs[0..4]`.  Both `oracle/` (its own
C generator) and the CUDA generator consume these numbers; neither imports the
other.

It also offers tiny numpy graph builders (path, star, random simple graphs)
used by the tests to feed both sides identical CSR arrays.
"""
from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# Generator parameters
# ---------------------------------------------------------------------------

GEN_ER, GEN_RMAT, GEN_GRID = 0, 1, 2
P_CONST, P_WIC, P_UNIFORM = 0, 1, 2  # P_UNIFORM: p ~ U(lo, hi), cfg['p_range'] (R19)


def rmat_thresholds(a: float, b: float, c: float) -> tuple[int, int, int]:
    """Integer quadrant thresholds for a 53-bit uniform draw: a | a+b | a+b+c.

    Computed once here (IEEE double, floor) so both generators compare against
    the same integers.
    """
    s = float(1 << 53)
    return (int(np.floor(a * s)), int(np.floor((a + b) * s)),
            int(np.floor((a + b + c) * s)))


def diag_threshold(pdiag: float) -> int:
    return int(np.floor(pdiag * 4294967296.0))


CONFIGS = {
    # BASELINE.json configs[0]: tiny ER parity graph
    "c1": dict(name="tiny-er", gen=GEN_ER, n=4096, m=32768, gen_seed=1,
               pmodel=P_CONST, p=0.05, R=64, k=8, hash_seed=1, alpha=None),
    # configs[1]: social-shaped R-MAT scale 22, ef 16 (the N=1 bench workload)
    "c2": dict(name="social-rmat-s22", gen=GEN_RMAT, scale=22, ef=16,
               abc=(0.57, 0.19, 0.19), permute=1, gen_seed=1,
               pmodel=P_CONST, p=0.02, R=256, k=100, hash_seed=1, alpha=None),
    # configs[2]: 4096x4096 grid + random diagonals
    "c3": dict(name="road-grid-4096", gen=GEN_GRID, W=4096, H=4096, pdiag=0.3,
               gen_seed=1, pmodel=P_CONST, p=0.5, R=256, k=50, hash_seed=1,
               alpha=None),
    # configs[3]: twitter-shaped R-MAT scale 26, ef 24, WIC probabilities
    "c4": dict(name="twitter-rmat-s26-wic", gen=GEN_RMAT, scale=26, ef=24,
               abc=(0.57, 0.19, 0.19), permute=1, gen_seed=1,
               pmodel=P_WIC, p=None, R=256, k=100, hash_seed=1, alpha=None),
    # configs[4]: web-shaped R-MAT scale 28, ef 32, compressed (alpha=1/16)
    "c5": dict(name="web-rmat-s28-compressed", gen=GEN_RMAT, scale=28, ef=32,
               abc=(0.6, 0.15, 0.15), permute=1, gen_seed=1,
               pmodel=P_CONST, p=0.01, R=256, k=100, hash_seed=1,
               alpha=1.0 / 16),
}


def config(name: str, **over) -> dict:
    c = dict(CONFIGS[name])
    c.update(over)
    if c["gen"] == GEN_RMAT:
        c["n"] = 1 << c["scale"]
        c["rmat_t"] = rmat_thresholds(*c["abc"])
    if c["gen"] == GEN_GRID:
        c["n"] = c["W"] * c["H"]
        c["diag_t"] = diag_threshold(c["pdiag"])
    return c


# ---------------------------------------------------------------------------
# Tiny CSR builders for tests (numpy only)
# ---------------------------------------------------------------------------

def csr_from_edges(n: int, edges) -> tuple[np.ndarray, np.ndarray]:
    """Symmetric simple CSR (sorted lists, no loops, no duplicates)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if len(e):
        e = e[e[:, 0] != e[:, 1]]
        lo = np.minimum(e[:, 0], e[:, 1])
        hi = np.maximum(e[:, 0], e[:, 1])
        key = np.unique(lo * (1 << 32) + hi)
        lo, hi = key >> 32, key & 0xFFFFFFFF
        src = np.concatenate([lo, hi])
        dst = np.concatenate([hi, lo])
        order = np.lexsort((dst, src))
        src, dst = src[order], dst[order]
    else:
        src = dst = np.zeros(0, np.int64)
    off = np.zeros(n + 1, np.uint64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off).astype(np.uint64)
    return off, dst.astype(np.uint32)


def path_graph(L: int):
    return csr_from_edges(L, [(i, i + 1) for i in range(L - 1)])


def star_graph(d: int, center: int = 0):
    leaves = [v for v in range(d + 1) if v != center]
    return csr_from_edges(d + 1, [(center, v) for v in leaves])


def random_graph(n: int, m: int, seed: int):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, size=4 * m + 8)
    v = rng.integers(0, n, size=4 * m + 8)
    keep = u != v
    pairs = np.stack([np.minimum(u, v), np.maximum(u, v)], 1)[keep]
    _, idx = np.unique(pairs[:, 0] * n + pairs[:, 1], return_index=True)
    pairs = pairs[np.sort(idx)][:m]
    return csr_from_edges(n, pairs)


def random_powerlaw_graph(n: int, m: int, seed: int, skew: float = 1.5):
    """Heavy-tailed degrees (Zipf-like endpoint choice) with isolated vertices."""
    rng = np.random.default_rng(seed)
    w = 1.0 / np.arange(1, n + 1) ** (1.0 / skew)
    w /= w.sum()
    perm = rng.permutation(n)
    u = perm[rng.choice(n, size=4 * m + 8, p=w)]
    v = perm[rng.choice(n, size=4 * m + 8, p=w)]
    keep = u != v
    pairs = np.stack([np.minimum(u, v), np.maximum(u, v)], 1)[keep]
    _, idx = np.unique(pairs[:, 0] * n + pairs[:, 1], return_index=True)
    pairs = pairs[np.sort(idx)][:m]
    return csr_from_edges(n, pairs)
