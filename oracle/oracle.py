"""ctypes wrapper of the C oracle (oracle/pacim_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference leg of bench.py.  The product path
(paper_2311_07554_b200/) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "pacim_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

UNSET = 0xFFFFFFFF


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (single-threaded, no intrinsics)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC",
                               "-o", LIB, SRC, "-lm", "-pthread"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u64, u32, i64, dbl, i32 = C.c_uint64, C.c_uint32, C.c_int64, C.c_double, C.c_int
        P = C.c_void_p
        sig = {
            "orc_mix64": (u64, [u64]),
            "orc_hash_r": (u64, [u64, u32]),
            "orc_hash_e": (u64, [u64, u32, u32]),
            "orc_hash_edge": (u64, [u64, u32, u32, u32]),
            "orc_t32_const": (u64, [dbl]),
            "orc_t32_wic": (u64, [u64, u64]),
            "orc_t32_uniform": (u64, [u64, u32, u32]),
            "orc_live_decor": (i32, [u64, u32, u32, u32, u64]),
            "orc_simulate_ic": (u64, [u32, P, P, i32, u64, P, u32, u32, u64]),
            "orc_live": (i32, [u64, u32, u32, u32, u64]),
            "orc_sketch_labels": (C.c_long, [u32, P, P, i32, u64, u64, u32, P, P]),
            "orc_greedy": (i32, [u32, P, P, i32, u64, u32, u64, u32, P, P, P, P]),
            "orc_verify": (i32, [u32, P, P, i32, u64, u32, u64, u32, P, P, i32, P]),
            "orc_is_center": (i32, [u64, u32, u64]),
            "orc_centers": (u32, [u32, u64, u64, P, P]),
            "orc_compressed_sketch": (i32, [u32, P, P, i32, u64, u64, u32, u64, P, P]),
            "orc_get_center": (None, [u32, P, P, i32, u64, u64, u32, P, P, P, P, u32,
                                      P, P, P]),
            "orc_greedy_alg3": (i32, [u32, P, P, i32, u64, u32, u64, u64, u32, P, P, P, P]),
            "orc_gen_er": (C.c_long, [u32, u64, u64, P]),
            "orc_gen_rmat": (C.c_long, [i32, u32, u64, u64, u64, i32, u64, P]),
            "orc_gen_grid": (C.c_long, [u32, u32, u64, u64, P]),
            "orc_csr_from_keys": (None, [u32, u64, P, P, P]),
            "orc_gen_rmat_csr_mt": (C.c_long, [i32, u32, u64, u64, u64, i32, u64, i32, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- hash / T32
def mix64(z: int) -> int:
    return lib().orc_mix64(z)


def hash_edge(seed: int, u: int, v: int, r: int) -> int:
    return lib().orc_hash_edge(seed, u, v, r)


def t32_const(p: float) -> int:
    return lib().orc_t32_const(p)


def t32_wic(du: int, dv: int) -> int:
    return lib().orc_t32_wic(du, dv)


def uniform_param(lo: float, hi: float) -> int:
    """R19: the Uniform model's packed parameter H << 32 | L (IEEE double floors)."""
    L = t32_const(lo)
    H = min(t32_const(hi), (1 << 32) - 1)
    L = min(L, H)
    return (H << 32) | L


def t32_uniform(packed: int, u: int, v: int) -> int:
    return lib().orc_t32_uniform(packed, u, v)


def hash_r(seed: int, r: int) -> int:
    return int(lib().orc_hash_r(seed, r))


def live(seed: int, u: int, v: int, r: int, t32: int) -> bool:
    return bool(lib().orc_live(seed, u, v, r, t32))


# ------------------------------------------------------------------ graphs
class Graph:
    """Host CSR (off u64[n+1], nbr u32[2m]) plus the sorted upper key list."""

    def __init__(self, n, off, nbr, keys=None):
        self.n = int(n)
        self.off = np.ascontiguousarray(off, dtype=np.uint64)
        self.nbr = np.ascontiguousarray(nbr, dtype=np.uint32)
        self.keys = keys

    @property
    def m(self):
        return int(self.off[-1]) // 2


def csr_from_keys(n: int, keys: np.ndarray) -> Graph:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    m = len(keys)
    off = np.zeros(n + 1, np.uint64)
    nbr = np.zeros(2 * m, np.uint32)
    lib().orc_csr_from_keys(n, m, _p(keys), _p(off), _p(nbr))
    return Graph(n, off, nbr, keys)


def gen_er(n: int, m: int, gen_seed: int) -> Graph:
    keys = np.zeros(m, np.uint64)
    got = lib().orc_gen_er(n, m, gen_seed, _p(keys))
    if got < 0:
        raise ValueError("orc_gen_er failed")
    return csr_from_keys(n, keys)


def gen_rmat(scale: int, ef: int, thr, permute: int, gen_seed: int) -> Graph:
    keys = np.zeros(ef << scale, np.uint64)
    m = lib().orc_gen_rmat(scale, ef, thr[0], thr[1], thr[2], permute, gen_seed, _p(keys))
    keys = keys[:m].copy()
    return csr_from_keys(1 << scale, keys)


def gen_rmat_mt(scale: int, ef: int, thr, permute: int, gen_seed: int,
                threads: int | None = None) -> Graph:
    """Threaded copy of gen_rmat (same CSR bit for bit; input side only)."""
    threads = threads or os.cpu_count() or 1
    cap = ef << scale
    keys = np.empty(cap, np.uint64)
    tmp = np.empty(cap, np.uint64)
    n = 1 << scale
    off = np.empty(n + 1, np.uint64)
    # the CSR has 2m entries, m <= cap: sized after the call from off[n]
    nbr = np.empty(2 * cap, np.uint32)
    m = lib().orc_gen_rmat_csr_mt(scale, ef, thr[0], thr[1], thr[2], permute, gen_seed, threads,
                                  _p(keys), _p(tmp), _p(off), _p(nbr))
    if m < 0:
        raise MemoryError("orc_gen_rmat_csr_mt")
    del tmp
    return Graph(n, off, nbr[:2 * m].copy(), keys[:m].copy())


def gen_grid(W: int, H: int, d32: int, gen_seed: int) -> Graph:
    keys = np.zeros(3 * W * H, np.uint64)
    m = lib().orc_gen_grid(W, H, d32, gen_seed, _p(keys))
    keys = keys[:m].copy()
    return csr_from_keys(W * H, keys)


def gen_config(cfg: dict, threads: int | None = None) -> Graph:
    """threads > 1: the threaded R-MAT generator (identical output)."""
    from inputs import GEN_ER, GEN_RMAT, GEN_GRID
    if cfg["gen"] == GEN_RMAT and threads and threads > 1:
        return gen_rmat_mt(cfg["scale"], cfg["ef"], cfg["rmat_t"], cfg["permute"], cfg["gen_seed"],
                           threads)
    if cfg["gen"] == GEN_ER:
        return gen_er(cfg["n"], cfg["m"], cfg["gen_seed"])
    if cfg["gen"] == GEN_RMAT:
        return gen_rmat(cfg["scale"], cfg["ef"], cfg["rmat_t"], cfg["permute"], cfg["gen_seed"])
    if cfg["gen"] == GEN_GRID:
        return gen_grid(cfg["W"], cfg["H"], cfg["diag_t"], cfg["gen_seed"])
    raise ValueError(cfg["gen"])


def model_args(cfg: dict):
    """(model, t32) for a config: the oracle quantises p itself."""
    if cfg["pmodel"] == 1:
        return 1, 0
    if cfg["pmodel"] == 2:
        return 2, uniform_param(*cfg["p_range"])
    return 0, t32_const(cfg["p"])


# ---------------------------------------------------------------- sketches
def sketch_labels(g: Graph, model: int, t32: int, seed: int, r: int):
    label = np.zeros(g.n, np.uint32)
    size = np.zeros(g.n, np.uint32)
    ncc = lib().orc_sketch_labels(g.n, _p(g.off), _p(g.nbr), model, t32, seed, r,
                                  _p(label), _p(size))
    if ncc < 0:
        raise MemoryError
    return label, size


def greedy(g: Graph, model: int, t32: int, R: int, seed: int, k: int, want_gain0=False):
    seeds = np.zeros(k, np.uint32)
    gain = np.zeros(k, np.int64)
    sigma = np.zeros(k, np.int64)
    gain0 = np.zeros(g.n, np.int64) if want_gain0 else None
    rc = lib().orc_greedy(g.n, _p(g.off), _p(g.nbr), model, t32, R, seed, k,
                          _p(seeds), _p(gain), _p(sigma),
                          _p(gain0) if gain0 is not None else None)
    if rc != 0:
        raise RuntimeError(f"orc_greedy rc={rc}")
    return seeds, gain, sigma, gain0


VERIFY_RC = {0: "certified", 1: "claimed gain differs from the oracle's gain of the claimed seed",
             2: "another vertex beats the claimed seed (gain desc, id asc)",
             3: "claimed seed repeats or is out of range", -1: "out of memory"}


def verify(g: Graph, model: int, t32: int, R: int, seed: int, seeds, gain_num,
           threads: int | None = None):
    """Verify mode: certify a claimed greedy sequence.  Returns
    (rc, info): rc 0 = the sequence is exactly derive mode's; info = (step,
    oracle argmax, its gain, claimed seed's true gain) at the first failure,
    (k, 0, 0, covered entries) on success."""
    s = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint32))
    gn = np.ascontiguousarray(np.asarray(gain_num, dtype=np.int64))
    assert len(s) == len(gn)
    info = np.zeros(4, np.int64)
    if threads is None:
        threads = os.cpu_count() or 1
    rc = lib().orc_verify(g.n, _p(g.off), _p(g.nbr), model, t32, R, seed, len(s), _p(s), _p(gn),
                          int(threads), _p(info))
    return int(rc), tuple(int(x) for x in info)


def centers(n: int, seed: int, a32: int):
    center_of = np.zeros(n, np.uint32)
    cs = np.zeros(n, np.uint32)
    rho = lib().orc_centers(n, seed, a32, _p(cs), _p(center_of))
    return cs[:rho].copy(), center_of


def compressed_sketch(g: Graph, model, t32, seed, r, a32):
    cs, _ = centers(g.n, seed, a32)
    rho = len(cs)
    lab = np.zeros(max(rho, 1), np.uint32)
    sz = np.zeros(max(rho, 1), np.uint32)
    lib().orc_compressed_sketch(g.n, _p(g.off), _p(g.nbr), model, t32, seed, r, a32,
                                _p(lab), _p(sz))
    return lab[:rho], sz[:rho]


def get_center(g: Graph, model, t32, seed, r, center_of, clabel, csize, is_seed, v):
    d, l, vis = C.c_int64(), C.c_int64(), C.c_uint64()
    clabel = np.ascontiguousarray(clabel, np.uint32)
    csize = np.ascontiguousarray(csize, np.uint32)
    is_seed = np.ascontiguousarray(is_seed, np.uint8)
    lib().orc_get_center(g.n, _p(g.off), _p(g.nbr), model, t32, seed, r, _p(center_of),
                         _p(clabel), _p(csize), _p(is_seed), v,
                         C.byref(d), C.byref(l), C.byref(vis))
    return d.value, l.value, vis.value


def greedy_alg3(g: Graph, model, t32, R, seed, a32, k):
    seeds = np.zeros(k, np.uint32)
    gain = np.zeros(k, np.int64)
    sigma = np.zeros(k, np.int64)
    visits = C.c_uint64()
    rc = lib().orc_greedy_alg3(g.n, _p(g.off), _p(g.nbr), model, t32, R, seed, a32, k,
                               _p(seeds), _p(gain), _p(sigma), C.byref(visits))
    if rc != 0:
        raise RuntimeError(rc)
    return seeds, gain, sigma, visits.value


# ----------------------------------------------------------- NEXT f3
DECOR = 1 << 8  # model word bit: the decorrelated hash rule (R20)


def live_decor(seed: int, u: int, v: int, r: int, t32: int) -> bool:
    return bool(lib().orc_live_decor(seed, u, v, r, t32))


def simulate_ic(g: Graph, model: int, t32: int, seeds, nsims: int, mc_seed: int) -> int:
    """R21: total vertices reached from `seeds` over nsims Monte-Carlo worlds."""
    s = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint32))
    return int(lib().orc_simulate_ic(g.n, _p(g.off), _p(g.nbr), model, t32, _p(s), len(s), nsims,
                                     mc_seed))
