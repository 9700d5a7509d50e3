"""Pins of the oracle's VERIFY mode (GeneralGreedy P:396-401,
Alg. 1 NextSeed / MarkSeed P:524-530, tie by id P:2285-2286) and of the R2
domain separation, CPU only.

verify() certifies a claimed (seed, gain) sequence.  It is pinned against
things other than itself:
* brute-force GeneralGreedy recomputing N(S) from scipy connected components
  of the materialised sampled graphs: its sequence is accepted;
* every one-step corruption (gain +-1, a seed swapped with the runner-up or
  with a later seed, a repeated seed, the last seed replaced) is rejected at
  the corrupted step;
* the committed derive-mode golden of c1 (tests/golden/c1.json) is accepted
  (c2's, 22 min of single-thread derive mode, was verified once in 63 s with
  8 threads).
"""
import json
import math
import os

import numpy as np
import pytest

import inputs
from tests.test_oracle_pins import (PS, brute_greedy, materialise, model_of, scipy_labels,
                                    tiny_graph)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("i", range(14))
def test_verify_accepts_brute_force_greedy(orc, i):
    g = tiny_graph(i)
    if g.n > 60:
        return
    p = PS[(i + 2) % len(PS)]
    model, t32 = model_of(orc, p)
    R, k, seed = [3, 8][i % 2], min(7, g.n), 70 + i
    labs = [scipy_labels(g.n, materialise(orc, g, model, t32, seed, r))[0] for r in range(R)]
    S, G, _ = brute_greedy(g.n, labs, k)
    for th in (1, 3):
        rc, info = orc.verify(g, model, t32, R, seed, S, G, threads=th)
        assert rc == 0, info
    # rejections, each at the corrupted step
    for j in range(k):
        for d in (-1, 1):
            G2 = list(G)
            G2[j] += d
            rc, info = orc.verify(g, model, t32, R, seed, S, G2, threads=2)
            assert rc == 1 and info[0] == j
    for j in range(k - 1):
        S2 = list(S)
        S2[j], S2[j + 1] = S2[j + 1], S2[j]
        if S2 == S:
            continue
        rc, info = orc.verify(g, model, t32, R, seed, S2, G, threads=2)
        assert rc in (1, 2) and info[0] == j
    S2 = list(S)
    S2[-1] = S[0]
    rc, info = orc.verify(g, model, t32, R, seed, S2, G, threads=1)
    assert rc == 3 and info[0] == k - 1
    others = [v for v in range(g.n) if v not in S]
    if others:
        # a vertex that is not the argmax at the last step: its true gain is
        # claimed, so (a) holds and (b) must catch it (or its gain ties with a
        # smaller id, also (b)); if it happens to carry the same gain with a
        # larger id than s_k, (b) again.
        S2 = list(S)
        S2[-1] = others[-1]
        rc, info = orc.verify(g, model, t32, R, seed, S2, G, threads=1)
        assert rc in (1, 2) and info[0] == k - 1


CASES = [
    (lambda: inputs.random_graph(200, 600, 1), 0.05, 64, 10),
    (lambda: inputs.random_powerlaw_graph(2000, 8000, 3), 0.02, 64, 16),
    (lambda: inputs.random_powerlaw_graph(1500, 9000, 4), "wic", 33, 12),
    (lambda: inputs.random_graph(300, 900, 6), 1.0, 5, 6),
    (lambda: inputs.random_graph(300, 900, 7), 0.0, 7, 5),
    (lambda: inputs.star_graph(50), 0.3, 64, 4),
    (lambda: inputs.path_graph(257), 0.9, 40, 7),
    (lambda: inputs.random_powerlaw_graph(3000, 20000, 12), ("unif", 0.0, 0.1), 64, 12),
    (lambda: inputs.random_graph(40, 80, 5), 0.5, 3, 40),      # k = n: every vertex
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_verify_accepts_derive_mode(orc, i):
    """verify(derive(x)) on the tiny corpus, incl. k = n and all-zero-gain
    tails (p = 0, p = 1): accepted; the covered entries equal sigma_num_k."""
    from oracle.oracle import Graph
    fn, p, R, k = CASES[i]
    off, nbr = fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    k = min(k, g.n)
    s, gn, sg, _ = orc.greedy(g, model, t32, R, 500 + i, k)
    rc, info = orc.verify(g, model, t32, R, 500 + i, s, gn, threads=4)
    assert rc == 0 and info[0] == k
    assert info[3] == sg[-1]         # Σ|∪ C_r(s)| = N(S_k)
    bad = gn.copy()
    bad[k // 2] += 1
    assert orc.verify(g, model, t32, R, 500 + i, s, bad, threads=4)[0] == 1


def test_verify_dense_step_lists(orc):
    """A giant first CC (p = 1 on a connected graph: C_r(s_1) = V in every
    sketch) overflows the per-thread list into the dense accumulator."""
    from oracle.oracle import Graph
    off, nbr = inputs.path_graph(300)
    g = Graph(300, off, nbr)
    s, gn, _, _ = orc.greedy(g, 0, 1 << 32, 6, 3, 5)
    assert list(gn) == [6 * 300, 0, 0, 0, 0]
    for th in (1, 2, 5):
        assert orc.verify(g, 0, 1 << 32, 6, 3, s, gn, threads=th)[0] == 0


def test_verify_c1_golden(orc):
    """BASELINE.json configs[0] at full size: the committed derive-mode golden
    is accepted; its one-seed swap is rejected."""
    gold = json.load(open(os.path.join(GOLD, "c1.json")))
    cfg = inputs.config("c1")
    g = orc.gen_config(cfg)
    model, t32 = orc.model_args(cfg)
    rc, info = orc.verify(g, model, t32, cfg["R"], cfg["hash_seed"], gold["seeds"],
                          gold["gain_num"])
    assert rc == 0, info and info[3] == gold["sigma_num"][-1]
    s = list(gold["seeds"])
    s[1], s[2] = s[2], s[1]
    assert orc.verify(g, model, t32, cfg["R"], cfg["hash_seed"], s, gold["gain_num"])[0] != 0


# ---------------------------------------------------- F4 domain separation
def test_domain_separation_edge_0_r(orc):
    """SURVEY F4 / reading R2: hash(r) and hash(e) use disjoint key domains
    (bit 63 set for sketches).  Without it the key of edge (0, r) equals the
    key of sketch r, hash_edge(0, r, r) = 0 and the edge is live in sketch r
    for every p > 0.  With it, over 2000 hash seeds, the edge (0, r) is live
    in sketch r with frequency p (binomial, 5 sigma), and hash_edge != 0."""
    p = 0.05
    t = orc.t32_const(p)
    for r in (1, 2, 7, 255):
        cnt = 0
        for seed in range(2000):
            assert orc.hash_edge(seed, 0, r, r) != 0
            cnt += orc.live(seed, 0, r, r, t)
        assert abs(cnt - 2000 * p) < 5 * math.sqrt(2000 * p * (1 - p)), (r, cnt)


# ------------------------------------------------ the CELF reference (f2)
@pytest.mark.parametrize("i", range(6))
def test_celf_reference_is_general_greedy(orc, i):
    """tests/celf_ref.py (the literal heap-based CELF the library's CELF
    counter is checked against) selects GeneralGreedy's sequence on the
    oracle's sketches (lazy evaluation is exact under submodularity), and its
    re-evaluation count lies between k - 1 and (k - 1) * n."""
    from tests.celf_ref import celf_reevaluations
    g = tiny_graph(i)
    p = PS[(i + 3) % len(PS)]
    model, t32 = model_of(orc, p)
    R, k, seed = 6, min(6, g.n), 90 + i
    labs, sizes = zip(*[orc.sketch_labels(g, model, t32, seed, r) for r in range(R)])
    s, gn, reev = celf_reevaluations(labs, sizes, g.n, k)
    es, egn, _, _ = orc.greedy(g, model, t32, R, seed, k)
    assert s == list(es) and gn == list(egn)
    assert k - 1 <= reev <= (k - 1) * g.n
