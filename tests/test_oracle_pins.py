"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a published test vector, a
closed form, a library routine on a special case (scipy connected components
on the materialised sampled graph), brute force on tiny inputs, an invariant,
or an exact enumeration with a statistical bound.  See DESIGN.md §Oracle.
"""
import itertools
import math

import numpy as np
import pytest
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components

import inputs

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


# --------------------------------------------------------------------- hash
def test_mix64_published_splitmix64_vectors(orc):
    # splitmix64 (Steele, Lea, Flood 2014; Vigna's reference splitmix64.c)
    # seeded with 0 produces 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4,
    # 0x06c45d188009454f: next() = mix64(state += GOLDEN).
    expect = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    got = [orc.mix64((i * GOLDEN) & M64) for i in (1, 2, 3)]
    assert got == expect


def test_t32_closed_forms(orc):
    # R3: T32 = floor(p * 2^32); exact dyadic cases and the p=1 cap.
    assert orc.t32_const(0.0) == 0
    assert orc.t32_const(0.25) == 1 << 30
    assert orc.t32_const(0.5) == 1 << 31
    assert orc.t32_const(1.0) == 1 << 32
    assert orc.t32_const(1.5) == 1 << 32
    # BASELINE.json configs: p = 0.05, 0.02, 0.01 -> floor of the exact product
    for p, t in [(0.05, 214748364), (0.02, 85899345), (0.01, 42949672)]:
        assert orc.t32_const(p) == t
        assert abs(t / 2**32 - p) < 2**-32


def test_t32_wic_matches_paper_formula(orc):
    # P:2034 / P:2013: p_uv = 2/(d_u + d_v), capped at 1 (BASELINE.json c4).
    rng = np.random.default_rng(0)
    for du, dv in rng.integers(1, 10**6, size=(2000, 2)):
        t = orc.t32_wic(int(du), int(dv))
        p = min(1.0, 2.0 / (int(du) + int(dv)))
        assert 0 <= p * 2**32 - t < 1.0 + 1e-6
    assert orc.t32_wic(1, 1) == 1 << 32       # two leaves: always live
    assert orc.t32_wic(1, 2) == (1 << 33) // 3  # path 0-1-2, edge (0,1): p = 2/3


def test_t32_uniform_pins(orc):
    """R19 (P:2032 'draw a uniform random number from x to y'; SPEC S:31 'per-edge
    value drawn deterministically from the edge key'): lo = hi reduces to the
    constant threshold; every value lies in [L, H]; symmetric in (u, v); over
    2e5 edges the mean is (L + H) / 2 within 5 sigma of a uniform law and a
    20-bin histogram passes chi-square at 1e-4."""
    rng = np.random.default_rng(7)
    us = rng.integers(0, 1 << 31, 200000)
    vs = rng.integers(0, 1 << 31, 200000)
    for p in (0.0, 0.02, 0.5):
        P = orc.uniform_param(p, p)
        assert all(orc.t32_uniform(P, int(u), int(v)) == orc.t32_const(p)
                   for u, v in zip(us[:200], vs[:200]))
    lo, hi = 0.1, 0.3
    P = orc.uniform_param(lo, hi)
    L, H = P & 0xFFFFFFFF, P >> 32
    assert L == orc.t32_const(lo) and H == orc.t32_const(hi)
    t = np.array([orc.t32_uniform(P, int(u), int(v)) for u, v in zip(us, vs)], np.float64)
    assert t.min() >= L and t.max() <= H
    assert all(orc.t32_uniform(P, int(u), int(v)) == orc.t32_uniform(P, int(v), int(u))
               for u, v in zip(us[:500], vs[:500]))
    x = (t - L) / (H - L)
    assert abs(x.mean() - 0.5) < 5 * math.sqrt(1 / 12 / len(x))
    cnt = np.histogram(x, bins=20, range=(0, 1))[0]
    chi2 = ((cnt - len(x) / 20) ** 2 / (len(x) / 20)).sum()
    assert chi2 < 53.0  # chi-square 19 dof, p = 1e-4
    assert orc.uniform_param(0.5, 1.0) >> 32 == (1 << 32) - 1  # hi = 1: H capped below 2^32


def test_live_symmetry_and_extremes(orc):
    rng = np.random.default_rng(1)
    for _ in range(500):
        u, v = (int(x) for x in rng.integers(0, 2**31 - 1, 2))
        if u == v:
            continue
        r = int(rng.integers(0, 1024))
        seed = int(rng.integers(0, 2**63))
        assert orc.hash_edge(seed, u, v, r) == orc.hash_edge(seed, v, u, r)
        assert not orc.live(seed, u, v, r, 0)           # p = 0: never
        assert orc.live(seed, u, v, r, 1 << 32)         # p = 1: always
        t = int(rng.integers(1, 2**32))
        assert orc.live(seed, u, v, r, t) == orc.live(seed, v, u, r, t)


@pytest.mark.parametrize("p", [0.02, 0.3])
def test_live_fraction_is_p(orc, p):
    # Each sketch is a Bernoulli(p) world: for a fixed r, the edge hashes are
    # uniform, so the live fraction over many edges is p (binomial 5 sigma).
    t = orc.t32_const(p)
    rng = np.random.default_rng(2)
    E = 20000
    us = rng.integers(0, 2**30, E)
    vs = rng.integers(2**30, 2**31 - 1, E)
    for r in (0, 7, 123):
        cnt = sum(orc.live(5, int(u), int(v), r, t) for u, v in zip(us, vs))
        assert abs(cnt - p * E) < 5 * math.sqrt(E * p * (1 - p))


# --------------------------------------------------------------- sketches
def materialise(orc, g, model, t32, seed, r):
    """Live edge list of G'_r, one oracle liveness call per undirected edge."""
    deg = np.diff(g.off.astype(np.int64))
    out = []
    for u in range(g.n):
        for e in range(int(g.off[u]), int(g.off[u + 1])):
            v = int(g.nbr[e])
            if v <= u:
                continue
            t = (orc.t32_wic(int(deg[u]), int(deg[v])) if model == 1 else
                 orc.t32_uniform(t32, u, v) if model == 2 else t32)
            if orc.live(seed, u, v, r, t):
                out.append((u, v))
    return out


def scipy_labels(n, edges):
    """Canonical (min-id) component labels and sizes via scipy."""
    if edges:
        e = np.array(edges)
        A = coo_matrix((np.ones(len(e)), (e[:, 0], e[:, 1])), shape=(n, n))
    else:
        A = coo_matrix((n, n))
    _, lab = connected_components(A, directed=False)
    minid = np.full(lab.max() + 1, n, np.int64)
    np.minimum.at(minid, lab, np.arange(n))
    sizes = np.bincount(lab)
    return minid[lab], sizes[lab]


def tiny_graph(i):
    n = [12, 30, 60, 120][i % 4]
    m = [15, 60, 150, 200][i % 4]
    if i % 3 == 0:
        off, nbr = inputs.random_powerlaw_graph(n, m, seed=100 + i)
    else:
        off, nbr = inputs.random_graph(n, m, seed=100 + i)
    from oracle.oracle import Graph
    return Graph(n, off, nbr)


PS = [0.0, 0.05, 0.2, 0.5, 1.0, "wic", ("unif", 0.0, 0.1), ("unif", 0.1, 0.3), ("unif", 0.3, 0.9)]


def model_of(orc, p):
    """(model, t32): constant, WIC (R4) or Uniform U(lo, hi) (R19)."""
    if p == "wic":
        return 1, 0
    if isinstance(p, tuple):
        return 2, orc.uniform_param(p[1], p[2])
    return 0, orc.t32_const(p)


@pytest.mark.parametrize("i", range(18))
def test_sketch_labels_equal_scipy_on_materialised_graph(orc, i):
    g = tiny_graph(i)
    p = PS[i % len(PS)]
    model, t32 = model_of(orc, p)
    for r in (0, 3, 17):
        seed = 11 + i
        lab, sz = orc.sketch_labels(g, model, t32, seed, r)
        elab, esz = scipy_labels(g.n, materialise(orc, g, model, t32, seed, r))
        assert np.array_equal(lab, elab)
        assert np.array_equal(sz, esz)


def test_sketch_p0_singletons_p1_components(orc):
    g = tiny_graph(2)
    lab, sz = orc.sketch_labels(g, 0, 0, 3, 5)
    assert np.array_equal(lab, np.arange(g.n)) and np.all(sz == 1)
    lab, sz = orc.sketch_labels(g, 0, 1 << 32, 3, 5)
    edges = [(u, int(v)) for u in range(g.n) for v in g.nbr[g.off[u]:g.off[u + 1]] if v > u]
    elab, esz = scipy_labels(g.n, edges)
    assert np.array_equal(lab, elab) and np.array_equal(sz, esz)
    for r in range(4):  # sizes sum to n per sketch (each CC counted once)
        lab, sz = orc.sketch_labels(g, 0, orc.t32_const(0.3), 9, r)
        assert sum(sz[lab == np.arange(g.n)]) == g.n


# ----------------------------------------------------------------- greedy
def brute_greedy(n, labs, k):
    """GeneralGreedy on N(S) = sum_r |union_{s in S} C_r(s)|,
    recomputed from scratch for every candidate; ties -> smallest id."""
    R = len(labs)
    sizes = [np.bincount(l, minlength=n) for l in labs]

    def N(S):
        return sum(sum(int(sizes[r][c]) for c in {int(labs[r][s]) for s in S}) for r in range(R))

    S, gains, sig = [], [], []
    for _ in range(k):
        base = N(S)
        best = None
        for v in range(n):
            if v in S:
                continue
            gv = N(S + [v]) - base
            if best is None or gv > best[0]:
                best = (gv, v)
        S.append(best[1])
        gains.append(best[0])
        sig.append(base + best[0])
    return S, gains, sig


@pytest.mark.parametrize("i", range(14))
def test_greedy_equals_brute_force(orc, i):
    g = tiny_graph(i)
    if g.n > 60:
        return
    p = PS[(i + 1) % len(PS)]
    model, t32 = model_of(orc, p)
    R, k, seed = [4, 16][i % 2], min(6, g.n), 40 + i
    seeds, gain, sigma, gain0 = orc.greedy(g, model, t32, R, seed, k, want_gain0=True)
    labs = [scipy_labels(g.n, materialise(orc, g, model, t32, seed, r))[0] for r in range(R)]
    S, G, SG = brute_greedy(g.n, labs, k)
    assert list(seeds) == S
    assert list(gain) == G
    assert list(sigma) == SG
    # gain0 = R * Marginal(empty, v) = sum_r |C_r(v)|
    exp0 = sum(np.bincount(l, minlength=g.n)[l] for l in labs)
    assert np.array_equal(gain0, exp0)
    assert all(a >= b for a, b in zip(gain, gain[1:]))  # submodularity


def test_greedy_closed_forms(orc):
    from oracle.oracle import Graph
    # two disjoint paths: sizes 5 (ids 3..7) and 3 (ids 0..2), plus isolated 8, 9
    off, nbr = inputs.csr_from_edges(10, [(0, 1), (1, 2), (3, 4), (4, 5), (5, 6), (6, 7)])
    g = Graph(10, off, nbr)
    R = 8
    s, gn, sg, _ = orc.greedy(g, 0, 1 << 32, R, 1, 5)
    # p=1: largest CC first (min id 3), then size-3 CC (min id 0), then the
    # isolated vertices 8, 9, then all gains 0 -> smallest non-seed id (1).
    assert list(s) == [3, 0, 8, 9, 1]
    assert list(gn) == [5 * R, 3 * R, R, R, 0]
    assert list(sg) == [5 * R, 8 * R, 9 * R, 10 * R, 10 * R]
    # p=0: every vertex a singleton in every sketch -> gains R, seeds 0..k-1
    s, gn, sg, _ = orc.greedy(g, 0, 0, R, 1, 4)
    assert list(s) == [0, 1, 2, 3] and list(gn) == [R] * 4
    # star with centre 0, p=1: all d+1 vertices tie at R(d+1): seed 0, then 0s
    off, nbr = inputs.star_graph(6)
    g = Graph(7, off, nbr)
    s, gn, _, _ = orc.greedy(g, 0, 1 << 32, R, 2, 3)
    assert list(s) == [0, 1, 2] and list(gn) == [7 * R, 0, 0]
    # path of L vertices, p=1: every vertex gains R*L, vertex 0 wins
    off, nbr = inputs.path_graph(9)
    g = Graph(9, off, nbr)
    s, gn, _, _ = orc.greedy(g, 0, 1 << 32, R, 2, 2)
    assert list(s) == [0, 1] and list(gn) == [9 * R, 0]


@pytest.mark.parametrize("i", range(6))
def test_greedy_one_minus_inv_e_of_brute_force_opt(orc, i):
    # greedy achieves (1-1/e) OPT of the (coverage) estimator.
    g = tiny_graph(i * 4)  # n = 12
    p = [0.2, 0.5, "wic"][i % 3]
    model, t32 = model_of(orc, p)
    R, seed = 8, 70 + i
    labs = [scipy_labels(g.n, materialise(orc, g, model, t32, seed, r))[0] for r in range(R)]
    sizes = [np.bincount(l, minlength=g.n) for l in labs]

    def N(S):
        return sum(sum(int(sizes[r][c]) for c in {int(labs[r][s]) for s in S}) for r in range(R))

    for k in (1, 2, 3):
        _, _, sigma, _ = orc.greedy(g, model, t32, R, seed, k)
        opt = max(N(list(S)) for S in itertools.combinations(range(g.n), k))
        assert sigma[-1] >= (1 - 1 / math.e) * opt - 1e-9
        assert sigma[-1] <= opt


# ----------------------------------------------------- sigma estimation
def exact_sigma(n, edges, probs, S):
    """sigma(S) by enumerating all 2^m live-edge worlds (P:375-377 IC)."""
    tot = 0.0
    m = len(edges)
    for mask in range(1 << m):
        pr = 1.0
        live = []
        for j in range(m):
            if mask >> j & 1:
                pr *= probs[j]
                live.append(edges[j])
            else:
                pr *= 1 - probs[j]
        if pr == 0:
            continue
        lab, _ = scipy_labels(n, live)
        reach = {int(l) for l in lab[list(S)]}
        tot += pr * sum(1 for x in lab if int(x) in reach)
    return tot


@pytest.mark.parametrize("case", ["star", "path", "er8", "wic", "unif"])
def test_sigma_hat_unbiased_across_hash_seeds(orc, case):
    """Mean over hash seeds of sigma_hat(S) = gain0/R equals exact sigma(S)
    within 4.5 empirical standard errors (F1: the literal rule correlates
    sketches, so the bound uses the across-seed variance, never Var/R)."""
    from oracle.oracle import Graph
    if case == "star":
        n, edges, p = 6, [(0, i) for i in range(1, 6)], 0.3
    elif case == "path":
        n, edges, p = 5, [(i, i + 1) for i in range(4)], 0.5
    elif case == "er8":
        off, nbr = inputs.random_graph(8, 11, seed=3)
        edges = [(u, int(v)) for u in range(8) for v in nbr[off[u]:off[u + 1]] if v > u]
        n, p = 8, 0.3
    elif case == "wic":
        n, edges, p = 7, [(0, 1), (1, 2), (2, 3), (0, 3), (3, 4), (4, 5), (5, 6)], "wic"
    else:
        n, edges, p = 7, [(0, 1), (1, 2), (2, 3), (0, 3), (3, 4), (4, 5), (5, 6)], ("unif", 0.1, 0.6)
    off, nbr = inputs.csr_from_edges(n, edges)
    g = Graph(n, off, nbr)
    deg = np.diff(off.astype(np.int64))
    if p == "wic":
        model, t32 = 1, 0
        probs = [orc.t32_wic(int(deg[u]), int(deg[v])) / 2**32 for u, v in edges]
    elif isinstance(p, tuple):
        model, t32 = 2, orc.uniform_param(p[1], p[2])
        probs = [orc.t32_uniform(t32, u, v) / 2**32 for u, v in edges]
    else:
        model, t32 = 0, orc.t32_const(p)
        probs = [t32 / 2**32] * len(edges)
    R, NS = 64, 400
    est = np.array([orc.greedy(g, model, t32, R, 1000 + s, 1, want_gain0=True)[3] / R
                    for s in range(NS)])
    mean, se = est.mean(0), est.std(0, ddof=1) / math.sqrt(NS)
    for v in range(n):
        ex = exact_sigma(n, edges, probs, [v])
        assert abs(mean[v] - ex) <= 4.5 * se[v] + 1e-9, (v, mean[v], ex, se[v])
    if case == "star":  # closed form sigma({c}) = 1 + d p
        assert abs(exact_sigma(n, edges, probs, [0]) - (1 + 5 * probs[0])) < 1e-12
    if case == "path":  # from an endpoint: sum_{i<L} p^i
        assert abs(exact_sigma(n, edges, probs, [0]) - sum(0.5**i for i in range(5))) < 1e-12


# ------------------------------------------------------ threaded generator
@pytest.mark.parametrize("scale,ef,abc,threads", [(9, 16, (0.57, 0.19, 0.19), 3),
                                                  (13, 24, (0.57, 0.19, 0.19), 8),
                                                  (14, 32, (0.6, 0.15, 0.15), 5)])
def test_threaded_rmat_generator_equals_plain(orc, scale, ef, abc, threads):
    """The threaded R-MAT input generator (bench reference arm, c4 at full
    size) produces the plain generator's keys and CSR bit for bit."""
    cfg = inputs.config("c2", scale=scale, ef=ef, abc=abc)
    a = orc.gen_config(cfg)
    b = orc.gen_config(cfg, threads=threads)
    assert np.array_equal(a.keys, b.keys)
    assert np.array_equal(a.off, b.off) and np.array_equal(a.nbr, b.nbr)
