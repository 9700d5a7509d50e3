"""Oracle pins of NEXT row f3: the decorrelated hash rule (R20)
and the Monte-Carlo sigma(S) simulator (R21).  CPU only."""
import math

import numpy as np
import pytest

import inputs
from tests.test_oracle_pins import exact_sigma, materialise, scipy_labels, tiny_graph


def test_decor_live_fraction_and_independence(orc):
    """R20: live fraction p within 5 sigma; two sketches are live together with
    probability p^2 (independent), while the literal rule makes sketches
    whose hash(r) share the leading bits nearly identical."""
    p = 0.05
    t = orc.t32_const(p)
    rng = np.random.default_rng(3)
    us, vs = rng.integers(0, 1 << 20, 40000), rng.integers(0, 1 << 20, 40000)
    E = len(us)
    # two sketches with equal top 5 bits of hash(r) under seed 9 (w = clz(T - 1) = 4)
    hr = [orc.hash_r(9, r) >> 59 for r in range(64)]
    r1 = 0
    r2 = next(r for r in range(1, 64) if hr[r] == hr[r1])
    lit1 = np.array([orc.live(9, int(u), int(v), r1, t) for u, v in zip(us, vs)])
    lit2 = np.array([orc.live(9, int(u), int(v), r2, t) for u, v in zip(us, vs)])
    dec1 = np.array([orc.live_decor(9, int(u), int(v), r1, t) for u, v in zip(us, vs)])
    dec2 = np.array([orc.live_decor(9, int(u), int(v), r2, t) for u, v in zip(us, vs)])
    sd = math.sqrt(E * p * (1 - p))
    assert abs(dec1.sum() - p * E) < 5 * sd and abs(dec2.sum() - p * E) < 5 * sd
    both = (dec1 & dec2).sum()
    assert abs(both - p * p * E) < 5 * math.sqrt(E * p * p)
    assert (lit1 & lit2).sum() > 3 * p * p * E  # the literal rule's correlation (F1)


@pytest.mark.parametrize("i", range(6))
def test_decor_labels_equal_scipy(orc, i):
    g = tiny_graph(i)
    model, t32 = orc.DECOR | 0, orc.t32_const([0.1, 0.3, 0.6][i % 3])
    for r in (0, 5):
        lab, sz = orc.sketch_labels(g, model, t32, 21 + i, r)
        live = [(u, v) for u in range(g.n) for v in map(int, g.nbr[g.off[u]:g.off[u + 1]])
                if v > u and orc.live_decor(21 + i, u, v, r, t32)]
        elab, esz = scipy_labels(g.n, live)
        assert np.array_equal(lab, elab) and np.array_equal(sz, esz)


def test_decor_sigma_hat_unbiased(orc):
    """Decorrelated sketches: the mean over hash seeds of sigma_hat equals the
    exact sigma within 4.5 standard errors, and — sketches now independent —
    the across-seed spread is close to sd(|reach|) / sqrt(R)."""
    from oracle.oracle import Graph
    n, edges, p = 6, [(0, i) for i in range(1, 6)], 0.3
    off, nbr = inputs.csr_from_edges(n, edges)
    g = Graph(n, off, nbr)
    t32 = orc.t32_const(p)
    R, NS = 64, 300
    est = np.array([orc.greedy(g, orc.DECOR, t32, R, 500 + s, 1, want_gain0=True)[3][0] / R
                    for s in range(NS)])
    ex = exact_sigma(n, edges, [t32 / 2**32] * len(edges), [0])
    assert abs(est.mean() - ex) <= 4.5 * est.std(ddof=1) / math.sqrt(NS)
    sd1 = math.sqrt(5 * p * (1 - p))  # |reach(0)| - 1 ~ Binomial(5, p)
    assert 0.7 * sd1 / math.sqrt(R) < est.std(ddof=1) < 1.4 * sd1 / math.sqrt(R)


def test_mc_closed_forms(orc):
    """R21: p = 0 reaches exactly S; p = 1 reaches the union of S's CCs."""
    g = tiny_graph(3)
    S = [0, 5, 7]
    assert orc.simulate_ic(g, 0, 0, S, 50, 1) == 50 * 3
    lab, _ = scipy_labels(g.n, [(u, int(v)) for u in range(g.n)
                                for v in g.nbr[g.off[u]:g.off[u + 1]] if v > u])
    reach = sum(1 for x in lab if x in {lab[s] for s in S})
    assert orc.simulate_ic(g, 0, 1 << 32, S, 50, 1) == 50 * reach


@pytest.mark.parametrize("case", ["const", "wic", "unif"])
def test_mc_matches_exact_sigma(orc, case):
    """The MC estimate of sigma(S) over 4000 worlds equals the exact sigma (all
    2^m live-edge worlds enumerated) within 5 standard errors of the per-world
    spread, for the three probability models."""
    from oracle.oracle import Graph
    n, edges = 7, [(0, 1), (1, 2), (2, 3), (0, 3), (3, 4), (4, 5), (5, 6), (1, 5)]
    off, nbr = inputs.csr_from_edges(n, edges)
    g = Graph(n, off, nbr)
    deg = np.diff(off.astype(np.int64))
    if case == "const":
        model, t32 = 0, orc.t32_const(0.4)
        probs = [t32 / 2**32] * len(edges)
    elif case == "wic":
        model, t32 = 1, 0
        probs = [orc.t32_wic(int(deg[u]), int(deg[v])) / 2**32 for u, v in edges]
    else:
        model, t32 = 2, orc.uniform_param(0.1, 0.7)
        probs = [orc.t32_uniform(t32, u, v) / 2**32 for u, v in edges]
    S = [0, 4]
    N = 4000
    per = np.array([orc.simulate_ic(g, model, t32, S, 1, 77 + i) for i in range(400)], float)
    tot = orc.simulate_ic(g, model, t32, S, N, 5)
    ex = exact_sigma(n, edges, probs, S)
    assert abs(tot / N - ex) <= 5 * per.std(ddof=1) / math.sqrt(N)
    assert abs(per.mean() - ex) <= 5 * per.std(ddof=1) / math.sqrt(len(per))
