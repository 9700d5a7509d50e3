"""Pins of the oracle's Alg. 3 transcription (compressed sketches, GetCenter,
MarkSeed) and of the input generators (CPU only)."""
import numpy as np
import pytest

import inputs
from tests.test_oracle_pins import materialise, scipy_labels, tiny_graph


@pytest.mark.parametrize("i", range(6))
def test_compressed_sketch_matches_scipy(orc, i):
    # label[i] = smallest center index j with c_j in c_i's CC;
    # size[i] = CC size when label[i] = i.
    g = tiny_graph(i)
    model, t32 = (0, orc.t32_const([0.2, 0.5, 0.05][i % 3]))
    seed, a32 = 21 + i, [1 << 30, 1 << 31, 1 << 28][i % 3]
    cs, _ = orc.centers(g.n, seed, a32)
    for r in (0, 5):
        lab, sz = orc.compressed_sketch(g, model, t32, seed, r, a32)
        vlab, vsz = scipy_labels(g.n, materialise(orc, g, model, t32, seed, r))
        for ci, c in enumerate(cs):
            same = [j for j, cj in enumerate(cs) if vlab[cj] == vlab[c]]
            assert lab[ci] == min(same)
            assert sz[ci] == (vsz[c] if lab[ci] == ci else 0)


def test_centers_bernoulli_alpha(orc):
    # R9: each vertex is a center independently with probability A32/2^32.
    n = 200000
    for a32 in (1 << 28, 1 << 30):
        cs, _ = orc.centers(n, 9, a32)
        p = a32 / 2**32
        assert abs(len(cs) - p * n) < 5 * np.sqrt(n * p * (1 - p))
    cs, _ = orc.centers(100, 9, 1 << 32)
    assert len(cs) == 100  # alpha = 1: all centers


def test_get_center_trivia(orc):
    from oracle.oracle import Graph
    # SPEC S:187-189 style: (a) connected graph p=1, v a center, no seeds ->
    # (n, label); (b) p=0, v not a center, not a seed -> (1, -1); (c) CC {a,b}
    # with no center, a in S -> get_center(b) = (0, -1).
    off, nbr = inputs.path_graph(8)
    g = Graph(8, off, nbr)
    seed = 3
    a32 = 1 << 31
    cs, center_of = orc.centers(8, seed, a32)
    assert 0 < len(cs) < 8
    lab, sz = orc.compressed_sketch(g, 0, 1 << 32, seed, 0, a32)
    no_seed = np.zeros(8, np.uint8)
    d, l, vis = orc.get_center(g, 0, 1 << 32, seed, 0, center_of, lab, sz, no_seed, int(cs[0]))
    assert (d, l, vis) == (8, 0, 1)
    nonc = [v for v in range(8) if center_of[v] == 0xFFFFFFFF][0]
    lab0, sz0 = orc.compressed_sketch(g, 0, 0, seed, 0, a32)
    d, l, vis = orc.get_center(g, 0, 0, seed, 0, center_of, lab0, sz0, no_seed, nonc)
    assert (d, l, vis) == (1, -1, 1)
    # two-vertex CC without any center (a32 = 0 -> no centers at all)
    off, nbr = inputs.csr_from_edges(4, [(0, 1)])
    g = Graph(4, off, nbr)
    _, center_of = orc.centers(4, seed, 0)
    is_seed = np.array([1, 0, 0, 0], np.uint8)
    empty = np.zeros(1, np.uint32)
    assert orc.get_center(g, 0, 1 << 32, seed, 0, center_of, empty, empty, is_seed, 1)[:2] == (0, -1)
    assert orc.get_center(g, 0, 1 << 32, seed, 0, center_of, empty, empty,
                          np.zeros(4, np.uint8), 1)[:2] == (2, -1)


@pytest.mark.parametrize("i", range(8))
def test_alg3_greedy_equals_memoised_greedy(orc, i):
    """Compression transparency: Alg. 3's exhaustive
    greedy over compressed sketches with any alpha picks the same seeds and
    gains as the memoised (alpha=1) definition."""
    g = tiny_graph(i % 2)  # n = 12 or 30
    p = [0.2, 0.5, "wic", 1.0][i % 4]
    model, t32 = (1, 0) if p == "wic" else (0, orc.t32_const(p))
    a32 = [0, 1 << 29, 1 << 31, 1 << 32][i % 4]
    R, k, seed = 6, 4, 90 + i
    s1, g1, sg1, _ = orc.greedy(g, model, t32, R, seed, k)
    s2, g2, sg2, _ = orc.greedy_alg3(g, model, t32, R, seed, a32, k)
    assert list(s1) == list(s2) and list(g1) == list(g2) and list(sg1) == list(sg2)


def test_thm31_visit_bound(orc):
    # Thm 3.1: expected BFS visits until a center <= 1/alpha on a
    # large connected sampled graph; SPEC S:529 bound 2/alpha.  p=0: exactly 1.
    from oracle.oracle import Graph
    n = 10000
    off, nbr = inputs.random_graph(n, 4 * n, seed=5)
    g = Graph(n, off, nbr)
    alpha_a32 = int(0.1 * 2**32)
    seed = 4
    _, center_of = orc.centers(n, seed, alpha_a32)
    lab, sz = orc.compressed_sketch(g, 0, 1 << 32, seed, 0, alpha_a32)
    rng = np.random.default_rng(0)
    no_seed = np.zeros(n, np.uint8)
    vis = [orc.get_center(g, 0, 1 << 32, seed, 0, center_of, lab, sz, no_seed, int(v))[2]
           for v in rng.integers(0, n, 300)]
    assert np.mean(vis) <= 2 / 0.1
    lab0, sz0 = orc.compressed_sketch(g, 0, 0, seed, 0, alpha_a32)
    vis0 = [orc.get_center(g, 0, 0, seed, 0, center_of, lab0, sz0, no_seed, int(v))[2]
            for v in rng.integers(0, n, 50)]
    assert set(vis0) == {1}


# -------------------------------------------------------------- generators
def check_csr(g):
    off, nbr = g.off.astype(np.int64), g.nbr.astype(np.int64)
    assert off[0] == 0 and np.all(np.diff(off) >= 0) and off[-1] == len(nbr)
    src = np.repeat(np.arange(g.n), np.diff(off))
    assert np.all(src != nbr)
    key = src * g.n + nbr
    assert np.all(np.diff(key) > 0)  # sorted lists, no duplicates
    rkey = np.sort(nbr * g.n + src)
    assert np.array_equal(rkey, key)  # symmetric


def test_gen_er(orc):
    g = orc.gen_er(4096, 32768, 1)
    assert g.m == 32768
    check_csr(g)
    g2 = orc.gen_er(300, 2000, 7)
    check_csr(g2)
    assert g2.m == 2000


def test_gen_grid(orc):
    W, H = 64, 48
    d32 = inputs.diag_threshold(0.3)
    g = orc.gen_grid(W, H, d32, 1)
    check_csr(g)
    ndiag = g.m - (2 * W * H - W - H)
    cells = (W - 1) * (H - 1)
    assert abs(ndiag - 0.3 * cells) < 5 * np.sqrt(cells * 0.21)


def test_gen_rmat(orc):
    c = inputs.config("c2", scale=12, ef=16)
    g = orc.gen_rmat(12, 16, c["rmat_t"], 1, 1)
    check_csr(g)
    deg = np.diff(g.off.astype(np.int64))
    assert 0.6 * 16 * 4096 < g.m <= 16 * 4096
    assert deg.max() > 20 * deg.mean()  # heavy tail (a = 0.57)
    # permutation is a bijection: same degree multiset with/without it
    g0 = orc.gen_rmat(12, 16, c["rmat_t"], 0, 1)
    assert np.array_equal(np.sort(np.diff(g0.off.astype(np.int64))), np.sort(deg))
