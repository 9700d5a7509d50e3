"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element on identical seeded inputs.  Everything is integer, so the
bar is bit-exact: canonical labels, CC sizes (via gain0), per-step gains,
seeds, sigma numerators, and the generated CSR itself."""
import hashlib
import json
import os

import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def pc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2311_07554_b200 import build
    build.build()
    import paper_2311_07554_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(pc):
    c = pc.Context(0)
    yield c
    c.close()


def load_host(ctx, g, model, t32, validate=2):
    ctx.pacim_load_graph(g.off, g.nbr, model, t32, validate)


def full_parity(orc, ctx, g, model, t32, R, seed, k, check_labels=True):
    load_host(ctx, g, model, t32)
    ctx.pacim_build_sketches(R, seed)
    s, gn, sg, sigma = ctx.pacim_select_seeds(k)
    es, egn, esg, eg0 = orc.greedy(g, model, t32, R, seed, k, want_gain0=True)
    assert np.array_equal(ctx.pacim_get_gain0(), eg0)
    if check_labels:
        for r in range(R):
            lab, _ = orc.sketch_labels(g, model, t32, seed, r)
            assert np.array_equal(ctx.pacim_get_labels(r), lab), r
    assert list(s) == list(es)
    assert list(gn) == list(egn)
    assert list(sg) == list(esg)
    assert np.allclose(sigma, esg / R)
    return s, gn


# ------------------------------------------------------------ tiny corpus
CASES = [
    # (graph builder, p, R, k)
    (lambda: inputs.random_graph(200, 600, 1), 0.05, 64, 10),
    (lambda: inputs.random_graph(500, 3000, 2), 0.2, 4, 20),
    (lambda: inputs.random_powerlaw_graph(2000, 8000, 3), 0.02, 64, 16),
    (lambda: inputs.random_powerlaw_graph(1500, 9000, 4), "wic", 33, 12),
    (lambda: inputs.random_graph(300, 900, 5), 0.5, 1, 8),
    (lambda: inputs.random_graph(300, 900, 6), 1.0, 5, 6),
    (lambda: inputs.random_graph(300, 900, 7), 0.0, 7, 5),
    (lambda: inputs.random_powerlaw_graph(4000, 30000, 8), 0.05, 256, 30),
    (lambda: inputs.star_graph(50), 0.3, 64, 4),
    (lambda: inputs.path_graph(257), 0.9, 40, 7),
    (lambda: inputs.random_powerlaw_graph(3000, 20000, 12), ("unif", 0.0, 0.1), 64, 12),
    (lambda: inputs.random_graph(2000, 8000, 13), ("unif", 0.1, 0.3), 32, 10),
    (lambda: inputs.star_graph(3000), 0.1, 32, 5),  # hub of expected live degree 300: hot CCs
]


def model_of(orc, p):
    """(model, t32) for the oracle and the library alike: constant, WIC, or
    Uniform U(lo, hi) (R19; the library's own pacim_threshold_uniform must
    give the oracle's packed parameter)."""
    if p == "wic":
        return 1, 0
    if isinstance(p, tuple):
        from paper_2311_07554_b200 import pacim_threshold_uniform
        t = orc.uniform_param(p[1], p[2])
        assert pacim_threshold_uniform(p[1], p[2]) == t
        return 2, t
    return 0, orc.t32_const(p)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_tiny_corpus_parity(orc, ctx, i):
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    full_parity(orc, ctx, g, model, t32, R, 1000 + i, min(k, g.n))


@pytest.mark.parametrize("i", [0, 2, 3, 7, 10])
def test_compact_store_csr_direct(orc, ctx, i, monkeypatch):
    """The compact store's mask and union passes over the CSR-direct edge
    form (PACIM_UCSR=4, no edge lists derived): the oracle's parity."""
    monkeypatch.setenv("PACIM_UCSR", "4")
    test_tiny_corpus_parity_compact_store(orc, ctx, i, monkeypatch)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_tiny_corpus_parity_compact_store(orc, ctx, i, monkeypatch):
    """The compact store forced (PACIM_STORE=compact; by default a one-GPU
    build takes the dense store when it fits, a sharded build the compact
    one): the same oracle parity.  Sketches with more than half of their
    (vertex, sketch) pairs non-singleton keep the dense store."""
    monkeypatch.setenv("PACIM_STORE", "compact")
    test_tiny_corpus_parity(orc, ctx, i)
    st = ctx.pacim_get_stats()
    assert st["store"] == 1 or st["nnonsingle"] > 0.5 * st["rows"] * st["R_local"]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_tiny_corpus_parity_dense_store(orc, ctx, i, monkeypatch):
    """The dense vertex-major store (the layout dense sketches such as c3
    use; PACIM_STORE=dense forces it): the same oracle parity."""
    monkeypatch.setenv("PACIM_STORE", "dense")
    test_tiny_corpus_parity(orc, ctx, i)
    assert ctx.pacim_get_stats()["store"] == 0


def gapped_graph(nv, m, gap, seed):
    """random_graph's edges on the ids v * gap + v % 5 of a graph with
    nv * gap vertices: runs of isolated vertices longer than 255, so the
    edge stream's vertex and row deltas overflow their bytes."""
    off, nbr = inputs.random_graph(nv, m, seed)
    e = [(u * gap + u % 5, int(v) * gap + int(v) % 5)
         for u in range(nv) for v in nbr[int(off[u]):int(off[u + 1])] if v > u]
    return inputs.csr_from_edges(nv * gap, e)


@pytest.mark.parametrize("ucsr", ["1", "0", "2", "3", "4"])
@pytest.mark.parametrize("i", [0, 2, 3, 7, 10, 12, -1])
def test_dense_store_edge_streams(orc, ctx, i, ucsr, monkeypatch):
    """The dense store's upper-edge stream (UpperCsr: neighbours, row deltas
    and the neighbours' rows per edge; 1, the default when the edge lists
    would take more than a fifth of the device), the edge lists
    keys / ckeys (0), the neighbours' rows from the rank map (2), every delta
    capped so the offsets walk and the rank map serve every edge (3), the
    CSR-direct form (4: no per-edge array, the default when not even the
    stream fits — c5): the
    same oracle parity (labels, gain0, seeds, gains).  i = -1: a graph whose
    runs of isolated vertices exceed a byte (deltas overflow naturally)."""
    monkeypatch.setenv("PACIM_STORE", "dense")
    monkeypatch.setenv("PACIM_UCSR", ucsr)
    if i < 0:
        from oracle.oracle import Graph
        off, nbr = gapped_graph(300, 2400, 301, 17)
        g = Graph(len(off) - 1, off, nbr)
        model, t32 = model_of(orc, 0.2)
        full_parity(orc, ctx, g, model, t32, 48, 777, 10)
    else:
        test_tiny_corpus_parity(orc, ctx, i)
    assert ctx.pacim_get_stats()["store"] == 0


@pytest.mark.parametrize("narrow", ["1", "0"])
@pytest.mark.parametrize("R", [1, 31, 32, 33, 64, 65, 100, 128, 129])
def test_gain_narrow_store(orc, ctx, R, narrow, monkeypatch):
    """gain0 of narrow dense stores (B <= 128 slots: S = 1, 2, 4 slots per
    lane, 32 / S rows per warp iteration, row sums through shared memory)
    against the oracle, and the generic kernel (PACIM_GAIN_NARROW=0)."""
    from oracle.oracle import Graph
    monkeypatch.setenv("PACIM_STORE", "dense")
    monkeypatch.setenv("PACIM_GAIN_NARROW", narrow)
    off, nbr = inputs.random_powerlaw_graph(3000, 20000, 61)
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, 0.1)
    full_parity(orc, ctx, g, model, t32, R, 900 + R, 8)


@pytest.mark.parametrize("hl", ["1", "0", "40"])
@pytest.mark.parametrize("bits", ["1", "2", "6"])
@pytest.mark.parametrize("i", [0, 3, 7, 9, 10, 12])
def test_dense_store_slot_epochs(orc, ctx, i, bits, hl, monkeypatch):
    """Slot epochs of the dense store (no reset pass between builds; a full
    reset every 2^bits builds): a run of builds with changing hash seeds —
    through the epoch wrap — each equal to the oracle (labels of every
    sketch, gain0, seeds and gains), and a repeated selection on the last.
    hl: the compression reads k_edges' hook list (the non-root slots) from
    the second build on (1, the default; not case 9, whose sketches are
    dense in non-roots), never (0), or the list overflows its capacity (40:
    the compression streams the store instead, decided on the device)."""
    monkeypatch.setenv("PACIM_STORE", "dense")
    monkeypatch.setenv("PACIM_EPOCH_BITS", bits)
    monkeypatch.setenv("PACIM_HOOKLIST", hl)
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    k = min(k, g.n)
    load_host(ctx, g, model, t32)
    for t in range(5):
        seed = 4000 + 7 * i + t
        ctx.pacim_build_sketches(R, seed)
        st = ctx.pacim_get_stats()
        assert st["store"] == 0
        # (the first build of a load may already use the list when the last
        # graph loaded had the same shape: the hints survive such reloads)
        want = hl == "1" and i != 9 and R >= 16
        if t >= 1 or not want:
            assert st["build_hook_list"] == int(want), (t, st["build_hook_list"])
        for r in range(R):
            lab, _ = orc.sketch_labels(g, model, t32, seed, r)
            assert np.array_equal(ctx.pacim_get_labels(r), lab), (t, r)
        es, egn, esg, eg0 = orc.greedy(g, model, t32, R, seed, k, want_gain0=True)
        assert np.array_equal(ctx.pacim_get_gain0(), eg0), t
        for rep in range(2 if t == 4 else 1):
            s, gn, sg, _ = ctx.pacim_select_seeds(k)
            assert list(s) == list(es) and list(gn) == list(egn), (t, rep)


@pytest.mark.parametrize("env", [{}, {"PACIM_NO_HOT": "1"}, {"PACIM_NO_HOT": "1", "PACIM_BIG_T": "30"}])
def test_compact_store_hot_and_dense_cover(orc, ctx, env, monkeypatch):
    """The hub's CCs (hot: no member lists, covered by the build's hot sums),
    and CCs above the list limit covered by the dense pass over the entries:
    the oracle's greedy either way."""
    monkeypatch.setenv("PACIM_STORE", "compact")
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    test_tiny_corpus_parity(orc, ctx, 12)
    st = ctx.pacim_get_stats()
    assert st["store"] == 1
    if not env:
        assert st["select_hotsum_steps"] >= 1
    elif "PACIM_BIG_T" in env:
        assert st["select_dense_steps"] >= 1


@pytest.mark.parametrize("pl", ["0", "64"])
@pytest.mark.parametrize("i", [0, 2, 3, 7, 10, 12])
def test_compact_store_pair_list_modes(orc, ctx, i, pl, monkeypatch):
    """The compact store's union pass without the mask pass's pair list
    (PACIM_CS_PAIRLIST=0: every edge hashed again) and with a list too small
    for the live pairs (64: overflow, the full pass runs instead): the same
    oracle parity and the same live-pair count as the default list."""
    monkeypatch.setenv("PACIM_STORE", "compact")
    test_tiny_corpus_parity(orc, ctx, i)
    live = ctx.pacim_get_stats()["live_pairs"]
    monkeypatch.setenv("PACIM_CS_PAIRLIST", pl)
    test_tiny_corpus_parity(orc, ctx, i)
    st = ctx.pacim_get_stats()
    assert st["live_pairs"] == live
    assert st["store"] == 1 or st["nnonsingle"] > 0.5 * st["rows"] * st["R_local"]


@pytest.mark.parametrize("i", [0, 2, 3, 7, 10, 12])
def test_compact_store_used(orc, ctx, i, monkeypatch):
    """The compact store's entries are exactly the non-singleton (vertex,
    sketch) pairs of the oracle's labels, its roots the CCs of >= 2."""
    monkeypatch.setenv("PACIM_STORE", "compact")
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    full_parity(orc, ctx, g, model, t32, R, 1000 + i, min(k, g.n), check_labels=False)
    st = ctx.pacim_get_stats()
    assert st["store"] == 1
    nons = 0
    roots = 0
    for r in range(R):
        lab, size = orc.sketch_labels(g, model, t32, 1000 + i, r)
        nons += int((size > 1).sum())
        roots += int(((size > 1) & (lab == np.arange(g.n))).sum())
    assert st["nnonsingle"] == nons and st["ncomp"] == roots


@pytest.mark.parametrize("i", [0, 2, 3, 5, 7, 9, 10])
def test_dense_cover_path(orc, ctx, i, monkeypatch):
    """Force components of >= 8 vertices out of the member index so MarkSeed
    covers them with the dense pass over the store (the path big components
    take at full scale)."""
    monkeypatch.setenv("PACIM_BIG_T", "8")
    test_tiny_corpus_parity(orc, ctx, i)


@pytest.mark.parametrize("env", [
    {"PACIM_NO_WARP_BFS": "1"},                        # every CC through the queue
    {"PACIM_NO_WARP_BFS": "1", "PACIM_CHUNK": "2"},    # rows split into 2-edge chunk items
    {"PACIM_CHUNK": "3", "PACIM_BIG_T": "40"},         # all three cover paths mixed
    {"PACIM_NO_WARP_BFS": "1", "PACIM_HUB_DEG": "4", "PACIM_FORCE_HLA": "1"},  # hubs via live lists
    {"PACIM_HUB_DEG": "2", "PACIM_FORCE_HLA": "1", "PACIM_CHUNK": "5"},
])
@pytest.mark.parametrize("i", [0, 2, 3, 7, 8, 9, 11])
def test_traversal_paths(orc, ctx, i, env, monkeypatch):
    """The shared traversal of the cover step (row items and chunk items of
    the work queue) of the dense store, forced on the tiny corpus by shrinking
    the chunk size and disabling the warp-local BFS; must give the oracle's
    greedy."""
    monkeypatch.setenv("PACIM_STORE", "dense")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    test_tiny_corpus_parity(orc, ctx, i)


@pytest.mark.parametrize("budget", ["1000", "6000", "40000"])
@pytest.mark.parametrize("i", [0, 1, 2, 5, 7, 9])
def test_window_layout(orc, ctx, i, budget, monkeypatch):
    """Store split into slot windows (one bucket of sketches, or a slice of
    one, at a time over the bucket's edges) -- the layout the L2-resident
    build uses at c2 -- forced on the tiny corpus with a small budget: labels,
    gain0 and the greedy must equal the oracle's, also with the dense pass."""
    monkeypatch.setenv("PACIM_L2_BUDGET", budget)
    test_tiny_corpus_parity(orc, ctx, i)
    monkeypatch.setenv("PACIM_BIG_T", "10")
    test_tiny_corpus_parity(orc, ctx, i)


@pytest.mark.parametrize("i", [0, 2, 3, 5, 7, 8, 10])
def test_decorrelated_rule(orc, ctx, i):
    """NEXT f3, R20: sketches sampled with live <=> hi32(mix64(hash(r) ^
    hash(e))) < T32 (every sketch a candidate for every edge): labels, gain0
    and the greedy equal the oracle's with the same rule."""
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    ctx.pacim_set_hash_rule(1)
    try:
        load_host(ctx, g, model, t32)
        ctx.pacim_build_sketches(R, 2000 + i)
        s, gn, sg, _ = ctx.pacim_select_seeds(min(k, g.n))
        es, egn, esg, eg0 = orc.greedy(g, model | orc.DECOR, t32, R, 2000 + i, min(k, g.n),
                                       want_gain0=True)
        assert np.array_equal(ctx.pacim_get_gain0(), eg0)
        for r in range(0, R, max(1, R // 8)):
            lab, _ = orc.sketch_labels(g, model | orc.DECOR, t32, 2000 + i, r)
            assert np.array_equal(ctx.pacim_get_labels(r), lab), r
        assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    finally:
        ctx.pacim_set_hash_rule(0)


def test_edge_cases(orc, ctx, pc):
    from oracle.oracle import Graph
    # single vertex, no edges, k = n = 1
    off, nbr = inputs.csr_from_edges(1, [])
    full_parity(orc, ctx, Graph(1, off, nbr), 0, 1 << 31, 3, 1, 1)
    # edgeless graph: every CC a singleton, gains R, seeds 0..k-1
    off, nbr = inputs.csr_from_edges(64, [])
    s, gn = full_parity(orc, ctx, Graph(64, off, nbr), 0, 1 << 32, 9, 2, 64)
    assert list(s) == list(range(64)) and set(gn) == {9}
    # k = n on a small graph (gains reach 0; smallest-id non-seed rule)
    off, nbr = inputs.random_graph(40, 60, 9)
    full_parity(orc, ctx, Graph(40, off, nbr), 0, orc.t32_const(0.6), 12, 3, 40)
    # errors surface as exceptions, never silent
    with pytest.raises(pc.PacimError):
        ctx.pacim_select_seeds(0)
    bad_off = np.array([0, 1, 2], np.uint64)
    with pytest.raises(pc.PacimError):
        ctx.pacim_load_graph(bad_off, np.array([1, 1], np.uint32), 0, 1, 1)  # self loop at 1
    with pytest.raises(pc.PacimError):
        ctx.pacim_build_sketches(4, 1)  # graph dropped by the failed load -> ESTATE
    with pytest.raises(pc.PacimError):  # asymmetric CSR
        ctx.pacim_load_graph(np.array([0, 1, 1], np.uint64), np.array([1], np.uint32), 0, 1, 2)


def upper_of(off, nbr):
    """The upper CSR (row u keeps its neighbours > u) of a symmetric CSR."""
    off = np.asarray(off, np.int64)
    nbr = np.asarray(nbr, np.uint32)
    n = len(off) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    keep = nbr.astype(np.int64) > rows
    uoff = np.zeros(n + 1, np.uint64)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=uoff[1:])
    return uoff, nbr[keep]


@pytest.mark.parametrize("mode", ["sync", "async"])
@pytest.mark.parametrize("i", range(len(CASES)))
def test_upper_csr_load(orc, ctx, i, mode):
    """H0 from the upper CSR (pacim_load_graph_upper[_async]: each edge once,
    the device builds the symmetric CSR — the transpose by a target
    histogram, atomic cursors and a segmented sort): exactly the symmetric CSR
    (pacim_get_graph), then the oracle's greedy on it."""
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    uo, un = upper_of(off, nbr)
    if mode == "sync":
        ctx.pacim_load_graph_upper(uo, un, model, t32, 1)
    else:
        ctx.pacim_load_graph_upper_async(uo, un, model, t32)
    seed = 1500 + i
    ctx.pacim_build_sketches(R, seed)  # commits an asynchronous load
    o2, n2 = ctx.pacim_get_graph()
    assert np.array_equal(o2, np.asarray(off, np.uint64)) and np.array_equal(n2, np.asarray(nbr, np.uint32))
    s, gn, sg, _ = ctx.pacim_select_seeds(min(k, g.n))
    es, egn, esg, eg0 = orc.greedy(g, model, t32, R, seed, min(k, g.n), want_gain0=True)
    assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    assert np.array_equal(ctx.pacim_get_gain0(), eg0)


@pytest.mark.parametrize("ucsr", ["0", "1", "4"])
@pytest.mark.parametrize("sel", [0, 1, 2])
@pytest.mark.parametrize("i", [0, 3, 7, 10, 12])
def test_upper_load_deferred_sym(orc, ctx, i, sel, ucsr, monkeypatch):
    """An upper-loaded graph keeps the upper CSR and the symmetric offsets;
    its symmetric neighbour lists are built only when something reads them
    (pc_ensure_sym).  Without pacim_get_graph first: the build (edge lists or
    the upper-edge stream) and every selector — incremental (cover
    traversal: builds the lists), prefix doubling, Win-Tree — equal the
    oracle; then a compressed build (probes: lists), Monte Carlo, and the
    symmetric CSR read back."""
    from oracle.oracle import Graph
    monkeypatch.setenv("PACIM_STORE", "dense")
    monkeypatch.setenv("PACIM_UCSR", ucsr)
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    uo, un = upper_of(off, nbr)
    if i % 2:
        ctx.pacim_load_graph_upper(uo, un, model, t32, 1)
    else:
        ctx.pacim_load_graph_upper_async(uo, un, model, t32)
    k = min(k, g.n)
    seed = 2500 + i
    ctx.pacim_set_selector(sel)
    try:
        ctx.pacim_build_sketches(R, seed)
        s, gn, sg, _ = ctx.pacim_select_seeds(k)
    finally:
        ctx.pacim_set_selector(0)
    es, egn, esg, eg0 = orc.greedy(g, model, t32, R, seed, k, want_gain0=True)
    assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    assert np.array_equal(ctx.pacim_get_gain0(), eg0)
    if sel == 0:
        ctx.pacim_build_sketches(R, seed, 1 << 30)  # alpha = 1/4: Get-center probes
        s2, gn2, _, _ = ctx.pacim_select_seeds(k)
        assert list(s2) == list(es) and list(gn2) == list(egn)
        seeds = [0, g.n // 2]
        assert ctx.pacim_simulate_ic(seeds, 5, 9) == orc.simulate_ic(g, model, t32, seeds, 5, 9)
    o2, n2 = ctx.pacim_get_graph()
    assert np.array_equal(o2, np.asarray(off, np.uint64)) and np.array_equal(n2, np.asarray(nbr, np.uint32))


@pytest.mark.parametrize("ucsr", [None, "1", "4"])
def test_upper_csr_load_edge_cases(orc, ctx, pc, ucsr, monkeypatch):
    """Upper loads: no edges, isolated vertices between and after the edges,
    a hub whose lower list spans many chunks, and invalid upper CSRs (an entry
    v <= u, unsorted rows, v >= n, offsets[n] != m) raise — with each form of
    the build's edge stream."""
    from oracle.oracle import Graph
    if ucsr:
        monkeypatch.setenv("PACIM_UCSR", ucsr)
    ctx.pacim_load_graph_upper(np.zeros(9, np.uint64), np.zeros(0, np.uint32), 0, 1 << 31, 1)
    o2, n2 = ctx.pacim_get_graph()
    assert list(o2) == [0] * 9 and len(n2) == 0
    # vertex 3000 adjacent to every even vertex below it (its lower list: 1500
    # entries), isolated odd vertices, a tail of isolated vertices
    edges = [(v, 3000) for v in range(0, 3000, 2)] + [(v, v + 2) for v in range(0, 2990, 6)]
    off, nbr = inputs.csr_from_edges(3100, edges)
    uo, un = upper_of(off, nbr)
    ctx.pacim_load_graph_upper(uo, un, 0, orc.t32_const(0.3), 1)
    o2, n2 = ctx.pacim_get_graph()
    assert np.array_equal(o2, np.asarray(off, np.uint64)) and np.array_equal(n2, np.asarray(nbr, np.uint32))
    ctx.pacim_build_sketches(16, 5)
    s, gn, _, _ = ctx.pacim_select_seeds(5)
    es, egn, _, _ = orc.greedy(Graph(3100, off, nbr), 0, orc.t32_const(0.3), 16, 5, 5)
    assert list(s) == list(es) and list(gn) == list(egn)
    for bad_off, bad_nbr in [([0, 1, 1], [0]),          # v == u
                             ([0, 2, 2, 2], [2, 1]),    # unsorted row
                             ([0, 1, 1], [5]),          # v >= n
                             ([0, 1, 2], [1, 2])]:      # row 1: 2 >= n
        with pytest.raises(pc.PacimError):
            ctx.pacim_load_graph_upper(np.array(bad_off, np.uint64), np.array(bad_nbr, np.uint32),
                                       0, 1 << 31, 1)
    with pytest.raises(pc.PacimError):  # offsets[n] != m
        ctx.pacim_load_graph_upper(np.array([0, 2, 2], np.uint64), np.array([1], np.uint32),
                                   0, 1 << 31, 1)


def test_upper_csr_load_c2(ctx):
    """The full c2 graph through the upper load: the device-built symmetric
    CSR equals the generated one (sha256 of both arrays)."""
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config("c2")
    pipeline.generate(ctx, cfg)
    off, nbr = ctx.pacim_get_graph()
    h = (sha(off), sha(nbr))
    uo, un = upper_of(off, nbr)
    assert len(un) * 2 == len(nbr)
    ctx.pacim_load_graph_upper(uo, un, *pipeline.model_of(cfg), 1)
    o2, n2 = ctx.pacim_get_graph()
    assert (sha(o2), sha(n2)) == h


@pytest.mark.parametrize("ucsr", [None, "1", "4"])
@pytest.mark.parametrize("p", [0.4, "wic", ("unif", 0.2, 0.6)])
def test_load_derivation_shapes(orc, ctx, p, ucsr, monkeypatch):
    """The load's edge pass (rows of CSR entries from the 32-entry chunk
    table, one packed (degree, row + hub flag) gather per entry) on shapes
    that stress it: isolated vertices between and after the edges, a hub whose
    list spans several chunks next to degree-1 rows, a chunk starting inside a
    row; and an edgeless graph.  Labels, gain0 and the greedy equal the
    oracle's under the constant, WIC and Uniform models — with each form of
    the build's edge stream (ucsr: default lists, the stream, CSR-direct)."""
    from oracle.oracle import Graph
    if ucsr:
        monkeypatch.setenv("PACIM_UCSR", ucsr)
    model, t32 = model_of(orc, p)
    n = 300
    edges = [(0, v) for v in range(5, 300, 2)] + [(7, 9), (11, 13), (250, 251), (3, 290)]
    off, nbr = inputs.csr_from_edges(n, edges)
    assert off[1] > 64 and (np.diff(off.astype(np.int64)) == 0).sum() > 100
    full_parity(orc, ctx, Graph(n, off, nbr), model, t32, 16, 77, 6)
    off, nbr = inputs.csr_from_edges(40, [])
    full_parity(orc, ctx, Graph(40, off, nbr), model, t32, 5, 78, 4)


@pytest.mark.parametrize("big_t,ucsr", [(None, None), ("8", None), (None, "1"), (None, "4")])
@pytest.mark.parametrize("R,p", [(1000, 0.02), (1023, 0.1), (520, "wic")])
def test_many_sketches(orc, ctx, R, p, big_t, ucsr, monkeypatch):
    """R above 256 on one GPU (several 256-slot blocks per store row, up to
    1024 slots, odd counts): labels of sampled sketches, gain0 and the greedy
    equal the oracle's, also with the dense pass forced."""
    from oracle.oracle import Graph
    if big_t:
        monkeypatch.setenv("PACIM_BIG_T", big_t)
    if ucsr:
        monkeypatch.setenv("PACIM_UCSR", ucsr)
    off, nbr = inputs.random_powerlaw_graph(600, 2400, 31)
    g = Graph(600, off, nbr)
    model, t32 = model_of(orc, p)
    load_host(ctx, g, model, t32)
    ctx.pacim_build_sketches(R, 41)
    s, gn, sg, _ = ctx.pacim_select_seeds(12)
    es, egn, esg, eg0 = orc.greedy(g, model, t32, R, 41, 12, want_gain0=True)
    assert np.array_equal(ctx.pacim_get_gain0(), eg0)
    for r in (0, R // 2, R - 1):
        lab, _ = orc.sketch_labels(g, model, t32, 41, r)
        assert np.array_equal(ctx.pacim_get_labels(r), lab), r
    assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)


def test_too_many_sketches_fail_cleanly(ctx, pc):
    """More local sketches than the selection supports: an error, never a
    wrong answer."""
    off, nbr = inputs.random_graph(100, 300, 3)
    ctx.pacim_load_graph(off, nbr, 0, 1 << 30, 1)
    try:
        ctx.pacim_build_sketches(2048, 1)
        ctx.pacim_select_seeds(3)
    except pc.PacimError:
        return
    raise AssertionError("R = 2048 on one GPU must be rejected")


def test_hot_sums_dense_step(orc, ctx, monkeypatch):
    """The hub (a star's center) chosen first with its CCs above the dense
    threshold in every sketch: the select covers them from the build's
    per-vertex hot sums (one vector pass, no dense pass over the store); the
    greedy equals the oracle's, and a second selection repeats it."""
    from oracle.oracle import Graph
    monkeypatch.setenv("PACIM_BIG_T", "8")
    off, nbr = inputs.star_graph(50)
    g = Graph(len(off) - 1, off, nbr)
    full_parity(orc, ctx, g, 0, orc.t32_const(0.3), 64, 1008, 4)
    assert ctx.pacim_get_stats()["select_hotsum_steps"] == 1
    s, gn, sg, _ = ctx.pacim_select_seeds(4)
    es, egn, esg, _ = orc.greedy(g, 0, orc.t32_const(0.3), 64, 1008, 4)
    assert list(s) == list(es) and list(gn) == list(egn)


@pytest.mark.parametrize("R,gr", [(100, "2"), (37, "2"), (256, "4"), (100, "0")])
def test_hot_gain_pass_ragged(orc, ctx, monkeypatch, R, gr):
    """The gain pass with hot sums (register-cached hot roots, B <= 256) on
    a ragged sketch count and an odd row count, giant hot CCs in some slots
    only (PACIM_BIG_T = 765 between the slots' hub CC sizes): gain0, labels and the
    greedy equal the oracle's for both row groupings and the generic kernel."""
    from oracle.oracle import Graph
    monkeypatch.setenv("PACIM_BIG_T", "765")
    monkeypatch.setenv("PACIM_GAIN_HOT", gr)
    off, nbr = inputs.random_powerlaw_graph(2001, 9000, 21)
    g = Graph(2001, off, nbr)
    hub = int(np.argmax(np.diff(off)))
    sizes = []
    for r in range(R):  # the hub's CC per sketch: giant in some slots only
        lab, _ = orc.sketch_labels(g, 0, orc.t32_const(0.12), 77, r)
        sizes.append(int(np.sum(lab == lab[hub])))
    assert min(sizes) <= 765 < max(sizes), (min(sizes), max(sizes))
    full_parity(orc, ctx, g, 0, orc.t32_const(0.12), R, 77, 12, check_labels=R <= 100)


def test_determinism(orc, ctx):
    from oracle.oracle import Graph
    off, nbr = inputs.random_powerlaw_graph(3000, 20000, 11)
    g = Graph(3000, off, nbr)
    load_host(ctx, g, 0, orc.t32_const(0.1))
    ctx.pacim_build_sketches(128, 5)
    a = ctx.pacim_select_seeds(20)
    b = ctx.pacim_select_seeds(20)  # repeated select restarts from S = empty
    ctx.pacim_build_sketches(128, 5)
    c = ctx.pacim_select_seeds(20)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    for x, y in zip(a, c):
        assert np.array_equal(x, y)


# ------------------------------------------------------------- generators
@pytest.mark.parametrize("name,over", [
    ("c1", {}),
    ("c2", {"scale": 14, "ef": 16}),
    ("c4", {"scale": 13, "ef": 24}),
    ("c5", {"scale": 13, "ef": 32}),
    ("c3", {"W": 300, "H": 200}),
])
def test_generator_matches_oracle(orc, ctx, name, over):
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config(name, **over)
    n, m = pipeline.generate(ctx, cfg)
    g = orc.gen_config(cfg)
    assert (n, m) == (g.n, g.m)
    off, nbr = ctx.pacim_get_graph()
    assert np.array_equal(off, g.off)
    assert np.array_equal(nbr, g.nbr)


@pytest.mark.parametrize("name,over,buckets", [
    ("c2", {"scale": 14, "ef": 16}, "4"),
    ("c4", {"scale": 13, "ef": 24}, "8"),
    ("c5", {"scale": 13, "ef": 32}, "2"),
    ("c5", {"scale": 15, "ef": 32}, "16"),
])
def test_bucketed_generator_matches_oracle(orc, ctx, name, over, buckets, monkeypatch):
    """The source-bucketed R-MAT generator (the one that builds c5 at full
    scale) gives the oracle's CSR bit for bit."""
    monkeypatch.setenv("PACIM_GEN_BUCKETS", buckets)
    test_generator_matches_oracle(orc, ctx, name, over)


@pytest.mark.parametrize("upper", ["1", "0"])
@pytest.mark.parametrize("i", [0, 1, 2, 5, 6, 7, 8, 9, -1])
def test_lean_graph(orc, ctx, i, upper, monkeypatch):
    """Lean graphs (no edge list, rows = vertex ids, k_edges over the CSR):
    labels, gain0 and the greedy equal the oracle's (constant p).  upper:
    the pass visits the upper entries only (by the upper offsets, the
    default) or every CSR entry, dropping the lower ones (0).  i = -1: runs
    of isolated vertices longer than the row search's linear steps."""
    monkeypatch.setenv("PACIM_LEAN", "1")
    monkeypatch.setenv("PACIM_LEAN_UPPER", upper)
    if i < 0:
        from oracle.oracle import Graph
        off, nbr = gapped_graph(300, 2400, 301, 18)
        g = Graph(len(off) - 1, off, nbr)
        model, t32 = model_of(orc, 0.2)
        full_parity(orc, ctx, g, model, t32, 48, 778, 10)
    else:
        test_tiny_corpus_parity(orc, ctx, i)
    st = ctx.pacim_get_stats()
    assert st["rows"] == st["n"]


def test_c1_full(orc, ctx):
    """BASELINE.json configs[0] end to end: generated on the GPU, all 64
    sketches' labels, gain0, seeds, gains, sigma vs the oracle."""
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config("c1")
    pipeline.generate(ctx, cfg)
    g = orc.gen_config(cfg)
    model, t32 = orc.model_args(cfg)
    ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"])
    s, gn, sg, _ = ctx.pacim_select_seeds(cfg["k"])
    es, egn, esg, eg0 = orc.greedy(g, model, t32, cfg["R"], cfg["hash_seed"], cfg["k"], True)
    assert np.array_equal(ctx.pacim_get_gain0(), eg0)
    for r in range(cfg["R"]):
        assert np.array_equal(ctx.pacim_get_labels(r), orc.sketch_labels(g, model, t32, 1, r)[0])
    assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    gold = json.load(open(os.path.join(GOLD, "c1.json")))
    assert list(s) == gold["seeds"] and list(gn) == gold["gain_num"]


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_config_golden(ctx, name):
    """Full-size configs[1], configs[2] (launch configuration of bench.py)
    against golden files written by tests/golden/make_golden.py (oracle only)."""
    path = os.path.join(GOLD, f"{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    gold = json.load(open(path))
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config(name)
    n, m = pipeline.generate(ctx, cfg)
    assert (n, m) == (gold["n"], gold["m"])
    off, nbr = ctx.pacim_get_graph()
    assert sha(off) == gold["off_sha256"] and sha(nbr) == gold["nbr_sha256"]
    ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"])
    s, gn, sg, _ = ctx.pacim_select_seeds(cfg["k"])
    assert list(s) == gold["seeds"]
    assert list(gn) == gold["gain_num"]
    assert list(sg) == gold["sigma_num"]
    g0 = ctx.pacim_get_gain0()
    assert sha(g0) == gold["gain0_sha256"]
    for r, h in gold["label_sha256"].items():
        assert sha(ctx.pacim_get_labels(int(r))) == h, r
    st = ctx.pacim_get_stats()
    assert st["nmember"] + (n * cfg["R"] - st["nmember"]) == n * cfg["R"]


def test_c4_full_scale_certified(orc, ctx):
    """BASELINE.json configs[3] at full size (n = 2^26, m = 1.57e9, WIC, R =
    256, k = 100) in bench.py's launch configuration: the generated CSR and
    two sketches' canonical labels against the oracle's golden digests, then
    the GPU's whole greedy sequence (seeds AND per-step gains) CERTIFIED by
    the oracle's verify mode (GeneralGreedy P:396-401, Alg. 1
    P:524-530): a passing sequence is exactly derive mode's output."""
    path = os.path.join(GOLD, "c4.json")
    gold = json.load(open(path))
    from oracle.oracle import Graph
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config("c4")
    n, m = pipeline.generate(ctx, cfg)
    assert (n, m) == (gold["n"], gold["m"])
    off, nbr = ctx.pacim_get_graph()
    assert sha(off) == gold["off_sha256"] and sha(nbr) == gold["nbr_sha256"]
    ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"])
    for r, h in gold["label_sha256"].items():
        lab = ctx.pacim_get_labels(int(r))
        assert sha(lab) == h, r
        roots = lab == np.arange(n, dtype=np.uint32)
        sz = np.bincount(lab, minlength=n)[lab]
        st = gold["cc_stats"][r]
        assert int(roots.sum()) == st["ncc"] and int((sz > 1).sum()) == st["nonsingleton"]
        del lab, roots, sz
    s, gn, sg, _ = ctx.pacim_select_seeds(cfg["k"])
    assert list(sg) == list(np.cumsum(gn))
    g = Graph(n, off, nbr)
    model, t32 = orc.model_args(cfg)
    rc, info = orc.verify(g, model, t32, cfg["R"], cfg["hash_seed"], s, gn)
    assert rc == 0, (orc.VERIFY_RC[rc], info)
    assert info[3] == sg[-1]          # Σ_r |∪_i C_r(s_i)| = N(S_k)


@pytest.mark.parametrize("form", ["direct"])
def test_c5_shape_scale25_certified(orc, ctx, form, monkeypatch):
    """BASELINE.json configs[4]'s generator and method (web R-MAT .6/.15/.15/.1,
    ef 32, p = 0.01, R = 256, compressed alpha = 1/16, k = 100) at scale 25
    (n = 2^25): the full-size c5 CSR (58 GB) does not fit the oracle's host,
    so SURVEY 8(c)'s fallback scale is used.  The GPU's CSR equals the
    oracle generator's (golden digest, tests/golden/c5_s25_graph.json), and
    the GPU's seeds and gains are certified by the oracle's verify mode.
    form "direct": the path c5 takes at full scale (the CSR-direct edge form
    — no edge lists, rows by the rank map — and the source-bucketed
    generator); the lean layout (rows = vertex ids) is covered by the small
    lean tests."""
    path = os.path.join(GOLD, "c5_s25_graph.json")
    gold = json.load(open(path))
    lean = False
    if form == "direct":
        monkeypatch.setenv("PACIM_UCSR", "4")
        monkeypatch.setenv("PACIM_GEN_BUCKETS", "8")
    from oracle.oracle import Graph
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config("c5", scale=25)
    n, m = pipeline.generate(ctx, cfg)
    assert (n, m) == (gold["n"], gold["m"])
    off, nbr = ctx.pacim_get_graph()
    assert sha(off) == gold["off_sha256"] and sha(nbr) == gold["nbr_sha256"]
    s, gn, sg, _ = pipeline.run(ctx, cfg)
    st = ctx.pacim_get_stats()
    assert st["compressed"] == 1 and st["rho"] < n // 8
    assert bool(st["lean"]) == lean
    g = Graph(n, off, nbr)
    model, t32 = orc.model_args(cfg)
    rc, info = orc.verify(g, model, t32, cfg["R"], cfg["hash_seed"], s, gn)
    assert rc == 0, (orc.VERIFY_RC[rc], info)
    assert info[3] == sg[-1]


# ------------------------------------------------ multi-rank primitives
@pytest.mark.parametrize("big_t,chunk", [(None, None), ("6", None), (None, "3")])
def test_rank_emulation_matches_single(orc, pc, big_t, chunk, monkeypatch):
    """Sketch sharding r = rank mod P with the per-step primitives, ranks run
    one after another on one GPU (no waiting kernels), the collective replaced
    by a host sum: identical to the single-ctx greedy."""
    if big_t:
        monkeypatch.setenv("PACIM_BIG_T", big_t)
    if chunk:
        monkeypatch.setenv("PACIM_CHUNK", chunk)
        monkeypatch.setenv("PACIM_HUB_DEG", "6")
        monkeypatch.setenv("PACIM_FORCE_HLA", "1")
        monkeypatch.setenv("PACIM_NO_WARP_BFS", "1")
    from oracle.oracle import Graph
    from paper_2311_07554_b200 import dist
    off, nbr = inputs.random_powerlaw_graph(3000, 15000, 21)
    g = Graph(3000, off, nbr)
    t32 = orc.t32_const(0.08)
    R, seed, k = 48, 7, 15
    es, egn, esg, _ = orc.greedy(g, 0, t32, R, seed, k)
    for P in (2, 3):
        ctxs = []
        for rank in range(P):
            c = pc.Context(0)
            c.pacim_load_graph(off, nbr, 0, t32, 1)
            c.pacim_build_sketches(R, seed, 1 << 32, rank, P)
            ctxs.append(c)
        for mode, cap in (("sparse", None), ("dense", None), ("sparse", 40)):
            for c in ctxs:
                c.pacim_select_reset()
            seeds, gains, sig = dist.emulated_select(ctxs, g.n, k, device="cuda", cap=cap,
                                                     mode=mode)
            assert list(seeds) == list(es) and list(gains) == list(egn), (mode, cap)
            assert list(sig) == list(esg)
        for c in ctxs:
            c.close()


# ------------------------------------------------ Monte-Carlo sigma (f3)
@pytest.mark.parametrize("i,nsims", [(0, 300), (3, 600), (8, 257), (10, 64), (11, 513), (6, 100)])
def test_simulate_ic_equals_oracle(orc, ctx, i, nsims):
    """R21: the GPU's multi-simulation BFS reaches exactly the oracle's total
    over the same counter-based worlds (const, WIC and Uniform models; batch
    tails of 1..31 simulations; repeated seed ids)."""
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    load_host(ctx, g, model, t32)
    seeds = [0, min(5, g.n - 1), g.n // 2, 0]
    got = ctx.pacim_simulate_ic(seeds, nsims, 31 + i)
    assert got == orc.simulate_ic(g, model, t32, sorted(set(seeds)), nsims, 31 + i)


# ------------------------------------------------------ lazy selector (f2)
@pytest.mark.parametrize("i", [0, 2, 3, 5, 6, 7, 9, 10])
def test_lazy_selector_equals_oracle(orc, ctx, i):
    """NEXT f2: the lazy selector (stale bounds, prefix-doubling evaluations)
    returns GeneralGreedy's sequence (R17), and never evaluates fewer than k
    candidates nor more than k * n."""
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    k = min(k, g.n)
    load_host(ctx, g, model, t32)
    ctx.pacim_build_sketches(R, 3000 + i)
    ctx.pacim_set_selector(1)
    try:
        s, gn, sg, _ = ctx.pacim_select_seeds(k)
        st = ctx.pacim_get_stats()
        s2, gn2, _, _ = ctx.pacim_select_seeds(k)  # repeated: restarts from S = empty
    finally:
        ctx.pacim_set_selector(0)
    es, egn, esg, _ = orc.greedy(g, model, t32, R, 3000 + i, k)
    assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    assert list(s2) == list(es) and list(gn2) == list(egn)
    assert k - 1 <= st["select_evaluations"] <= k * g.n
    s3, gn3, _, _ = ctx.pacim_select_seeds(k)  # the incremental selector on the same store
    assert list(s3) == list(es)


def test_load_graph_async(orc, ctx):
    """Pipelined loads (pacim_load_graph_async): two graphs enqueued, each
    committed by the build that follows; results equal the oracle's, and a
    third pending load is rejected (ESTATE) while two are in flight."""
    import torch
    from oracle.oracle import Graph
    from paper_2311_07554_b200 import PacimError
    gs = [inputs.random_powerlaw_graph(900, 4000, 71), inputs.random_graph(700, 2500, 72)]
    pinned = []
    for off, nbr in gs:
        po = torch.from_numpy(off.astype(np.uint64)).pin_memory().numpy()
        pn = torch.from_numpy(nbr.astype(np.uint32)).pin_memory().numpy()
        pinned.append((po, pn))
    t32 = orc.t32_const(0.1)
    ctx.pacim_load_graph_async(*pinned[0], 0, t32)
    ctx.pacim_load_graph_async(*pinned[1], 0, t32)
    with pytest.raises(PacimError):
        ctx.pacim_load_graph_async(*pinned[0], 0, t32)
    for i, (off, nbr) in enumerate(gs):
        g = Graph(len(off) - 1, off, nbr)
        ctx.pacim_build_sketches(24, 80 + i)  # commits graph i
        assert ctx.pacim_graph_info() == (g.n, g.m)
        s, gn, sg, _ = ctx.pacim_select_seeds(6)
        es, egn, esg, eg0 = orc.greedy(g, 0, t32, 24, 80 + i, 6, want_gain0=True)
        assert np.array_equal(ctx.pacim_get_gain0(), eg0)
        assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    # a synchronous load discards pending ones
    ctx.pacim_load_graph_async(*pinned[0], 0, t32)
    off, nbr = gs[1]
    ctx.pacim_load_graph(off, nbr, 0, t32, 1)
    ctx.pacim_build_sketches(24, 81)
    assert ctx.pacim_graph_info() == (len(off) - 1, len(nbr) // 2)


def test_workspace_context(orc, pc):
    """pacim_create with a caller-owned (torch) workspace: every device buffer
    is carved from it; results equal the oracle's; a workspace too small for
    the build fails with ENOMEM (no silent cudaMalloc)."""
    import torch
    from oracle.oracle import Graph
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    c = pc.Context(0, workspace=ws)
    try:
        for i in (2, 3, 7):
            build_fn, p, R, k = CASES[i]
            off, nbr = build_fn()
            g = Graph(len(off) - 1, off, nbr)
            model, t32 = model_of(orc, p)
            full_parity(orc, c, g, model, t32, R, 1000 + i, min(k, g.n), check_labels=False)
            assert c.pacim_get_stats()["device_bytes"] <= ws.numel()
    finally:
        c.close()
    small = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    c = pc.Context(0, workspace=small)
    try:
        off, nbr = inputs.random_powerlaw_graph(4000, 30000, 8)
        with pytest.raises(pc.PacimError) as ei:
            c.pacim_load_graph(off, nbr, 0, orc.t32_const(0.05), 1)
            c.pacim_build_sketches(256, 1)
        assert ei.value.code == -2
    finally:
        c.close()


# ------------------------------------------------ sharded select in the library (NCCL)
def _dist_ctx(pc):
    from paper_2311_07554_b200 import pacim_nccl_unique_id
    c = pc.Context(0)
    c.pacim_init_comm(0, 1, pacim_nccl_unique_id())
    return c


@pytest.mark.parametrize("i,env", [
    (0, {}), (2, {}), (3, {}), (7, {}), (9, {}), (10, {}),
    (7, {"PACIM_DIST_CAP": "4"}),                  # list overflow -> robust replay
    (3, {"PACIM_STORE": "dense"}),                 # dense store: robust path
    (12, {}),                                      # the hub's CCs: all-reduced hot sums
    (12, {"PACIM_NO_HOT": "1", "PACIM_BIG_T": "50"}),  # list-less big CCs: replay
    (2, {"PACIM_BIG_T": "6"}),                     # big CCs that are not the hub's: replay
    (7, {"PACIM_DIST_ROBUST": "1"}),
])
def test_dist_select_world1(orc, pc, i, env, monkeypatch):
    """pacim_init_comm + pacim_select_seeds on a sharded build (dist.cu: NCCL
    all-reduce of gain0, per-step ncclAllGather of fixed-size delta lists, the
    robust dense all-reduce replay) at world 1 (one GPU here; PACIM_FORCE_DIST
    runs the sharded code): the oracle's greedy, seeds and gains."""
    monkeypatch.setenv("PACIM_FORCE_DIST", "1")
    monkeypatch.setenv("PACIM_STORE", "compact")  # the fast path's store (unless overridden)
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    k = min(k, g.n)
    c = _dist_ctx(pc)
    try:
        c.pacim_load_graph(g.off, g.nbr, model, t32, 1)
        c.pacim_build_sketches(R, 1000 + i, 1 << 32, 0, 1)
        es, egn, esg, eg0 = orc.greedy(g, model, t32, R, 1000 + i, k, want_gain0=True)
        assert np.array_equal(c.pacim_get_gain0(), eg0)
        for rep in range(2):  # repeated: the covered flags are restored
            s, gn, sg, _ = c.pacim_select_seeds(k)
            assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg), rep
        st = c.pacim_get_stats()
        if "PACIM_DIST_CAP" in env or "PACIM_NO_HOT" in env:
            assert st["select_dist_replays"] == 1
        elif i == 12 and not env:
            assert st["select_dist_replays"] == 0 and st["store"] == 1
    finally:
        c.close()


@pytest.mark.parametrize("i,env", [
    (0, {}), (2, {}), (3, {}), (7, {}), (9, {}), (10, {}), (12, {}),
    (7, {"PACIM_EP_CAP": "100"}),                  # pair list overflow: the pass repeated
    (12, {"PACIM_NO_HOT": "1", "PACIM_BIG_T": "50"}),
])
def test_dist_edge_partitioned_world1(orc, pc, i, env, monkeypatch):
    """The edge-partitioned sharded build (dist.cu pc_cs_ep_pairs: the rank's
    edge range against all sketches, pairs routed to the sketches' owners,
    the compact store built from the received pairs) at world 1 (PACIM_EP=1):
    labels of every sketch, gain0, the live-pair count of the mask-pass build,
    and the oracle's greedy through the NCCL select."""
    monkeypatch.setenv("PACIM_FORCE_DIST", "1")
    monkeypatch.setenv("PACIM_STORE", "compact")
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    k = min(k, g.n)
    c = _dist_ctx(pc)
    try:
        c.pacim_load_graph(g.off, g.nbr, model, t32, 1)
        c.pacim_build_sketches(R, 1000 + i, 1 << 32, 0, 1)
        live = c.pacim_get_stats()["live_pairs"]
        monkeypatch.setenv("PACIM_EP", "1")
        c.pacim_build_sketches(R, 1000 + i, 1 << 32, 0, 1)
        st = c.pacim_get_stats()
        assert st["live_pairs"] == live
        if st["store"] == 1:
            for r in range(R):
                lab, _ = orc.sketch_labels(g, model, t32, 1000 + i, r)
                assert np.array_equal(c.pacim_get_labels(r), lab), r
        es, egn, esg, eg0 = orc.greedy(g, model, t32, R, 1000 + i, k, want_gain0=True)
        assert np.array_equal(c.pacim_get_gain0(), eg0)
        s, gn, sg, _ = c.pacim_select_seeds(k)
        assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    finally:
        c.close()


def test_dist_select_world1_compressed(orc, pc, monkeypatch):
    """Compressed store (Alg. 3) under the sharded select: robust path."""
    monkeypatch.setenv("PACIM_FORCE_DIST", "1")
    from oracle.oracle import Graph
    off, nbr = inputs.random_powerlaw_graph(2000, 8000, 42)
    g = Graph(2000, off, nbr)
    t32 = orc.t32_const(0.05)
    c = _dist_ctx(pc)
    try:
        c.pacim_load_graph(off, nbr, 0, t32, 1)
        c.pacim_build_sketches(40, 5, 1 << 28, 0, 1)
        s, gn, sg, _ = c.pacim_select_seeds(10)
        es, egn, esg, _ = orc.greedy(g, 0, t32, 40, 5, 10)
        assert list(s) == list(es) and list(gn) == list(egn)
    finally:
        c.close()


# ------------------------------------------------ f2: Win-Tree and the CELF count
from tests.celf_ref import celf_reevaluations  # noqa: E402


@pytest.mark.parametrize("store", ["compact", "dense"])
@pytest.mark.parametrize("i", [0, 2, 3, 7, 8, 10, 12])
def test_wintree_selector_equals_oracle(orc, ctx, i, store, monkeypatch):
    """NEXT f2: the Win-Tree selector returns GeneralGreedy's
    sequence (R17) on both stores; its re-evaluations are at least one per
    step and at most k * n."""
    monkeypatch.setenv("PACIM_STORE", store)
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    k = min(k, g.n)
    load_host(ctx, g, model, t32)
    ctx.pacim_build_sketches(R, 3000 + i)
    ctx.pacim_set_selector(2)
    try:
        s, gn, sg, _ = ctx.pacim_select_seeds(k)
        st = ctx.pacim_get_stats()
        s2, gn2, _, _ = ctx.pacim_select_seeds(k)  # repeated: restarts from S = empty
    finally:
        ctx.pacim_set_selector(0)
    es, egn, esg, _ = orc.greedy(g, model, t32, R, 3000 + i, k)
    assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    assert list(s2) == list(es) and list(gn2) == list(egn)
    assert k <= st["select_evaluations"] <= k * g.n


@pytest.mark.parametrize("i", [0, 2, 3, 8, 12])
def test_celf_count_equals_celf(orc, ctx, i, monkeypatch):
    """The incremental selector's CELF counter (PACIM_CELF_COUNT=1) equals a
    literal heap-based CELF run on the oracle's sketches."""
    monkeypatch.setenv("PACIM_CELF_COUNT", "1")
    monkeypatch.setenv("PACIM_STORE", "compact")
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    k = min(k, g.n)
    load_host(ctx, g, model, t32)
    ctx.pacim_build_sketches(R, 4000 + i)
    s, gn, _, _ = ctx.pacim_select_seeds(k)
    labs, sizes = zip(*[orc.sketch_labels(g, model, t32, 4000 + i, r) for r in range(R)])
    cs, cg, reev = celf_reevaluations(labs, sizes, g.n, k)
    assert list(s) == cs and list(gn) == cg
    assert ctx.pacim_get_stats()["select_celf_evaluations"] == reev


@pytest.mark.parametrize("i", [3, 7])
def test_auto_selector(orc, ctx, i):
    """Selector 3 (auto): the Win-Tree under WIC, the incremental selector
    otherwise; GeneralGreedy's sequence either way."""
    from oracle.oracle import Graph
    build_fn, p, R, k = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    model, t32 = model_of(orc, p)
    load_host(ctx, g, model, t32)
    ctx.pacim_build_sketches(R, 5000 + i)
    ctx.pacim_set_selector(3)
    try:
        s, gn, sg, _ = ctx.pacim_select_seeds(k)
        st = ctx.pacim_get_stats()
    finally:
        ctx.pacim_set_selector(0)
    es, egn, esg, _ = orc.greedy(g, model, t32, R, 5000 + i, k)
    assert list(s) == list(es) and list(gn) == list(egn)
    assert (st["select_evaluations"] > 0) == (model == 1)
