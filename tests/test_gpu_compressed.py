"""GPU parity of the compressed store (H6c) and Get-center selection (H11)
against the oracle's Alg. 3 transcription and its greedy."""
import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


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


CASES = [
    # graph, p, R, k, a32
    (lambda: inputs.random_graph(300, 900, 41), 0.2, 16, 8, 1 << 28),
    (lambda: inputs.random_powerlaw_graph(2000, 8000, 42), 0.05, 64, 12, 1 << 28),
    (lambda: inputs.random_graph(3000, 9000, 43), 0.5, 8, 6, 1 << 28),      # giant CC > queue
    (lambda: inputs.random_graph(3000, 9000, 44), 0.5, 8, 6, 1 << 20),      # few centers: overflow
    (lambda: inputs.random_powerlaw_graph(1500, 9000, 45), "wic", 24, 10, 1 << 30),
    (lambda: inputs.random_graph(500, 1500, 46), 0.3, 12, 10, 0),           # alpha = 0: no centers
    (lambda: inputs.path_graph(700), 1.0, 4, 3, 1 << 27),
    (lambda: inputs.random_graph(400, 800, 47), 0.0, 5, 4, 1 << 29),
    (lambda: inputs.star_graph(5000), 0.5, 6, 3, 1 << 28),                   # hub: queue overflow
    (lambda: inputs.random_powerlaw_graph(20000, 60000, 49), 0.3, 8, 5, 1 << 24),
    (lambda: inputs.random_powerlaw_graph(3000, 15000, 50), ("unif", 0.0, 0.1), 32, 8, 1 << 28),
    (lambda: inputs.random_graph(2000, 8000, 51), ("unif", 0.1, 0.3), 16, 6, 1 << 28),
]


def run_case(orc, ctx, i, check_sketches=True):
    from oracle.oracle import Graph
    build_fn, p, R, k, a32 = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    if p == "wic":
        model, t32 = 1, 0
    elif isinstance(p, tuple):  # R19 Uniform U(lo, hi)
        model, t32 = 2, orc.uniform_param(p[1], p[2])
    else:
        model, t32 = 0, orc.t32_const(p)
    seed = 500 + i
    ctx.pacim_load_graph(g.off, g.nbr, model, t32, 2)
    ctx.pacim_build_sketches(R, seed, a32)
    st = ctx.pacim_get_stats()
    cs, _ = orc.centers(g.n, seed, a32)
    assert st["compressed"] == 1 and st["rho"] == len(cs)
    if check_sketches:
        for r in range(R):
            lab, sz = ctx.pacim_get_center_sketch(r)
            elab, esz = orc.compressed_sketch(g, model, t32, seed, r, a32)
            assert np.array_equal(lab, elab), r
            assert np.array_equal(sz, esz), r
    s, gn, sg, _ = ctx.pacim_select_seeds(k)
    es, egn, esg, eg0 = orc.greedy(g, model, t32, R, seed, k, want_gain0=True)
    assert np.array_equal(ctx.pacim_get_gain0(), eg0)
    assert list(s) == list(es)
    assert list(gn) == list(egn)
    assert list(sg) == list(esg)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_compressed_parity(orc, ctx, i):
    run_case(orc, ctx, i)


@pytest.mark.parametrize("i", [1, 2, 4])
def test_compressed_multibatch(orc, ctx, i, monkeypatch):
    monkeypatch.setenv("PACIM_BATCH", "3")  # 3 slots per build batch
    run_case(orc, ctx, i)


def test_compressed_equals_uncompressed_c1(ctx):
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config("c1")
    pipeline.generate(ctx, cfg)
    ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"])
    a = ctx.pacim_select_seeds(cfg["k"])
    ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"], 1 << 28)
    b = ctx.pacim_select_seeds(cfg["k"])
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_compressed_rank_emulation(orc, pc):
    from oracle.oracle import Graph
    from paper_2311_07554_b200 import dist
    off, nbr = inputs.random_powerlaw_graph(2500, 12000, 48)
    g = Graph(2500, off, nbr)
    t32 = orc.t32_const(0.08)
    R, seed, k = 20, 9, 10
    es, egn, esg, _ = orc.greedy(g, 0, t32, R, seed, k)
    ctxs = []
    for rank in range(2):
        c = pc.Context(0)
        c.pacim_load_graph(off, nbr, 0, t32, 1)
        c.pacim_build_sketches(R, seed, 1 << 28, rank, 2)
        ctxs.append(c)
    seeds, gains, sig = dist.emulated_select(ctxs, g.n, k, device="cuda")
    assert list(seeds) == list(es) and list(gains) == list(egn)
    for c in ctxs:
        c.close()


def test_c5_shape_scale16(orc, ctx):
    """BASELINE.json configs[4]'s shape (web R-MAT a,b,c,d = .6/.15/.15/.1, ef
    32, p = 0.01, R = 256, alpha = 1/16 compressed) at scale 16, generated on
    the GPU: seeds and gains equal the oracle's greedy (compression is
    transparent, R17), the generated CSR equals the oracle's."""
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config("c5", scale=16, k=20)
    n, m = pipeline.generate(ctx, cfg)
    g = orc.gen_config(cfg)
    assert (n, m) == (g.n, g.m)
    s, gn, sg, _ = pipeline.run(ctx, cfg)
    st = ctx.pacim_get_stats()
    assert st["compressed"] == 1 and st["rho"] < n // 8
    model, t32 = orc.model_args(cfg)
    es, egn, esg, _ = orc.greedy(g, model, t32, cfg["R"], cfg["hash_seed"], cfg["k"])
    assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)


@pytest.mark.parametrize("i", [1, 4, 10])
def test_compressed_decorrelated_rule(orc, ctx, i):
    """Compressed store + Get-center under the decorrelated rule (R20): the
    greedy equals the oracle's memoised greedy with the same rule."""
    from oracle.oracle import Graph
    build_fn, p, R, k, a32 = CASES[i]
    off, nbr = build_fn()
    g = Graph(len(off) - 1, off, nbr)
    if p == "wic":
        model, t32 = 1, 0
    elif isinstance(p, tuple):
        model, t32 = 2, orc.uniform_param(p[1], p[2])
    else:
        model, t32 = 0, orc.t32_const(p)
    ctx.pacim_set_hash_rule(1)
    try:
        ctx.pacim_load_graph(g.off, g.nbr, model, t32, 2)
        ctx.pacim_build_sketches(R, 900 + i, a32)
        s, gn, sg, _ = ctx.pacim_select_seeds(k)
        es, egn, esg, _ = orc.greedy(g, model | orc.DECOR, t32, R, 900 + i, k)
        assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)
    finally:
        ctx.pacim_set_hash_rule(0)


def test_c5_shape_scale16_lean_bucketed(orc, ctx, monkeypatch):
    """The c5 path at full scale — bucketed generator, lean graph, compressed
    store — at scale 16: the oracle's greedy."""
    monkeypatch.setenv("PACIM_GEN_BUCKETS", "8")
    monkeypatch.setenv("PACIM_LEAN", "1")
    test_c5_shape_scale16(orc, ctx)
    assert ctx.pacim_get_stats()["rows"] == 1 << 16


@pytest.mark.parametrize("i", [0, 1, 3, 9, 10])
def test_compressed_csr_direct(orc, ctx, i, monkeypatch):
    """Compressed builds over the CSR-direct edge form (PACIM_UCSR=4: c5's
    default at full scale — store rows compacted, no edge lists, no HLA)."""
    monkeypatch.setenv("PACIM_UCSR", "4")
    run_case(orc, ctx, i, check_sketches=True)


@pytest.mark.parametrize("upper", ["1", "0"])
@pytest.mark.parametrize("i", [0, 1, 3, 9])
def test_compressed_lean(orc, ctx, i, upper, monkeypatch):
    monkeypatch.setenv("PACIM_LEAN", "1")
    monkeypatch.setenv("PACIM_LEAN_UPPER", upper)
    run_case(orc, ctx, i, check_sketches=True)


@pytest.mark.parametrize("i", [1, 4, 8, 9, 10])
def test_compressed_hla(orc, ctx, i, monkeypatch):
    """Get-center probes expand a hub from the live hub adjacency the build
    recorded (forced; hub degree lowered to 4 so the small graphs have hubs): the
    seeds, gains and gain0 equal the oracle's greedy."""
    monkeypatch.setenv("PACIM_HUB_DEG", "4")
    monkeypatch.setenv("PACIM_HLA", "1")
    run_case(orc, ctx, i, check_sketches=False)
    st = ctx.pacim_get_stats()
    assert st["hubs"] > 0 and st["hla_entries"] > 0


@pytest.mark.parametrize("i", [4, 10])
def test_compressed_hla_multibatch(orc, ctx, i, monkeypatch):
    """HLA recorded across several build batches (3 sketches per batch)."""
    monkeypatch.setenv("PACIM_HUB_DEG", "4")
    monkeypatch.setenv("PACIM_HLA", "1")
    monkeypatch.setenv("PACIM_BATCH", "3")
    run_case(orc, ctx, i, check_sketches=False)
    assert ctx.pacim_get_stats()["hla_entries"] > 0


def test_compressed_no_hla_star(orc, ctx, monkeypatch):
    """PACIM_NO_HLA: hubs are scanned edge by edge (the star's hub has 4999
    neighbours > the default hub degree)."""
    monkeypatch.setenv("PACIM_NO_HLA", "1")
    run_case(orc, ctx, 8)
    st = ctx.pacim_get_stats()
    assert st["hubs"] == 1 and st["hla_entries"] == 0


@pytest.mark.parametrize("batch", [None, "100"])
def test_compressed_many_sketches(orc, ctx, batch, monkeypatch):
    """Compressed store with R = 700 (probe warps over many slots, several
    build batches when PACIM_BATCH = 100): the oracle's greedy and gain0."""
    from oracle.oracle import Graph
    if batch:
        monkeypatch.setenv("PACIM_BATCH", batch)
    off, nbr = inputs.random_powerlaw_graph(800, 3200, 61)
    g = Graph(800, off, nbr)
    t32 = orc.t32_const(0.08)
    ctx.pacim_load_graph(g.off, g.nbr, 0, t32, 2)
    ctx.pacim_build_sketches(700, 62, 1 << 29)
    assert ctx.pacim_get_stats()["compressed"] == 1
    s, gn, sg, _ = ctx.pacim_select_seeds(10)
    es, egn, esg, eg0 = orc.greedy(g, 0, t32, 700, 62, 10, want_gain0=True)
    assert np.array_equal(ctx.pacim_get_gain0(), eg0)
    assert list(s) == list(es) and list(gn) == list(egn) and list(sg) == list(esg)


@pytest.mark.parametrize("big", ["8", "40"])
@pytest.mark.parametrize("i", [1, 2, 4, 8, 9])
def test_compressed_hub_hotsum(orc, ctx, i, big, monkeypatch):
    """Covered CCs above a (lowered) size threshold: the batch rebuild + dense
    pass, or — when the hub (maximum-degree vertex) is the seed while its big
    CCs are all uncovered — the build's per-vertex hotsum; the greedy equals
    the oracle's."""
    monkeypatch.setenv("PACIM_CBIG_T", big)
    run_case(orc, ctx, i, check_sketches=False)
    if i == 8:  # the star's center is the hub and the first seed
        assert ctx.pacim_get_stats()["select_hotsum_steps"] == 1


@pytest.mark.parametrize("i", [2, 3, 9])
def test_compressed_batch_buffer_released(orc, ctx, i, monkeypatch):
    """The batch buffer released (forced before every cover step, as when the
    selection's traversal state needs the room) and re-created by the
    rebuilds of big CCs (threshold lowered, 3 sketches per batch): the
    oracle's greedy."""
    monkeypatch.setenv("PACIM_FORCE_RELEASE", "1")
    monkeypatch.setenv("PACIM_CBIG_T", "40")
    monkeypatch.setenv("PACIM_BATCH", "3")
    run_case(orc, ctx, i, check_sketches=False)
