"""Write tests/golden/<cfg>.json from the CPU oracle ONLY (no CUDA involved).

    python tests/golden/make_golden.py c1 c2 c3

Each file holds, for one BASELINE.json config: the generated graph's digests
(sha256 of the sorted upper key list and of the CSR arrays), the oracle's
greedy output (seeds, gain_num, sigma_num), a digest plus sampled entries of
gain0 = sum_r |C_r(v)|, and digests of the canonical label arrays of a few
sketches.  Digests are sha256 over little-endian array bytes.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
from oracle import oracle as O  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_idx(n: int, cnt: int = 64):
    rng = np.random.default_rng(12345)
    return sorted(set(int(x) for x in rng.integers(0, n, cnt)))


def make(name: str):
    cfg = inputs.config(name)
    t0 = time.time()
    g = O.gen_config(cfg)
    t_gen = time.time() - t0
    model, t32 = O.model_args(cfg)
    R, k, hs = cfg["R"], cfg["k"], cfg["hash_seed"]
    t0 = time.time()
    seeds, gain, sigma, gain0 = O.greedy(g, model, t32, R, hs, k, want_gain0=True)
    t_greedy = time.time() - t0
    lab_sk = sorted({0, 1, R // 2, R - 1})
    labels = {}
    for r in lab_sk:
        lab, _ = O.sketch_labels(g, model, t32, hs, r)
        labels[str(r)] = sha(lab)
    idx = sample_idx(g.n)
    out = dict(
        config=name, source="oracle/pacim_oracle.c via tests/golden/make_golden.py",
        n=g.n, m=g.m, t32=t32, model=model, R=R, k=k, hash_seed=hs,
        keys_sha256=sha(g.keys), off_sha256=sha(g.off), nbr_sha256=sha(g.nbr),
        seeds=[int(x) for x in seeds], gain_num=[int(x) for x in gain],
        sigma_num=[int(x) for x in sigma],
        gain0_sha256=sha(gain0), gain0_sum=int(gain0.sum()),
        gain0_samples={str(i): int(gain0[i]) for i in idx},
        label_sha256=labels,
        oracle_seconds=dict(generate=round(t_gen, 2), greedy=round(t_greedy, 2)),
    )
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(name, "done", out["oracle_seconds"], flush=True)


def make_partial(name: str, sketches):
    """Full-size configs whose greedy is out of single-thread reach (c4):
    graph digests plus the canonical labels / CC-size histogram of a few
    sketches, each by the oracle's BFS labelling."""
    cfg = inputs.config(name)
    t0 = time.time()
    g = O.gen_config(cfg)
    t_gen = time.time() - t0
    model, t32 = O.model_args(cfg)
    hs = cfg["hash_seed"]
    labels, hist = {}, {}
    t0 = time.time()
    for r in sketches:
        lab, size = O.sketch_labels(g, model, t32, hs, r)
        labels[str(r)] = sha(lab)
        roots = lab == np.arange(g.n, dtype=np.uint32)
        sz = size[roots].astype(np.int64)
        hist[str(r)] = dict(ncc=int(roots.sum()), nonsingleton=int((size > 1).sum()),
                            max=int(sz.max()), sum_sq=int((sz * sz).sum()))
    t_lab = time.time() - t0
    out = dict(config=name, partial=True,
               source="oracle/pacim_oracle.c via tests/golden/make_golden.py --partial",
               n=g.n, m=g.m, model=model, t32=t32, R=cfg["R"], hash_seed=hs,
               keys_sha256=sha(g.keys), off_sha256=sha(g.off), nbr_sha256=sha(g.nbr),
               label_sha256=labels, cc_stats=hist,
               oracle_seconds=dict(generate=round(t_gen, 2), label=round(t_lab, 2)))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(name, "partial done", out["oracle_seconds"], flush=True)


def make_graph(name: str, scale: int):
    """Graph-only golden of a config's generator at a reduced R-MAT scale
    (c5 at scale 25: its full-size CSR does not fit this host): n, m and the
    sha256 of the oracle's CSR.  The GPU test checks its own generator's CSR
    against it and then certifies the GPU's seeds and gains in verify mode."""
    cfg = inputs.config(name, scale=scale)
    t0 = time.time()
    g = O.gen_config(cfg)
    t_gen = time.time() - t0
    out = dict(config=name, scale=scale, graph_only=True,
               source="oracle/pacim_oracle.c via tests/golden/make_golden.py --graph",
               n=g.n, m=g.m, keys_sha256=sha(g.keys), off_sha256=sha(g.off),
               nbr_sha256=sha(g.nbr), oracle_seconds=dict(generate=round(t_gen, 2)))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{name}_s{scale}_graph.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(name, scale, "graph done", out["oracle_seconds"], flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--graph":
        make_graph(sys.argv[2], int(sys.argv[3]))
    elif sys.argv[1] == "--partial":
        make_partial(sys.argv[2], [int(x) for x in sys.argv[3].split(",")])
    else:
        for nm in sys.argv[1:]:
            make(nm)
