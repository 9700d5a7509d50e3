"""Multi-rank greedy (paper_2311_07554_b200/dist.py) on CPU with the gloo
backend, world_size 2 and 3: sketches sharded r % P == rank, per-step sparse
delta lists all-gathered (dense all-reduce fallback).  Each rank's local engine here is a test-only CPU stand-in built
from the oracle's sketch labels (the GPU tests run the same loop with the
CUDA engine); the result must equal the single-process oracle greedy."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import inputs


class OracleShard:
    """Test-only engine with the four per-rank primitives of include/pacim.h."""

    def __init__(self, g, model, t32, R, seed, rank, world):
        from oracle import oracle as O
        self.n = g.n
        self.lab = {r: O.sketch_labels(g, model, t32, seed, r)[0].astype(np.int64)
                    for r in range(rank, R, world)}
        self.size = {r: np.bincount(l, minlength=g.n) for r, l in self.lab.items()}
        self.covered = {r: set() for r in self.lab}

    def pacim_gain0_to_device(self, t):
        g0 = np.zeros(self.n, np.int64)
        for r, l in self.lab.items():
            g0 += self.size[r][l]
        t.copy_(torch.from_numpy(g0))

    def pacim_select_reset(self):
        self.covered = {r: set() for r in self.lab}

    def pacim_cover_local_sparse(self, s, delta, lv, ld, cap):
        tot, cnt = 0, 0
        for r, l in self.lab.items():
            c = int(l[s])
            if c in self.covered[r]:
                continue
            self.covered[r].add(c)
            sz = int(self.size[r][c])
            tot += sz
            mem = np.nonzero(l == c)[0]
            mem = mem[mem != s]  # the seed's own gain is set to -1 by the apply call
            delta[torch.from_numpy(mem)] -= sz
            for u in mem:
                if cnt < cap:
                    lv[cnt] = int(u)
                    ld[cnt] = -sz
                cnt += 1
        return cnt, tot

    def pacim_apply_deltas(self, gain, v, d, count, s=0xFFFFFFFF):
        gain.index_add_(0, v[:count].long(), d[:count])
        if s != 0xFFFFFFFF:
            gain[s] = -1

    def pacim_apply_dense(self, gain, delta, n, s=0xFFFFFFFF):
        gain += delta
        delta.zero_()
        if s != 0xFFFFFFFF:
            gain[s] = -1

    def pacim_clear_deltas(self, delta, v, count):
        delta[v[:count].long()] = 0

    def pacim_argmax_device(self, gain, n):
        g = int(gain.max())
        s = int(torch.nonzero(gain == g)[0])
        return s, g


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Graph
    from oracle import oracle as O
    from paper_2311_07554_b200 import dist as pdist
    off, nbr = case["graph"]
    g = Graph(len(off) - 1, off, nbr)
    eng = OracleShard(g, case["model"], case["t32"], case["R"], case["seed"], rank, world)
    seeds, gains, sig = pdist.distributed_select(eng, g.n, case["k"], torch.device("cpu"),
                                                 cap=case.get("cap"), mode=case.get("mode", "sparse"))
    out[rank] = (list(map(int, seeds)), list(map(int, gains)), list(map(int, sig)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mode,cap", [(2, "sparse", None), (3, "sparse", None),
                                            (2, "dense", None), (3, "sparse", 7)])
def test_sharded_greedy_equals_single(orc, world, mode, cap):
    """Sparse delta exchange (lists all-gathered), the dense all-reduce, and
    a list capacity small enough to force the dense fallback on some steps."""
    from oracle.oracle import Graph
    off, nbr = inputs.random_powerlaw_graph(400, 1500, 31)
    t32 = orc.t32_const(0.1)
    case = dict(graph=(off, nbr), model=0, t32=t32, R=24, seed=17, k=10, mode=mode, cap=cap)
    g = Graph(400, off, nbr)
    es, eg, esg, _ = orc.greedy(g, 0, t32, 24, 17, 10)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(worker, args=(world, free_port(), case, out), nprocs=world,
                       join=True, start_method="spawn")
    for r in range(world):
        s, gn, sg = out[r]
        assert s == list(es) and gn == list(eg) and sg == list(esg)


def test_wic_sharded(orc):
    from oracle.oracle import Graph
    off, nbr = inputs.random_graph(300, 1200, 32)
    case = dict(graph=(off, nbr), model=1, t32=0, R=16, seed=5, k=8)
    g = Graph(300, off, nbr)
    es, eg, esg, _ = orc.greedy(g, 1, 0, 16, 5, 8)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(worker, args=(2, free_port(), case, out), nprocs=2, join=True,
                       start_method="spawn")
    assert out[0][0] == list(es) and out[1][1] == list(eg)
