"""Multi-rank greedy over sketch shards.

Rank g holds the sketches r with r % P == g (pacim_build_sketches with
shard_rank=g, shard_world=P) over a replicated CSR.  Integer sums are
associative, so any partition gives the single-GPU result bit for bit.

Per greedy step every rank
  1. takes the argmax of the replicated global gain vector (identical on all
     ranks: same data, deterministic (gain desc, id asc) reduction),
  2. runs MarkSeed on its own sketches (pacim_cover_local), accumulating the
     member deltas into a dense int64 vector,
  3. all-reduces the deltas and the step's local gain sum (torch.distributed:
     NCCL on GPUs, gloo in the CPU tests), checks sum == argmax gain and
     applies the deltas; the seed's gain becomes -1.
gain0 is all-reduced once after the build.

Engines are any objects with the four per-rank primitives of include/pacim.h
(pacim_gain0_to_device, pacim_select_reset, pacim_cover_local,
pacim_argmax_device) — a paper_2311_07554_b200.Context on a GPU.
"""
from __future__ import annotations

import numpy as np
import torch


def _greedy(engines, n, k, device, reduce_tensor, reduce_int):
    gain = torch.zeros(n, dtype=torch.int64, device=device)
    tmp = torch.empty_like(gain)
    for e in engines:
        e.pacim_gain0_to_device(tmp)
        gain += tmp
    reduce_tensor(gain)
    for e in engines:
        e.pacim_select_reset()
    delta = torch.zeros_like(gain)
    seeds = np.zeros(k, np.uint32)
    gains = np.zeros(k, np.int64)
    for i in range(k):
        s, g = engines[0].pacim_argmax_device(gain, n)
        delta.zero_()
        loc = 0
        for e in engines:
            loc += e.pacim_cover_local(s, delta)
        tot = reduce_int(loc)
        reduce_tensor(delta)
        if tot != g:
            raise RuntimeError(f"step {i}: sum_r delta_r = {tot} != argmax gain {g}")
        gain += delta
        gain[s] = -1
        seeds[i] = s
        gains[i] = g
    return seeds, gains, np.cumsum(gains)


def distributed_select(engine, n: int, k: int, device, group=None):
    """This rank's part of the sharded greedy (call on every rank)."""
    import torch.distributed as dist

    def red_t(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    def red_i(x):
        t = torch.tensor([x], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return int(t.item())

    return _greedy([engine], n, k, device, red_t, red_i)


def emulated_select(engines, n: int, k: int, device="cuda"):
    """All shards in one process, one after another (rank emulation): the
    collectives become plain local sums."""
    return _greedy(engines, n, k, device, lambda t: None, lambda x: x)
