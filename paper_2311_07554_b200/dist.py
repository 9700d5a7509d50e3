"""Multi-rank greedy over sketch shards.

Rank g holds the sketches r with r % P == g (pacim_build_sketches with
shard_rank=g, shard_world=P) over a replicated CSR.  Integer sums are
associative, so any partition gives the single-GPU result bit for bit.

gain0 is all-reduced once after the build.  Per greedy step every rank
  1. takes the argmax of the replicated global gain vector (identical on all
     ranks: same data, deterministic (gain desc, id asc) reduction),
  2. runs MarkSeed on its own sketches (pacim_cover_local_sparse): the member
     updates go into a dense int64 delta vector AND a sparse list (vertex,
     delta) of at most `cap` entries,
  3. all-gathers a 3-word header (list length, local sum of delta_r, list
     overflow) and checks sum == argmax gain;
  4. sparse path (every list complete, total <= n / 8): all-gathers the lists
     (padded to the longest) and applies them (pacim_apply_deltas), then
     clears its own delta entries; dense fallback (a giant CC, e.g. the first
     steps of c3): all-reduces the delta vector (pacim_apply_dense).
The seed's gain becomes -1 in the apply call (R6).  Per step that is two small
collectives instead of an 8n-byte all-reduce.

Engines are any objects with the per-rank primitives of include/pacim.h
(pacim_gain0_to_device, pacim_select_reset, pacim_cover_local_sparse,
pacim_apply_deltas, pacim_apply_dense, pacim_clear_deltas,
pacim_argmax_device) — a paper_2311_07554_b200.Context on a GPU.
"""
from __future__ import annotations

import numpy as np
import torch

NONE = 0xFFFFFFFF


def init_comm(ctx, rank: int, world: int, group=None):
    """NCCL communicator of the library (pacim_init_comm): rank 0 makes the
    128-byte id, torch.distributed broadcasts it (host plumbing only); the
    sharded build then all-reduces gain0 and pacim_select_seeds runs the
    whole sharded greedy loop inside the library (dist.cu)."""
    import torch.distributed as dist
    from .binding import pacim_nccl_unique_id
    obj = [pacim_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.pacim_init_comm(rank, world, obj[0])


class _Shard:
    """One engine's step buffers: dense delta and the sparse list."""

    def __init__(self, eng, n, cap, device):
        self.eng = eng
        self.delta = torch.zeros(n, dtype=torch.int64, device=device)
        self.lv = torch.zeros(max(cap, 1), dtype=torch.int32, device=device)   # u32 ids
        self.ld = torch.zeros(max(cap, 1), dtype=torch.int64, device=device)
        self.cap = cap

    def cover(self, s):
        cnt, loc = self.eng.pacim_cover_local_sparse(s, self.delta, self.lv, self.ld, self.cap)
        return cnt, loc


def _gain0(engines, n, device, reduce_tensor):
    gain = torch.zeros(n, dtype=torch.int64, device=device)
    tmp = torch.empty_like(gain)
    for e in engines:
        e.pacim_gain0_to_device(tmp)
        gain += tmp
    reduce_tensor(gain)
    for e in engines:
        e.pacim_select_reset()
    return gain


def default_cap(n: int) -> int:
    return max(1024, n // 8)


def distributed_select(engine, n: int, k: int, device, group=None, cap: int | None = None,
                       mode: str = "sparse"):
    """This rank's part of the sharded greedy (call on every rank).  Returns
    (seeds, gain_num, sigma_num) — identical on every rank."""
    import torch.distributed as dist
    P = dist.get_world_size(group)
    cap = default_cap(n) if cap is None else cap
    gain = _gain0([engine], n, device, lambda t: dist.all_reduce(t, group=group))
    sh = _Shard(engine, n, cap, device)
    seeds = np.zeros(k, np.uint32)
    gains = np.zeros(k, np.int64)
    hall = torch.zeros(3 * P, dtype=torch.int64, device=device)
    for i in range(k):
        s, g = engine.pacim_argmax_device(gain, n)
        cnt, loc = sh.cover(s)
        hdr = torch.tensor([min(cnt, cap), loc, int(cnt > cap)], dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(hall, hdr, group=group)
        h = hall.view(P, 3).cpu().numpy()
        tot = int(h[:, 1].sum())
        if tot != g:
            raise RuntimeError(f"step {i}: sum_r delta_r = {tot} != argmax gain {g}")
        counts = h[:, 0]
        if mode == "dense" or h[:, 2].any() or int(counts.sum()) > n // 8:
            dist.all_reduce(sh.delta, group=group)  # dense fallback
            engine.pacim_apply_dense(gain, sh.delta, n, s)
        else:
            mc = int(counts.max())
            if mc:
                c = min(cnt, cap)
                sh.lv[c:mc] = 0  # neutral padding (delta 0)
                sh.ld[c:mc] = 0
                V = torch.empty(P * mc, dtype=torch.int32, device=device)
                D = torch.empty(P * mc, dtype=torch.int64, device=device)
                dist.all_gather_into_tensor(V, sh.lv[:mc].contiguous(), group=group)
                dist.all_gather_into_tensor(D, sh.ld[:mc].contiguous(), group=group)
                engine.pacim_apply_deltas(gain, V, D, P * mc, s)
                engine.pacim_clear_deltas(sh.delta, sh.lv, c)
            else:
                engine.pacim_apply_deltas(gain, sh.lv, sh.ld, 0, s)
        seeds[i] = s
        gains[i] = g
    return seeds, gains, np.cumsum(gains)


def emulated_select(engines, n: int, k: int, device="cuda", cap: int | None = None,
                    mode: str = "sparse"):
    """All shards in one process, one after another (rank emulation): the
    collectives become local concatenations / sums."""
    cap = default_cap(n) if cap is None else cap
    gain = _gain0(engines, n, device, lambda t: None)
    shards = [_Shard(e, n, cap, device) for e in engines]
    lead = engines[0]
    seeds = np.zeros(k, np.uint32)
    gains = np.zeros(k, np.int64)
    for i in range(k):
        s, g = lead.pacim_argmax_device(gain, n)
        res = [sh.cover(s) for sh in shards]
        tot = sum(loc for _, loc in res)
        if tot != g:
            raise RuntimeError(f"step {i}: sum_r delta_r = {tot} != argmax gain {g}")
        over = any(c > cap for c, _ in res)
        if mode == "dense" or over or sum(c for c, _ in res) > n // 8:
            for j, sh in enumerate(shards):
                sh.eng.pacim_apply_dense(gain, sh.delta, n, s if j == len(shards) - 1 else NONE)
        else:
            for j, (sh, (c, _)) in enumerate(zip(shards, res)):
                sh.eng.pacim_apply_deltas(gain, sh.lv, sh.ld, c, s if j == len(shards) - 1 else NONE)
                sh.eng.pacim_clear_deltas(sh.delta, sh.lv, c)
        seeds[i] = s
        gains[i] = g
    return seeds, gains, np.cumsum(gains)
