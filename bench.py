"""bench.py — sampled edge-tests/s and seconds-to-k-seeds of the PaC-IM hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one pass of the whole hot path over the resident synthetic graph:
pacim_build_sketches (hash + live test, union-find, compression, CC sizes in
the root slots, gain0) followed by pacim_select_seeds (k
greedy steps, H8-H12).  value = R*m / t_step summed over the job (m =
undirected edges; every logical (edge, sketch) test counted).  e2e repeats the
step through the public API from pinned HOST buffers: pacim_load_graph_async
(two loads in flight, each committed by the next build, so a step's H2D copy
overlaps the previous step's build and selection; every copy inside the timed
region) with the seeds/gains read back to the host.

N > 1 (torchrun): sketches are sharded r % N == rank over a replicated CSR,
each greedy step exchanges sparse gain deltas (NCCL all-gathers; a dense
all-reduce when a list overflows); total work is fixed (strong scaling).
--force-dist runs that per-step exchange even at one rank (testing).
Debugging: PACIM_BENCH_DEBUG=1 prints the e2e steps' wall times,
PACIM_E2E_SYNC=1 uses the unpipelined pacim_load_graph in the e2e loop.  Timing: CUDA events on the library's stream (= torch's
current stream), barrier + synchronize on both sides, max over ranks.

--impl reference times the CPU oracle (oracle/, single-threaded C) on a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "sampled edge-tests/s (R*m/t) for sketch build + k-seed selection; seconds to k seeds"
UNIT = "edge-tests/s"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                smax.append(float(p[1]))
            except ValueError:
                continue
            for nm, val in zip(names, p[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ roofline model
def kernel_bytes(st: dict, cfg: dict, k: int) -> dict:
    """Algorithmic bytes per launch of each kernel."""
    n, m, B, rows = st["n"], st["m"], st["R_local"], st["rows"]
    L = 4 * rows * B                      # the store: one u32 slot per (row, sketch)
    wic = 4 * m if cfg["pmodel"] != 0 else 0  # per-edge thresholds (WIC, Uniform)
    nonroot = st["nnonsingle"] - st["ncomp"]
    # the edge source is read once per build batch (compressed mode); a lean
    # graph's source is the CSR (u32 per entry, 2m entries), else the upper
    # edge list (u64 key + u64 row pair, + T32)
    nb = -(-B // st["batch_slots"]) if st.get("compressed") and st.get("batch_slots") else 1
    edge_src = 8 * m if st.get("lean") else 16 * m + wic
    return {
        "k_init": L,                                        # write every slot
        "k_edges": nb * edge_src + 8 * st["live_pairs"],    # edge source per pass, 2 slot reads per live pair
        "k_compress_count": L + 8 * nonroot,                # read slots; write root + count per non-root
        "k_gain0": L + 8 * n + 4 * nonroot,                 # slots, gain0, root-size reads
        # traversal reads (CSR entry + WIC threshold) + the dense passes over the
        # store + one read of the gains per step for the chunk maxima (upper bound)
        "k_select": (4 + (4 if cfg["pmodel"] != 0 else 0)) * st["select_edges"]
                    + L * st["select_dense_steps"] + k * 16 * 4096,
    }


def build_bytes(st: dict, cfg: dict) -> int:
    """CSR_upper * ceil(R_g/B) + 16 n R_g (B = sketches per pass:
    R_g uncompressed, the batch in compressed mode)."""
    if st.get("lean"):
        csr_upper = 8 * st["m"]  # the CSR itself (u32 per entry, 2m entries)
    else:
        csr_upper = 16 * st["m"]  # u64 hash key + u64 row pair per upper edge read by k_edges
    if cfg["pmodel"] != 0:
        csr_upper += 4 * st["m"]
    B = st["R_local"]
    nb = -(-B // st["batch_slots"]) if st.get("compressed") and st.get("batch_slots") else 1
    return csr_upper * nb + 16 * st["rows"] * B


def load_peaks():
    try:
        return json.load(open(PEAKS))
    except Exception:
        return {}


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


# ----------------------------------------------------------- CPU baseline
def oracle_sample(cfg, seconds_target=15.0, max_sketches=None, g=None):
    """Time the oracle's BFS sketch labelling (single thread) on sketches
    0,1,2,... of the workload until ~seconds_target; returns (tests/s, S, t, g)."""
    from oracle import oracle as O
    if g is None:
        g = O.gen_config(cfg)
    model, t32 = O.model_args(cfg)
    S, t = 0, 0.0
    while t < seconds_target and (max_sketches is None or S < max_sketches) and S < cfg["R"]:
        t0 = time.perf_counter()
        O.sketch_labels(g, model, t32, cfg["hash_seed"], S)
        t += time.perf_counter() - t0
        S += 1
    return (S * g.m / t if t > 0 else 0.0), S, t, g


def run_reference(args, cfg):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import oracle as O
    g = O.gen_config(cfg)
    per_step = max(1, args.ref_sketches)
    for _ in range(args.warmup):
        oracle_sample(cfg, 1e9, per_step, g)  # bounded by per_step sketches
    t = 0.0
    for _ in range(args.steps):
        _, S, dt, _ = oracle_sample(cfg, 1e9, per_step, g)
        t += dt
    value = args.steps * per_step * g.m / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * t / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg["name"], "n": g.n, "m": g.m, "R": cfg["R"], "k": cfg["k"],
                   "sample": f"{per_step} sketch(es) per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"oracle BFS labelling (orc_sketch_labels) of {per_step} of "
                                   f"{cfg['R']} sketches per step of {cfg['name']}, 1 thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--alpha", type=float, default=None,
                    help="override the config's alpha (< 1: compressed store)")
    ap.add_argument("--scale", type=int, default=None,
                    help="override the R-MAT scale (c5 at full scale needs 8 GPUs)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--ref-sketches", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="testing: NCCL process group and the per-step collectives even at one rank")
    args = ap.parse_args()
    args.e2e_steps = max(1, args.e2e_steps)  # the e2e number needs at least one step
    cfg = inputs.config(args.config, **({"scale": args.scale} if args.scale else {}))
    if args.alpha is not None:
        cfg["alpha"] = args.alpha
    if args.impl == "reference":

        run_reference(args, cfg)
        return
    k = args.k or cfg["k"]
    rank, world, local = env_rank()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2311_07554_b200 as P
    from paper_2311_07554_b200 import dist as pdist
    from paper_2311_07554_b200 import pipeline
    stream = torch.cuda.current_stream(dev)
    ctx = P.Context(local, stream.cuda_stream)
    n, m = pipeline.generate(ctx, cfg)
    pm, t32 = pipeline.model_of(cfg)
    a32 = pipeline.center_a32_of(cfg)
    R = cfg["R"]

    def barrier():
        if use_dist:
            torch.distributed.barrier()

    def step():
        ctx.pacim_build_sketches(R, cfg["hash_seed"], a32, rank, world)
        if not use_dist:
            return ctx.pacim_select_seeds(k)
        return pdist.distributed_select(ctx, n, k, dev)

    for _ in range(max(3, args.warmup)):
        step()
    # ---------------- device-resident timed region
    keys = ["t_build_ms", "t_init_ms", "t_edges_ms", "t_compress_ms", "t_gain_ms", "t_select_ms"]
    acc = {kk: 0.0 for kk in keys}
    launches = 0
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.15)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        out = step()
        st = ctx.stats_raw()  # the struct's fields, no dict: little host time between steps
        for kk in keys:
            acc[kk] += getattr(st, kk)
        launches += st.kernel_launches_build + (st.kernel_launches_select if world == 1 else 0)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = R * m / (ms_step / 1000.0)
    avg = {kk: acc[kk] / args.steps for kk in keys}
    st = ctx.pacim_get_stats()

    # ---------------- end to end through the public API (host CSR, pinned)
    off, nbr = ctx.pacim_get_graph()
    h_off = torch.from_numpy(off).pin_memory()
    h_nbr = torch.from_numpy(nbr).pin_memory()
    off_np, nbr_np = h_off.numpy(), h_nbr.numpy()

    # Pipelined through the public API: step i+1's host CSR is enqueued
    # (pacim_load_graph_async, pinned memory) before step i runs, so its H2D
    # copy overlaps step i's build and selection; the build of step i+1 commits
    # it (waits for the copy, derives the edge lists).  Every step's copy and
    # its seeds/gains read-back stay inside the timed region.
    # warm-up of the pipelined path: both staging slots allocated and used
    # (graphs whose two staged copies do not fit beside the resident one — c5
    # — take the unpipelined loop)
    _sync = bool(os.environ.get("PACIM_E2E_SYNC"))  # debugging: the unpipelined loop
    e2e_mode = ("pacim_load_graph_async from pinned host CSR, two loads in flight: "
                "the next steps' H2D copies overlap this step's build and selection")
    if not _sync:
        try:
            ctx.pacim_load_graph_async(off_np, nbr_np, pm, t32)
            ctx.pacim_load_graph_async(off_np, nbr_np, pm, t32)
            step()
            step()
        except P.PacimError as e:
            if "ENOMEM" not in str(e):
                raise
            _sync = True
            ctx.pacim_load_graph(off_np, nbr_np, pm, t32, 0)  # drops the pending loads
    if _sync:
        e2e_mode = "pacim_load_graph from pinned host CSR (two staged copies do not fit)"
        ctx.pacim_load_graph(off_np, nbr_np, pm, t32, 0)
        step()
    barrier()
    torch.cuda.synchronize(dev)
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    # two loads in flight: steps 0 and 1 enqueued up front; the build of step
    # i commits its graph (freeing that staging slot), then step i+2's load is
    # enqueued before step i's selection, so the copy engine never waits on
    # the host
    if not _sync:
        ctx.pacim_load_graph_async(off_np, nbr_np, pm, t32)
        if args.e2e_steps > 1:
            ctx.pacim_load_graph_async(off_np, nbr_np, pm, t32)
    _tw = [time.perf_counter()]
    for i in range(args.e2e_steps):
        if _sync:
            ctx.pacim_load_graph(off_np, nbr_np, pm, t32, 0)
        ctx.pacim_build_sketches(R, cfg["hash_seed"], a32, rank, world)  # commits step i's graph
        if i + 2 < args.e2e_steps and not _sync:
            ctx.pacim_load_graph_async(off_np, nbr_np, pm, t32)  # step i+2's input
        out = ctx.pacim_select_seeds(k) if not use_dist else pdist.distributed_select(ctx, n, k, dev)
        _tw.append(time.perf_counter())
        if os.environ.get("PACIM_BENCH_DEBUG"):
            _st = ctx.stats_raw()
            print("  step", i, "build", round(_st.t_build_ms, 2), "select", round(_st.t_select_ms, 2),
                  file=sys.stderr)
    f1.record(stream)
    if os.environ.get("PACIM_BENCH_DEBUG"):
        print("e2e wall ms per step:", [round(1e3 * (_tw[i + 1] - _tw[i]), 1) for i in range(len(_tw) - 1)],
              file=sys.stderr)
    torch.cuda.synchronize(dev)
    barrier()
    ms_e2e = f0.elapsed_time(f1)
    if world > 1:
        t = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e_value = R * m / (ms_e2e / args.e2e_steps / 1000.0)
    h2d = off.nbytes + nbr.nbytes
    d2h = k * (4 + 8 + 8 + 8)

    # ---------------- roofline (dominant kernel, live CUDA-event durations)
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "measured" if hbm else "fallback"
    hbm = hbm or 6650.0
    kb = kernel_bytes(st, cfg, k)
    dur = {"k_init": avg["t_init_ms"], "k_edges": avg["t_edges_ms"],
           "k_compress_count": avg["t_compress_ms"], "k_gain0": avg["t_gain_ms"],
           "k_select": avg["t_select_ms"]}
    dom = max(dur, key=lambda x: dur[x])
    achieved = kb[dom] / (dur[dom] / 1000.0) / 1e9
    traffic = load_traffic().get(args.config, {}).get(dom)
    bb = build_bytes(st, cfg)
    build_gbs = bb / (avg["t_build_ms"] / 1000.0) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                "traffic": traffic, "peak_source": peak_src,
                "share_of_step": round(dur[dom] / ms_step, 3),
                "kernel_ms": {kk: round(v, 4) for kk, v in dur.items()},
                "build": {"bytes": bb, "ms": round(avg["t_build_ms"], 4),
                          "achieved": round(build_gbs, 1), "frac": round(build_gbs / hbm, 4),
                          "model": "SURVEY 8(d): CSR_upper*ceil(R_g/B) + 16*rows*R_g, B = sketches per pass (R_g; the batch in compressed mode), rows = store rows; CSR_upper = the edge source k_edges reads (edge list, or the CSR itself for lean graphs)"}}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (counter-based generator, DESIGN.md §Input recipe)",
        "config": {"workload": cfg["name"] + (f"-scale{args.scale}" if args.scale else ""),
                   "config": args.config, "n": n, "m": m, "R": R, "k": k,
                   "alpha": cfg.get("alpha"),
                   "sketches_per_pass": st["R_local"], "parallelism": f"sketch-shard x{world}",
                   "l2": "inputs larger than L2 (store 4*n*R bytes, keys 8*m bytes)",
                   "arith": "u64 hash, u32 labels, i64 gains"},
        "seconds_to_k_seeds": ms_step / 1000.0,
        "build_tests_per_s": R * m / (avg["t_build_ms"] / 1000.0),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e / args.e2e_steps,
                "mode": e2e_mode},
        "gpu_launches": launches,
        "roofline": roofline,
        "clocks": clk,
        "stats": {kk: st[kk] for kk in ("rows", "ncomp", "nnonsingle", "live_pairs", "device_bytes",
                                        "select_dense_steps", "select_warp_slots",
                                        "select_deferred_slots", "select_row_items",
                                        "select_chunk_items", "select_edges")},
        "seeds_head": [int(x) for x in out[0][:8]],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, S, t, _ = oracle_sample(cfg, args.cpu_seconds)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": f"oracle BFS labelling of sketches 0..{S - 1} of {R} "
                                          f"({t:.1f} s, 1 thread) of {cfg['name']}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if use_dist:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
