"""bench.py — sampled edge-tests/s and seconds-to-k-seeds of the PaC-IM hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Default workload: c4 = BASELINE.json configs[3] (twitter-shaped R-MAT scale
26, WIC, R = 256, k = 100), the largest configuration that fits one GPU.

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

--impl reference times the CPU oracle (oracle/, plain C) on a bounded sample
of the same workload (rank 0 only): per step, the oracle's BFS labelling of
one sketch per host core (verify mode's sketch-parallel loop), on the graph
made by the oracle's own generator.  cpu_baseline (N = 1, rank 0) times the
same on the CSR read back from the device.
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

import numpy as np

# stdout carries only the JSON line: native output (the image sets
# NCCL_DEBUG=VERSION, whose banner NCCL prints to stdout at communicator
# init) goes to stderr — fd 1 is pointed at stderr and the JSON line is
# written to the saved original stdout
_JSON_FD = os.dup(1)
os.dup2(2, 1)


def emit(line: dict) -> None:
    os.write(_JSON_FD, (json.dumps(line) + "\n").encode())

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
        if os.environ.get("PACIM_CLOCK_MS") == "0":  # debugging: no sampler
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("PACIM_CLOCK_MS", "50")],
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
def build_terms(st: dict, cfg: dict) -> dict:
    """SURVEY §8(d), literally: Bytes_build = ceil(R_g/B) * CSR_upper + 16 n R_g
    [+ ceil(R_g/B) * 4m for per-edge WIC / Uniform thresholds], CSR_upper =
    4m + 8(n+1).  The label term is counted per store row (the non-isolated
    vertices the method labels; an isolated vertex is a singleton in every
    sketch and has no row) and, beside it, per vertex as the formula is
    written.  Random union traffic is NOT in the denominator (§8(d)); its
    model (64 B per live pair, uncached) is reported separately."""
    n, m, B, rows = st["n"], st["m"], st["R_local"], st["rows"]
    nb = -(-B // st["batch_slots"]) if st.get("compressed") and st.get("batch_slots") else 1
    csr = nb * ((4 * m + 8 * (n + 1)) + (4 * m if cfg["pmodel"] != 0 else 0))
    return {"csr": csr, "label_rows": 16 * rows * B, "label_n": 16 * n * B, "passes": nb,
            "union_random_model": 64 * st["live_pairs"]}


def kernel_bytes(st: dict, cfg: dict, k: int) -> dict:
    """Algorithmic bytes per launch of each build kernel, the §8(d) terms
    split over the kernels that move them (label term: 4 B init write, 8 B
    finalize read + write, 4 B gain-pass read per (row, sketch)), and of the
    selection (§8(d) "Selection": 12 B per member update + 4 B per (step,
    sketch) lookup; the argmax's 8n B per step is NOT counted: the chunk-maxima
    tournament does not read the whole gain vector per step)."""
    t = build_terms(st, cfg)
    L = 4 * st["rows"] * st["R_local"]
    return {
        "k_init": L,
        "k_edges": t["csr"],
        "k_compress_count": 2 * L,
        "k_gain0": L + 8 * st["n"],
        "k_select": 12 * st["select_member_updates"] + 4 * k * st["R_local"],
    }


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
def host_info() -> dict:
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def oracle_label_sample(g, cfg, sketches: int, threads: int):
    """Label sketches 0..sketches-1 of the workload with the oracle's BFS
    labelling (orc_verify with k = 0: the verify mode's sketch loop, one
    sketch per thread at a time); returns (seconds, tests/s)."""
    from oracle import oracle as O
    model, t32 = O.model_args(cfg)
    t0 = time.perf_counter()
    rc, _ = O.verify(g, model, t32, sketches, cfg["hash_seed"], [], [], threads=threads)
    dt = time.perf_counter() - t0
    assert rc == 0
    return dt, sketches * g.m / dt


def oracle_golden_seconds(name: str):
    """Measured single-thread derive-mode seconds to k seeds (golden files)."""
    try:
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"{name}.json")))
        return gold.get("oracle_seconds", {}).get("greedy")
    except OSError:
        return None


def run_reference(args, cfg):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    g = O.gen_config(cfg, threads=threads)
    t_gen = time.perf_counter() - t0
    per_step = args.ref_sketches or threads
    for _ in range(args.warmup):
        oracle_label_sample(g, cfg, per_step, threads)
    t = 0.0
    for _ in range(args.steps):
        dt, _ = oracle_label_sample(g, cfg, per_step, threads)
        t += dt
    value = args.steps * per_step * g.m / t
    sample = (f"oracle BFS labelling (orc_verify's sketch loop, k = 0) of sketches 0..{per_step - 1} "
              f"of {cfg['R']} per step of {cfg['name']}, {threads} threads (one sketch per thread); "
              f"graph from the oracle's own (threaded) generator in {t_gen:.0f} s, untimed")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * t / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg["name"], "n": g.n, "m": g.m, "R": cfg["R"], "k": cfg["k"],
                   "sample": f"{per_step} sketch(es) per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": sample, **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ------------------------------------------------------------------- ours
def upper_csr(off, nbr, chunk=1 << 28):
    """The upper CSR of a symmetric CSR (row u keeps its neighbours > u; the
    rows stay sorted), built on the host in chunks of rows."""
    n = len(off) - 1
    off = off.astype(np.int64)
    deg = np.diff(off)
    keep_cnt = np.zeros(n, dtype=np.uint64)
    parts = []
    a = 0
    while a < n:
        b = int(np.searchsorted(off, off[a] + chunk, side="right"))
        b = min(max(b - 1, a + 1), n)
        rows = np.repeat(np.arange(a, b, dtype=np.uint32), deg[a:b])
        seg = nbr[off[a]:off[b]]
        keep = seg > rows
        parts.append(seg[keep])
        cs = np.zeros(len(seg) + 1, dtype=np.uint64)
        np.cumsum(keep, out=cs[1:])
        rel = (off[a:b + 1] - off[a]).astype(np.int64)
        keep_cnt[a:b] = cs[rel[1:]] - cs[rel[:-1]]
        a = b
    uoff = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(keep_cnt, out=uoff[1:])
    return uoff, (np.concatenate(parts) if parts else np.zeros(0, np.uint32)).astype(np.uint32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4",
                    help="BASELINE.json config (default c4 = configs[3], the largest single-GPU one)")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--alpha", type=float, default=None,
                    help="override the config's alpha (< 1: compressed store)")
    ap.add_argument("--scale", type=int, default=None,
                    help="override the R-MAT scale (c5 at full scale needs 8 GPUs)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--ref-sketches", type=int, default=0,
                    help="sketches per reference step (default: one per host core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="testing: NCCL process group and the per-step collectives even at one rank")
    ap.add_argument("--selector", default="auto", choices=["auto", "incremental", "ptree", "wintree"],
                    help="pacim_set_selector: auto (default: the Win-Tree under WIC, else incremental; "
                         "sharded: incremental)")
    ap.add_argument("--py-dist", action="store_true",
                    help="multi-rank select through dist.py's per-step primitives (torch.distributed) "
                         "instead of the library's NCCL loop")
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
        if world == 1:
            os.environ["PACIM_FORCE_DIST"] = "1"  # the sharded code at one rank (testing)
    import paper_2311_07554_b200 as P
    from paper_2311_07554_b200 import dist as pdist
    from paper_2311_07554_b200 import pipeline
    stream = torch.cuda.current_stream(dev)
    ctx = P.Context(local, stream)  # torch's current stream (legacy default: cudaStreamLegacy)
    if use_dist and not args.py_dist:
        pdist.init_comm(ctx, rank, world)  # NCCL inside the library (pacim_init_comm)
    ctx.pacim_set_selector({"incremental": 0, "ptree": 1, "wintree": 2, "auto": 3}[args.selector])
    n, m = pipeline.generate(ctx, cfg)
    pm, t32 = pipeline.model_of(cfg)
    a32 = pipeline.center_a32_of(cfg)
    R = cfg["R"]

    def barrier():
        if use_dist:
            torch.distributed.barrier()

    def step():
        ctx.pacim_build_sketches(R, cfg["hash_seed"], a32, rank, world)
        if use_dist and args.py_dist:
            return pdist.distributed_select(ctx, n, k, dev)
        return ctx.pacim_select_seeds(k)  # sharded: the whole greedy loop in the library

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
    _tw0 = [time.perf_counter()]
    for _ in range(args.steps):
        out = step()
        _tw0.append(time.perf_counter())
        st = ctx.stats_raw()  # the struct's fields, no dict: little host time between steps
        for kk in keys:
            acc[kk] += getattr(st, kk)
        launches += st.kernel_launches_build + (st.kernel_launches_select if not args.py_dist else 0)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if os.environ.get("PACIM_BENCH_DEBUG"):
        print("timed wall ms per step:", [round(1e3 * (_tw0[i + 1] - _tw0[i]), 2) for i in range(len(_tw0) - 1)],
              file=sys.stderr)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = R * m / (ms_step / 1000.0)
    avg = {kk: acc[kk] / args.steps for kk in keys}
    st = ctx.pacim_get_stats()

    # ---------------- end to end through the public API (host CSR, pinned)
    # The input crosses PCIe as the upper CSR (each undirected edge once:
    # pacim_load_graph_upper_async; the device builds the symmetric CSR), half
    # the bytes of the symmetric CSR; PACIM_E2E_FULL=1 sends the symmetric CSR
    # (pacim_load_graph_async) instead
    # Lean graphs and compressed builds (c5) send the symmetric CSR: their
    # build or Get-center probes read it, and the device-side transpose of an
    # upper CSR needs 16 B of scratch per edge (133 GB at c5)
    out_dev = out  # the resident path's result: the e2e path must reproduce it
    off, nbr = ctx.pacim_get_graph()
    _full = (bool(os.environ.get("PACIM_E2E_FULL")) or bool(st.get("lean"))
             or a32 < (1 << 32))
    if not _full:
        off, nbr = upper_csr(off, nbr)
    h_off = torch.from_numpy(off).pin_memory()
    h_nbr = torch.from_numpy(nbr).pin_memory()
    off_np, nbr_np = h_off.numpy(), h_nbr.numpy()
    load_async = ctx.pacim_load_graph_async if _full else ctx.pacim_load_graph_upper_async

    def load_sync():
        if _full:
            ctx.pacim_load_graph(off_np, nbr_np, pm, t32, 0)
        else:
            ctx.pacim_load_graph_upper(off_np, nbr_np, pm, t32, 0)

    # Pipelined through the public API: step i+1's host CSR is enqueued
    # (pacim_load_graph_async, pinned memory) before step i runs, so its H2D
    # copy overlaps step i's build and selection; the build of step i+1 commits
    # it (waits for the copy, derives the edge lists).  Every step's copy and
    # its seeds/gains read-back stay inside the timed region.
    # warm-up of the pipelined path: both staging slots allocated and used
    # (graphs whose two staged copies do not fit beside the resident one — c5
    # — take the unpipelined loop)
    _sync = bool(os.environ.get("PACIM_E2E_SYNC"))  # debugging: the unpipelined loop
    src = ("symmetric CSR" if _full else
           "upper CSR (symmetric offsets from the degrees; the symmetric lists are built "
           "on the device only when read, never on this path)")
    e2e_mode = (f"{load_async.__name__} from the pinned host {src}, two loads in flight: "
                "the next steps' H2D copies overlap this step's build and selection")
    if not _sync:
        try:
            load_async(off_np, nbr_np, pm, t32)
            load_async(off_np, nbr_np, pm, t32)
            step()
            step()
        except P.PacimError as e:
            if "ENOMEM" not in str(e):
                raise
            _sync = True
            load_sync()  # drops the pending loads
    if _sync:
        e2e_mode = f"synchronous load from the pinned host {src} (two staged copies do not fit)"
        load_sync()
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
        load_async(off_np, nbr_np, pm, t32)
        if args.e2e_steps > 1:
            load_async(off_np, nbr_np, pm, t32)
    _tw = [time.perf_counter()]
    for i in range(args.e2e_steps):
        if _sync:
            load_sync()
        ctx.pacim_build_sketches(R, cfg["hash_seed"], a32, rank, world)  # commits step i's graph
        if i + 2 < args.e2e_steps and not _sync:
            load_async(off_np, nbr_np, pm, t32)  # step i+2's input
        out = (pdist.distributed_select(ctx, n, k, dev) if (use_dist and args.py_dist)
               else ctx.pacim_select_seeds(k))
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
    # the e2e path (host CSR, another load and derivation) must give the
    # resident path's seeds and gains bit for bit
    e2e_same = (np.array_equal(np.asarray(out[0]), np.asarray(out_dev[0]))
                and np.array_equal(np.asarray(out[1]), np.asarray(out_dev[1])))
    if not e2e_same:
        print("ERROR: the e2e seeds/gains differ from the resident path's", file=sys.stderr)
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
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if hbm else "fallback (B200_PROFILING.md)"
    hbm = hbm or 6650.0
    st["select_member_updates"] = int(out[2][-1]) if len(out[2]) else 0  # N(S_k): one update each
    kb = kernel_bytes(st, cfg, k)
    dur = {"k_init": avg["t_init_ms"], "k_edges": avg["t_edges_ms"],
           "k_compress_count": avg["t_compress_ms"], "k_gain0": avg["t_gain_ms"],
           "k_select": avg["t_select_ms"]}
    if kb["k_init"] and dur["k_init"] < 0.5 * kb["k_init"] / (hbm * 1e6):
        # faster than the store write could stream at peak: the dense store's
        # slot epochs replaced the reset by an epoch bump, so the
        # 4 B per (row, sketch) init write did not happen this step
        kb["k_init"] = 0
    dom = max(dur, key=lambda x: dur[x])
    achieved = kb[dom] / (dur[dom] / 1000.0) / 1e9
    traffic_all = load_traffic().get(args.config, {})
    bt = build_terms(st, cfg)
    tb = avg["t_build_ms"] / 1000.0
    b_rows = bt["csr"] + bt["label_rows"]
    b_n = bt["csr"] + bt["label_n"]
    te = dur["k_edges"] / 1000.0
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                "traffic": traffic_all.get(dom), "peak_source": peak_src,
                "share_of_step": round(dur[dom] / ms_step, 3),
                "kernel_ms": {kk: round(v, 4) for kk, v in dur.items()},
                "kernel_bytes": kb,
                "kernel_bytes_note": ("§8(d) terms per kernel (k_init 4 B, k_compress_count 8 B, k_gain0 4 B "
                                      "per (row, sketch)); a dense epoch build with the hook list "
                                      "(stats.build_hook_list = 1) compresses only the hooked slots, so "
                                      "k_compress_count's bytes / ms may exceed the HBM peak"),
                "build": {"model": "SURVEY 8(d): ceil(R_g/B)*(CSR_upper [+4m WIC/Uniform]) + 16*rows*R_g, "
                                   "CSR_upper = 4m + 8(n+1); rows = store rows (non-isolated vertices); "
                                   "'frac_n' counts 16*n*R_g as the formula is written",
                          "csr_bytes": bt["csr"], "label_bytes_rows": bt["label_rows"],
                          "label_bytes_n": bt["label_n"], "passes": bt["passes"],
                          "bytes": b_rows, "ms": round(avg["t_build_ms"], 4),
                          "achieved": round(b_rows / tb / 1e9, 1),
                          "frac": round(b_rows / tb / 1e9 / hbm, 4),
                          "frac_n": round(b_n / tb / 1e9 / hbm, 4),
                          "frac_vs_8TBs": round(b_rows / tb / 8e12, 4)},
                "k_edges": {"bytes": bt["csr"], "ms": round(dur["k_edges"], 4),
                            "achieved": round(bt["csr"] / te / 1e9, 1),
                            "frac": round(bt["csr"] / te / 1e9 / hbm, 4),
                            "union_random_bytes_model": bt["union_random_model"],
                            "traffic": traffic_all.get("k_edges"),
                            "note": "algorithmic = the CSR term only (8(d)); random union traffic "
                                    "(64 B per live pair uncached) reported beside it; traffic = "
                                    "ncu dram__bytes_read+write per launch (profiles/traffic.json)"}}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (counter-based generator, DESIGN.md §Input recipe)",
        "selector": args.selector,
        "select_path": ("dist.py per-step primitives (torch.distributed)" if (use_dist and args.py_dist)
                        else "library NCCL loop (pacim_init_comm)" if use_dist else "single GPU"),
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
                "same_seeds_and_gains_as_resident": bool(e2e_same),
                "mode": e2e_mode},
        "gpu_launches": launches,
        "roofline": roofline,
        "clocks": clk,
        "stats": {kk: st[kk] for kk in ("rows", "ncomp", "nnonsingle", "live_pairs", "device_bytes",
                                        "select_member_updates", "build_hook_list",
                                        "select_dense_steps", "select_warp_slots",
                                        "select_deferred_slots", "select_row_items",
                                        "select_chunk_items", "select_edges")},
        "seeds_head": [int(x) for x in out[0][:8]],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle labels the CSR read back from the device (its sha256 equals
        # the oracle generator's golden digest: tests/test_gpu_parity.py)
        from oracle.oracle import Graph
        threads = os.cpu_count() or 1
        dt, v = oracle_label_sample(Graph(n, off, nbr), cfg, threads, threads)
        per_sketch_1t = dt  # one sketch per thread: ~ one sketch's single-thread time
        line["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"oracle BFS labelling (orc_verify's sketch loop) of sketches 0..{threads - 1} "
                      f"of {R} of {cfg['name']}, {threads} threads, one sketch each ({dt:.1f} s), on "
                      f"the CSR read back from the device",
            "oracle_seconds_to_k_seeds": {
                "derive_1_thread_measured": oracle_golden_seconds(args.config),
                "verify_est_all_threads": round(dt * R / threads, 1),
                "derive_est_1_thread": round(per_sketch_1t * R, 1),
                "note": "derive_1_thread_measured: tests/golden/<cfg>.json (c1-c3); est: R sketch "
                        "labellings at the sampled rate (the selection of c4 adds seconds)"},
            **host_info()}
    if rank == 0:
        emit(line)
    ctx.close()
    if use_dist:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
