"""the compression sweep (Thm 3.1):
alpha in {1, 1/2, 1/4, 1/8, 1/16, 1/32} on one config; per alpha the store's
device bytes, build and select time, the mean Get-center visits until a
center is met (Thm 3.1: about 1/alpha), and whether the seeds equal the
uncompressed run's (compression is transparent, R17).

    python profiles/alpha_sweep.py --config c2 [--scale S] [--k K] > profiles/rNN_alpha_c2.md
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--alphas", default="1,0.5,0.25,0.125,0.0625,0.03125")
    a = ap.parse_args()
    import paper_2311_07554_b200 as P
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config(a.config, **({"scale": a.scale} if a.scale else {}))
    k = a.k or cfg["k"]
    ctx = P.Context(0)
    n, m = pipeline.generate(ctx, cfg)
    ctx.close()
    print(f"# alpha sweep — {cfg['name']}" + (f" scale {a.scale}" if a.scale else "")
          + f" (n = {n}, m = {m}, R = {cfg['R']}, k = {k}), B200, 1 GPU\n")
    print("Get-center visits / probe: vertices dequeued before a center is met (centers are\n"
          "recognised when discovered, so a center among the seed's live neighbours costs 0);\n"
          "Thm 3.1 bounds the expected visits by about 1/alpha.  Device total = every buffer\n"
          "the ctx holds (graph, store, selection state, scratch).\n")
    print("Store: alpha < 1: label + size (one u32 each, the covered flag in the size word) per\n"
          "(center, sketch); alpha = 1: the uncompressed store of a one-GPU build (dense\n"
          "vertex-major: one u32 per (non-isolated vertex, sketch)).\n"
          "Peak = the high-water mark of the ctx's device bytes over build + select (graph\n"
          "included; pacim_stats.device_peak_bytes).\n")
    print("| alpha | rho (centers) | sketch store (GB) | build scratch (GB) | device total (GB) "
          "| device peak (GB) | build ms | select ms | Get-center visits / probe | 1/alpha "
          "| seeds = alpha 1 |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    ref = None
    for al in [float(x) for x in a.alphas.split(",")]:
        # a fresh context per alpha: the peak is this alpha's alone (a ctx keeps
        # buffer capacity across builds)
        ctx = P.Context(0)
        ctx.pacim_set_selector(3)  # auto, as bench.py (alpha = 1 under WIC: the Win-Tree)
        pipeline.generate(ctx, cfg)
        a32 = 1 << 32 if al >= 1 else int(al * 4294967296.0)
        tb, ts = [], []
        for _ in range(a.reps):
            ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"], a32)
            out = ctx.pacim_select_seeds(k)
            st = ctx.pacim_get_stats()
            tb.append(st["t_build_ms"])
            ts.append(st["t_select_ms"])
        B = st["R_local"]
        if st["compressed"]:
            store = 2 * st["rho"] * B * 4  # label, size (+ covered bit) per (center, slot)
            scratch = (st["rows"] + st["rho"]) * st["batch_slots"] * 4  # one build batch
            vis = st["select_center_visits"] / max(st["select_center_found"], 1)
        elif st["store"] == 1:
            store = 12 * st["nnonsingle"] + st["rows"] * ((B + 31) // 32) * 8
            scratch = 4 * st["nnonsingle"]  # ranks in the CCs (member index build)
            vis = float("nan")
        else:
            store = st["rows"] * B * 4
            scratch = 0
            vis = float("nan")
        seeds = [int(x) for x in out[0]]
        if ref is None:
            ref = seeds
        print(f"| {al:g} | {st['rho']} | {store / 1e9:.3f} | {scratch / 1e9:.3f} "
              f"| {st['device_bytes'] / 1e9:.2f} | {st['device_peak_bytes'] / 1e9:.2f} "
              f"| {min(tb):.1f} | {min(ts):.1f} | {vis:.2f} | {1 / al:g} | {seeds == ref} |")
        ctx.close()


if __name__ == "__main__":
    main()
