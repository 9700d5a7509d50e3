"""influence quality of the seed sets: the paper's literal
rule vs the decorrelated rule (R20), each judged by Monte-Carlo
sigma(S) (R21, independent worlds) at k' = 1, 10, 50, 100, next to the
sketch estimate sigma_num / R.  Also the build/select time of each rule.

    python profiles/quality_f3.py --config c2 [--sims 2048] > profiles/rNN_quality_c2.md
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--sims", type=int, default=2048)
    a = ap.parse_args()
    import paper_2311_07554_b200 as P
    from paper_2311_07554_b200 import pipeline
    cfg = inputs.config(a.config, **({"scale": a.scale} if a.scale else {}))
    ctx = P.Context(0)
    n, m = pipeline.generate(ctx, cfg)
    k, R = cfg["k"], cfg["R"]
    print(f"# f3 quality — {cfg['name']} (n = {n}, m = {m}, R = {R}, k = {k}), B200\n")
    print(f"Monte-Carlo sigma(S) over {a.sims} independent worlds (R21, mc_seed 7); "
          "sketch estimate = sigma_num / R of the greedy.\n")
    print("| rule | build ms | select ms | k' | sketch sigma_hat | MC sigma | MC std err |")
    print("|---|---|---|---|---|---|---|")
    for rule, name in ((0, "literal P:3-4"), (1, "decorrelated R20")):
        ctx.pacim_set_hash_rule(rule)
        ctx.pacim_build_sketches(R, cfg["hash_seed"], pipeline.center_a32_of(cfg))
        seeds, gain, signum, sigma = ctx.pacim_select_seeds(k)
        st = ctx.pacim_get_stats()
        for kk in (1, 10, 50, k):
            if kk > k:
                continue
            S = [int(x) for x in seeds[:kk]]
            tot = ctx.pacim_simulate_ic(S, a.sims, 7)
            # standard error from 8 independent blocks of sims / 8 worlds
            blk = [ctx.pacim_simulate_ic(S, a.sims // 8, 1000 + b) / (a.sims // 8) for b in range(8)]
            mu = sum(blk) / 8
            se = math.sqrt(sum((x - mu) ** 2 for x in blk) / 7 / 8)
            print(f"| {name} | {st['t_build_ms']:.1f} | {st['t_select_ms']:.1f} | {kk} "
                  f"| {sigma[kk - 1]:.1f} | {tot / a.sims:.1f} | {se:.1f} |")
    ctx.pacim_set_hash_rule(0)
    ctx.close()


if __name__ == "__main__":
    main()
