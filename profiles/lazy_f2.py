"""the lazy (CELF-style) selector against the incremental
one on the same store: evaluations (the paper's re-evaluation counts,
P:1662-1693: social/web graphs need ~n evaluations over k = 100, road
graphs ~140), prefix-doubling rounds, time, and identical seeds (R17).

    python profiles/lazy_f2.py c2 c3 c4 > profiles/rNN_lazy.md
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402


def main():
    import paper_2311_07554_b200 as P
    from paper_2311_07554_b200 import pipeline
    print("# f2 — lazy vs incremental selection, B200, 1 GPU, uncompressed store\n")
    print("| config | n | k | incremental select ms | lazy select ms | evaluations "
          "| evaluations / n | doubling rounds | same seeds |")
    print("|---|---|---|---|---|---|---|---|---|")
    for name in sys.argv[1:] or ["c2"]:
        cfg = inputs.config(name)
        ctx = P.Context(0)
        n, m = pipeline.generate(ctx, cfg)
        ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"])
        k = cfg["k"]
        a = ctx.pacim_select_seeds(k)
        ti = ctx.pacim_get_stats()["t_select_ms"]
        ctx.pacim_set_selector(1)
        b = ctx.pacim_select_seeds(k)
        st = ctx.pacim_get_stats()
        ctx.pacim_set_selector(0)
        same = list(a[0]) == list(b[0]) and list(a[1]) == list(b[1])
        print(f"| {name} | {n} | {k} | {ti:.1f} | {st['t_select_ms']:.1f} | "
              f"{st['select_evaluations']} | {st['select_evaluations'] / n:.3f} | "
              f"{st['select_eval_rounds']} | {same} |")
        ctx.close()


if __name__ == "__main__":
    main()
