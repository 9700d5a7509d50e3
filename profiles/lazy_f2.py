"""the lazy selectors against the incremental one on the
same store, with CELF's evaluation count on the same gains:

* incremental (selector 0): member gains updated when a CC is covered; with
  PACIM_CELF_COUNT=1 it also counts the re-evaluations CELF would make
  (every non-seed whose stale score ranks at or above the step's winner);
* prefix doubling (selector 1, the P-tree scheme);
* Win-Tree (selector 2).

Each config runs twice: on the compact store (PACIM_STORE=compact; its
incremental selector carries the CELF counter) and on the dense store (the
one-GPU default; the CELF count of the compact run is the denominator, the
gains being identical).

The paper reports P-tree / Win-Tree evaluations at 1.03x / 1.7x CELF's
(P:1715-1720).  Re-evaluations exclude the initial n evaluations (gain0).

    python profiles/lazy_f2.py c2 c4 > profiles/rNN_lazy.md
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402


def main():
    os.environ["PACIM_CELF_COUNT"] = "1"
    import paper_2311_07554_b200 as P
    from paper_2311_07554_b200 import pipeline
    print("# f2 — lazy selectors vs incremental, with CELF's count, B200, 1 GPU\n")
    print("| config | store | n | k | incremental ms | CELF re-evals | prefix-doubling ms | "
          "its re-evals | / CELF | Win-Tree ms | its re-evals | / CELF | tree nodes | same seeds |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    celf_of = {}
    for name, store in [(c, s) for c in (sys.argv[1:] or ["c2"]) for s in ("compact", "dense")]:
        os.environ["PACIM_STORE"] = store
        cfg = inputs.config(name)
        ctx = P.Context(0)
        n, m = pipeline.generate(ctx, cfg)
        ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"])
        k = cfg["k"]
        a = ctx.pacim_select_seeds(k)
        st = ctx.pacim_get_stats()
        ti, store = st["t_select_ms"], st["store"]
        celf = celf_of.setdefault(name, st["select_celf_evaluations"])
        res = []
        for sel in (1, 2):
            ctx.pacim_set_selector(sel)
            b = ctx.pacim_select_seeds(k)
            s2 = ctx.pacim_get_stats()
            same = list(a[0]) == list(b[0]) and list(a[1]) == list(b[1])
            res.append((s2["t_select_ms"], s2["select_evaluations"], s2["select_eval_rounds"], same))
        ctx.pacim_set_selector(0)
        (t1, e1, _, ok1), (t2, e2, nodes, ok2) = res
        r1 = e1 / celf if celf else float("nan")
        r2 = e2 / celf if celf else float("nan")
        print(f"| {name} | {'compact' if store == 1 else 'dense'} | {n} | {k} | {ti:.1f} | {celf} | "
              f"{t1:.1f} | {e1} | {r1:.2f} | {t2:.1f} | {e2} | {r2:.2f} | {nodes} | {ok1 and ok2} |")
        ctx.close()


if __name__ == "__main__":
    main()
