"""Edge-partitioned sharded build (dist.cu pc_cs_ep_pairs), measured on ONE
GPU at world 1 (PACIM_FORCE_DIST + PACIM_EP: the rank tests all edges against
all R sketches, the exchange is a device copy) beside the mask-pass compact
build of the same shard, with PACIM_BUILD_TIMES phase marks on stderr.

At P ranks the EP pass of a rank covers 1/P of the edges for all R sketches
(its work divides by P: the pass is a stream over the edge range); what the
rank does after the exchange is the build of its R/P sketches from their
live pairs (profiles/shard_build.py measures that shard's phases).

    python profiles/ep_build.py c4 > profiles/rNN_ep_build_c4.md 2> ep.err
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402


def main():
    os.environ["PACIM_FORCE_DIST"] = "1"
    os.environ["PACIM_STORE"] = "compact"
    os.environ["PACIM_BUILD_TIMES"] = "1"
    import paper_2311_07554_b200 as P
    from paper_2311_07554_b200 import pacim_nccl_unique_id, pipeline
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    cfg = inputs.config(name)
    ctx = P.Context(0)
    ctx.pacim_init_comm(0, 1, pacim_nccl_unique_id())
    n, m = pipeline.generate(ctx, cfg)
    print(f"# edge-partitioned build at world 1 — {cfg['name']} (n = {n}, m = {m}, R = {cfg['R']}), one B200\n")
    print("| build | build ms (best of 3) | pairs pass ms | rest ms | live pairs | device GB |")
    print("|---|---|---|---|---|---|")
    for ep in ("0", "1"):
        os.environ["PACIM_EP"] = ep
        best = None
        for _ in range(3):
            ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"], 1 << 32, 0, 1)
            st = ctx.pacim_get_stats()
            if best is None or st["t_build_ms"] < best["t_build_ms"]:
                best = dict(st)
        st = best
        label = "edge-partitioned (pairs of all edges x all sketches, exchange, masks from pairs)" \
            if ep == "1" else "mask pass over all edges (per-rank scheme)"
        print(f"| {label} | {st['t_build_ms']:.1f} | {st['t_init_ms']:.1f} | "
              f"{st['t_build_ms'] - st['t_init_ms']:.1f} | {st['live_pairs']} | "
              f"{st['device_bytes'] / 1e9:.1f} |")
    ctx.close()


if __name__ == "__main__":
    main()
