"""Per-rank cost of a sharded build, measured on ONE GPU: the
build of rank 0's shard (sketches r = 0 mod P) for P = 1, 2, 4, 8 — the
build has no communication before the gain0 all-reduce, so rank 0's build
time on one B200 is its time in a P-GPU job.  With P > 1 the shard takes the
compact store (the sharded NCCL select walks its member lists).  Also the
gain0 all-reduce volume (8n bytes) and the store's bytes per rank.

    python profiles/shard_build.py c4 [compact|dense] > profiles/rNN_shard_build_c4.md

The second argument forces the store of the P > 1 shards (PACIM_STORE).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402


def main():
    import paper_2311_07554_b200 as P
    from paper_2311_07554_b200 import pipeline
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    if len(sys.argv) > 2:
        os.environ["PACIM_STORE"] = sys.argv[2]
    worlds = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8]
    cfg = inputs.config(name)
    ctx = P.Context(0)
    n, m = pipeline.generate(ctx, cfg)
    print(f"# per-rank sharded build — {cfg['name']} (n = {n}, m = {m}, R = {cfg['R']}), one B200\n")
    print("| P | sketches on rank 0 | store | build ms (best of 3) | mask / init ms | edges ms | "
          "compress ms | gain ms | store + lists GB | device GB |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for world in worlds:
        best = None
        for _ in range(3):
            ctx.pacim_build_sketches(cfg["R"], cfg["hash_seed"], 1 << 32, 0, world)
            st = ctx.pacim_get_stats()
            if best is None or st["t_build_ms"] < best["t_build_ms"]:
                best = dict(st)
        st = best
        B = st["R_local"]
        store = (12 * st["nnonsingle"] + st["rows"] * ((B + 31) // 32) * 8) if st["store"] == 1 \
            else 4 * st["rows"] * B
        print(f"| {world} | {B} | {'compact' if st['store'] == 1 else 'dense'} | {st['t_build_ms']:.1f} | "
              f"{st['t_init_ms']:.1f} | {st['t_edges_ms']:.1f} | {st['t_compress_ms']:.1f} | "
              f"{st['t_gain_ms']:.1f} | {store / 1e9:.2f} | {st['device_bytes'] / 1e9:.1f} |")
    print(f"\ngain0 all-reduce per build: {8 * n / 1e9:.3f} GB (int64 x n).")
    ctx.close()


if __name__ == "__main__":
    main()
