/*
 * pacim.h — C ABI of the B200-native PaC-IM hot path (arXiv 2311.07554).
 *
 * The calls follow the paper's problem statement and Alg. 1:
 *   pacim_load_graph / pacim_generate_graph   (graph G, edge model p; H0-H1)
 *   pacim_build_sketches(R, hash_seed, ...)   (Step 1: Sketch(r) for all r; H2-H7)
 *   pacim_select_seeds(k)                     (Step 2: k x NextSeed + MarkSeed; H8-H12)
 * Citation keys: P:n = PAPER.md line n; Hn = SURVEY.md §8(a) row; Rn = reading
 * n in DESIGN.md §"Readings of the paper".
 *
 * Conventions for every call:
 *  - Return value is a pacim_status; the message of the last failure is
 *    available from pacim_last_error(ctx) until the next call on that ctx.
 *    No exception or signal crosses the ABI.
 *  - "host" pointers are caller-owned CPU memory; the library copies what it
 *    needs before returning and never retains them.  "device" pointers are
 *    caller-owned CUDA memory on the ctx's device (e.g. torch tensors).
 *  - Every call is ordered on the ctx's stream and synchronises that stream
 *    before returning (outputs are ready when it returns).
 *  - One ctx per host thread; one ctx per GPU.  All device memory of a ctx is
 *    owned by it and released by pacim_destroy.
 *  - Vertex ids are uint32 < 2^31 (R2: bit 63 separates the sketch-id domain of
 *    the hash from the edge-key domain).  Edge counts are uint64.
 *  - The CSR is the symmetric simple graph: offsets u64[n+1] (offsets[0]=0,
 *    offsets[n]=nnz=2m, nondecreasing), neighbors u32[nnz], each list sorted
 *    ascending, no self-loops, no duplicates (P:1308 symmetrisation; R14).
 */
#ifndef PACIM_H
#define PACIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PACIM_API __attribute__((visibility("default")))
#else
#define PACIM_API
#endif

typedef struct pacim_ctx pacim_ctx;

typedef enum {
    PACIM_OK = 0,
    PACIM_EINVAL = -1,   /* bad argument (message names it) */
    PACIM_ENOMEM = -2,   /* device allocation failed */
    PACIM_ECUDA = -3,    /* CUDA runtime error (message has cudaGetErrorString) */
    PACIM_ESTATE = -5,   /* call out of order (load -> build -> select) */
    PACIM_ENOTIMPL = -6, /* combination not implemented */
    PACIM_ECHECK = -7,   /* an internal invariant check failed (message names it) */
    PACIM_ENCCL = -4     /* NCCL failure (message has ncclGetErrorString) */
} pacim_status;

/* Edge-probability models (P:1314-1317 constant p; P:2034 WIC). */
enum { PACIM_P_CONST = 0, PACIM_P_WIC = 1, PACIM_P_UNIFORM = 2 };
/* Synthetic generators (DESIGN.md §Input recipe). */
enum { PACIM_GEN_ER = 0, PACIM_GEN_RMAT = 1, PACIM_GEN_GRID = 2 };

typedef struct {
    /* sizes */
    uint32_t n;
    uint64_t m;                 /* undirected edges */
    uint32_t R;                 /* sketches in the job */
    uint32_t R_local;           /* sketches held by this ctx (shard) */
    uint32_t rho;               /* centers (compressed mode), else n */
    int compressed;
    uint64_t ncomp;             /* non-singleton components stored (uncompressed) */
    uint64_t nmember;           /* vertices in non-singleton components, summed over sketches */
    uint64_t live_pairs;        /* sum over local sketches of live edges (H2 count) */
    /* device time of the last build / select (CUDA events, ms) */
    double t_build_ms;
    double t_init_ms, t_edges_ms, t_compress_ms, t_compact_ms, t_gain_ms, t_centers_ms;
    double t_select_ms;
    uint64_t device_bytes;      /* bytes currently allocated by the ctx */
    uint64_t select_member_updates; /* gain updates applied by the last select */
    uint64_t select_bfs_visits;     /* Get-center / cover BFS vertex visits (compressed) */
    uint32_t kernel_launches_build; /* launches of library kernels in the last build */
    uint32_t kernel_launches_select;/* launches of library kernels in the last select */
    uint32_t rows;                  /* store rows = non-isolated vertices (isolated
                                       vertices are singletons in every sketch) */
    uint64_t nnonsingle;            /* (vertex, sketch) pairs in non-singleton CCs */
    /* cover-step diagnostics of the last select (uncompressed store) */
    uint64_t select_dense_steps;    /* steps that ran the dense pass (big CCs) */
    uint64_t select_warp_slots;     /* (step, slot) CCs enumerated by a warp-local BFS */
    uint64_t select_deferred_slots; /* (step, slot) CCs handed to the shared traversal */
    uint64_t select_row_items;      /* row expansions of the shared traversal */
    uint64_t select_chunk_items;    /* chunk items (CH-edge slices of long rows) */
    uint64_t select_inline_rows;    /* rows expanded without queueing (queue guard) */
    uint64_t select_edges;          /* CSR entries tested by the shared traversal */
    uint64_t select_center_visits;  /* compressed: Get-center vertices dequeued before a
                                       center was met, summed over probes (Thm 3.1) */
    uint64_t select_center_found;   /* compressed: probes that met a center */
    uint32_t batch_slots;           /* compressed: sketches per build batch (parent arrays
                                       rows x batch_slots u32 of scratch) */
    uint64_t select_evaluations;    /* lazy selector: fresh marginal-gain evaluations */
    uint64_t select_eval_rounds;    /* lazy selector: prefix-doubling batches */
    uint64_t hla_entries;           /* live hub adjacency of the last build: (hub, sketch,
                                       neighbour) entries, 0 if not recorded */
    uint32_t hubs;                  /* rows of degree > the hub degree (PACIM_HUB_DEG) */
    uint64_t select_hotsum_steps;   /* steps whose giant hot (hub's) CCs were covered from the
                                       build's per-vertex hot sums (compressed: no batch
                                       rebuild; uncompressed: no dense pass) */
    uint32_t lean;                  /* 1: lean graph (no edge lists; k_edges reads the CSR) */
    uint32_t store;                 /* store of the last build: 0 dense vertex-major
                                       (rows x R_local u32), 1 compact (entries only for
                                       the non-singleton (vertex, sketch) pairs, with a
                                       member index), 2 compressed (centers, Alg. 3) */
    uint32_t select_dist_replays;   /* sharded select: 1 if the fast path (fixed-size delta
                                       lists, no host sync per step) could not apply a step
                                       and the selection was re-run on the robust path */
    uint64_t device_peak_bytes;     /* high-water mark of device_bytes since the last
                                       pacim_build_sketches started (graph included) */
    uint64_t select_celf_evaluations; /* incremental selector with PACIM_CELF_COUNT=1: the
                                       re-evaluations CELF would make: at step
                                       i >= 2, every non-seed whose stale score ranks at or
                                       above the winner's fresh one (gain desc, id asc) */
    uint32_t build_hook_list;       /* dense store with slot epochs: 1 if the last build's
                                       compression read k_edges' hook list (the non-root
                                       slots) instead of streaming the store */
} pacim_stats;

/* --------------------------------------------------------------- lifecycle */

/* Create a context on CUDA device `device`.
 * workspace, ws_bytes: a caller-owned DEVICE buffer (e.g. a torch uint8
 *   tensor's data_ptr(), 256-byte aligned) from which the ctx carves every
 *   device allocation (first fit; ENOMEM when no hole is large enough), or
 *   NULL / 0 for cudaMalloc.  The caller keeps it alive until pacim_destroy.
 * cuda_stream: a cudaStream_t all work is ordered on (e.g.
 *   torch.cuda.current_stream().cuda_stream; pass cudaStreamLegacy = (void*)1
 *   for the legacy default stream, whose handle is 0), or NULL for a private
 *   non-blocking stream.
 * *out receives the ctx.  EINVAL if out is NULL, the device does not exist,
 * only one of workspace / ws_bytes is given or the workspace is misaligned;
 * ECUDA on runtime failure. */
PACIM_API int pacim_create(pacim_ctx **out, int device, void *workspace, size_t ws_bytes,
                           void *cuda_stream);

/* Free every device allocation of the ctx and the ctx itself.  NULL is a no-op. */
PACIM_API void pacim_destroy(pacim_ctx *ctx);

/* ------------------------------------------------------------ multi-GPU */
/* one process per GPU, sketches sharded r = rank (mod world)
 * over a replicated graph, NCCL over NVLink called from this library.
 *
 * pacim_nccl_unique_id: writes a new 128-byte ncclUniqueId to id_out (host
 * memory, caller-owned).  Rank 0 calls it and hands the bytes to the other
 * ranks (e.g. torch.distributed.broadcast_object_list).  EINVAL if NULL,
 * ENCCL on NCCL failure.
 *
 * pacim_init_comm: ncclCommInitRank(world, id, rank) on the ctx's device
 * (collective: every rank calls it with the same id).  Replaces an earlier
 * communicator of the ctx.  With it, a build whose (shard_rank, shard_world)
 * equals (rank, world) ends with one all-reduce of gain0 (pacim_get_gain0 then
 * returns the GLOBAL gains), and pacim_select_seeds runs the sharded greedy
 * loop: per step a fixed-size sparse delta exchange (ncclAllGather), no host
 * synchronisation per step (compact store), re-run on a dense per-step
 * all-reduce if a list overflows (pacim_stats.select_dist_replays).  Results
 * are identical on every rank and equal the one-GPU sequence.  EINVAL for a
 * bad rank / world / NULL id, ENCCL on NCCL failure.  Without a communicator
 * a sharded build keeps the per-rank step primitives below (gain0 is then the
 * rank's partial sum). */
PACIM_API int pacim_nccl_unique_id(void *id_out);
PACIM_API int pacim_init_comm(pacim_ctx *ctx, int rank, int world, const void *nccl_unique_id);

/* Message of the last failed call on ctx ("" if none).  Valid until the next
 * call on ctx.  With ctx == NULL: message of the last failed pacim_create. */
PACIM_API const char *pacim_last_error(const pacim_ctx *ctx);

/* Library version string (static storage). */
PACIM_API const char *pacim_version(void);

/* Quantise a probability to the 32-bit threshold T32 = floor(p * 2^32)
 * computed in IEEE double; p >= 1 gives 2^32 (always live), p <= 0 or NaN
 * gives 0 (R3; P:4 "hash_edge < p(u,v)"). */
PACIM_API uint64_t pacim_threshold_from_p(double p);

/* NEXT f3, R21: Monte-Carlo influence of the seed set S = seeds[0..ns) (HOST
 * array; repeated ids count once) under the IC model of the loaded graph
 * (its probability model): nsims independent worlds, simulation
 * i's edge e live iff hi32(mix64(mix64(K_mc ^ i) ^ key(e))) < T32(e),
 * K_mc = mix64(mc_seed ^ 0x4D435349434D4353).  *total (host) = the sum over
 * the worlds of |reach_i(S)|; sigma_hat(S) = *total / nsims.  Needs a loaded
 * graph (no sketches).  ESTATE without a graph, EINVAL for a seed >= n. */
PACIM_API int pacim_simulate_ic(pacim_ctx *ctx, const uint32_t *seeds, uint32_t ns,
                                uint32_t nsims, uint64_t mc_seed, uint64_t *total);

/* NEXT f2: the selector of pacim_select_seeds on an uncompressed store.
 * 0 (default) = incremental (member gains updated when a CC is covered);
 * 1 = lazy, prefix doubling (the P-tree scheme): stale upper
 *     bounds, fresh evaluations of prefixes of 1, 2, 4, ... candidates in
 *     (stale desc, id asc) order;
 * 2 = lazy, Win-Tree: an implicit winning tree over the stale
 *     bounds, FindMax pruning every subtree whose stale winner cannot beat the
 *     best fresh score (compact store; the dense store falls back to 1).
 * The lazy selectors count their re-evaluations (stats.select_evaluations;
 * Win-Tree: stats.select_eval_rounds = tree nodes explored).  With the
 * environment variable PACIM_CELF_COUNT=1 the incremental selector also counts
 * the re-evaluations CELF would make on the same gains
 * (stats.select_celf_evaluations).  All return the same sequence (R17).
 * EINVAL for another value. */
PACIM_API int pacim_set_selector(pacim_ctx *ctx, int selector);

/* NEXT f3, R20: the sampling rule of the sketches built after this call.
 * rule 0 (default) = the paper's P:3-4, hash(r) xor hash(e) < p(u,v);
 * rule 1 = decorrelated, hi32(mix64(hash(r) xor hash(e))) < T32(u,v)
 * (independent sketches; no candidate-bucket pruning, every sketch is tested
 * for every edge).  Drops built sketches (ESTATE for select until rebuilt);
 * EINVAL for another rule. */
PACIM_API int pacim_set_hash_rule(pacim_ctx *ctx, int rule);

/* The Uniform model's parameter (R19): L = floor(lo 2^32), H = min(floor(hi
 * 2^32), 2^32 - 1) in IEEE double, returned packed as H << 32 | L (L <= H);
 * lo, hi are clamped to [0, 1] and swapped if lo > hi. */
PACIM_API uint64_t pacim_threshold_uniform(double lo, double hi);

/* ------------------------------------------------------------------- graph */

/* H0/H1.  Load the symmetric CSR from HOST arrays offsets[n+1], neighbors[nnz]
 * and set the edge model: pmodel = PACIM_P_CONST with t32 = T32 in [0, 2^32]
 * (every edge live in sketch r iff hash_edge(u,v,r) < T32 * 2^32, R3),
 * or PACIM_P_WIC (t32 ignored; T32(u,v) = min(2^32, floor(2^33/(d_u+d_v))),
 * P:2034, R4), or PACIM_P_UNIFORM (p(u,v) ~ U(lo, hi) drawn from the edge key,
 * P:2032, R19: t32 = H << 32 | L from pacim_threshold_uniform, T32(u,v) =
 * L + ((H - L) * hi32(mix64((min<<32|max) ^ K_U))) >> 32).  validate: 0 = trust the caller; 1 = check offsets, id range,
 * sorted lists without loops or duplicates (EINVAL naming the first bad
 * vertex); 2 = also check symmetry.  EINVAL also for n == 0, n >= 2^31,
 * offsets[0] != 0, offsets[n] != nnz, nnz odd, t32 > 2^32.  Replaces any
 * previously loaded graph and drops existing sketches. */
PACIM_API int pacim_load_graph(pacim_ctx *ctx, uint32_t n, uint64_t nnz,
                     const uint64_t *offsets, const uint32_t *neighbors,
                     int pmodel, uint64_t t32, int validate);

/* H0, pipelined: the same load as pacim_load_graph (validate = 0), but the
 * host -> device copies are only enqueued (on a copy stream of the ctx) and the
 * call returns at once; the load is committed — copies awaited on the ctx
 * stream, the CSR swapped in, the edge lists derived — by the next
 * pacim_build_sketches (until then every other call sees the current graph),
 * so the copy of the next graph overlaps the build and selection of the
 * current one.  At most
 * two loads may be pending (ESTATE beyond); they are committed in call order.
 * The host arrays must stay valid and unmodified until the load is committed;
 * they should be pinned (page-locked), else the copy does not overlap.  EINVAL
 * as for pacim_load_graph (offsets[0], offsets[n], nnz, n, t32 checks). */
PACIM_API int pacim_load_graph_async(pacim_ctx *ctx, uint32_t n, uint64_t nnz,
                                     const uint64_t *offsets, const uint32_t *neighbors,
                                     int pmodel, uint64_t t32);

/* H0 from the UPPER CSR: each undirected edge {u, v} given once, in row
 * min(u, v) — uoffsets[n+1] (host, uoffsets[0] = 0, uoffsets[n] = m), and
 * uneighbors[m] (host): row u lists its neighbours v > u in increasing order.
 * Half the bytes of the symmetric CSR cross PCIe.  The upper CSR stays on the
 * device (SURVEY H0's build input: the dense store's build and the Win-Tree
 * selection read only the upper edges); the symmetric offsets come from the
 * degrees at once, and the symmetric neighbour lists (lower lists by a
 * transpose: stable radix sort of the upper pairs by target; rows = sorted
 * lower ++ upper) are built on the device only when something reads them
 * (traversal selections, Get-center probes, Monte Carlo, pacim_get_graph) —
 * the graph is exactly the one pacim_load_graph would load from the
 * symmetric CSR of the same edge set ("symmetrize", R14).  The
 * transpose needs 16 B of device scratch per edge (ENOMEM beyond: send the
 * symmetric CSR instead).  validate: 0 = trust
 * the caller; != 0 = check offsets, 0 <= u < v < n and strictly increasing
 * rows on the device (EINVAL naming the first bad vertex).  Other EINVAL and
 * the model as for pacim_load_graph; m = 0 is allowed (n isolated vertices).
 * The caller keeps ownership of the host arrays. */
PACIM_API int pacim_load_graph_upper(pacim_ctx *ctx, uint32_t n, uint64_t m,
                                     const uint64_t *uoffsets, const uint32_t *uneighbors,
                                     int pmodel, uint64_t t32, int validate);

/* Pipelined pacim_load_graph_upper (validate = 0): the copies of the upper
 * CSR are enqueued on the copy stream like pacim_load_graph_async; the next
 * pacim_build_sketches commits the load (degrees, symmetric offsets, the
 * build's edge form; the symmetric lists on first read, as above).  Same rules as pacim_load_graph_async (at most two
 * pending loads, host arrays valid and unmodified until committed, pinned
 * for overlap). */
PACIM_API int pacim_load_graph_upper_async(pacim_ctx *ctx, uint32_t n, uint64_t m,
                                           const uint64_t *uoffsets,
                                           const uint32_t *uneighbors, int pmodel,
                                           uint64_t t32);

/* As pacim_load_graph but offsets/neighbors are DEVICE pointers on the ctx's
 * device (copied device-to-device; the caller keeps ownership). */
PACIM_API int pacim_load_graph_device(pacim_ctx *ctx, uint32_t n, uint64_t nnz,
                            const uint64_t *d_offsets, const uint32_t *d_neighbors,
                            int pmodel, uint64_t t32, int validate);

/* H0 on the device: generate a synthetic graph (DESIGN.md §Input recipe) and
 * load it with edge model (pmodel, t32).  params (host, nparams entries):
 *   PACIM_GEN_ER:   {n, m}                       first m distinct pairs
 *   PACIM_GEN_RMAT: {scale, ef, ta, tab, tabc, permute}  53-bit quadrant thresholds
 *   PACIM_GEN_GRID: {W, H, d32}                  diagonal iff hash < d32
 * gen_seed keys the counter-based draws.  EINVAL for bad params / sizes. */
PACIM_API int pacim_generate_graph(pacim_ctx *ctx, int kind, const uint64_t *params,
                         int nparams, uint64_t gen_seed, int pmodel, uint64_t t32);

/* Sizes of the loaded graph (host outputs; either may be NULL). ESTATE if none. */
PACIM_API int pacim_graph_info(pacim_ctx *ctx, uint32_t *n, uint64_t *m);

/* Copy the loaded CSR to HOST arrays offsets_out[n+1], neighbors_out[2m]
 * (either may be NULL).  ESTATE if no graph. */
PACIM_API int pacim_get_graph(pacim_ctx *ctx, uint64_t *offsets_out, uint32_t *neighbors_out);

/* -------------------------------------------------------------- sketches */

/* Step 1 of Alg. 1: build this ctx's sketches, Sketch(r) for
 * every r in [0, R) with r % shard_world == shard_rank (shard_world = 1: all).
 * Sketch r is the CC structure of G'_r = {e : hash_edge(e, r) < T32(e)*2^32}
 * with K = mix64(hash_seed) keying both hash(r) and hash(edge) (R1, R2).
 * center_a32 selects the store (Thm 3.1):
 *   >= 2^32 : uncompressed (alpha = 1): per-vertex CC labels + sizes + member
 *             index (InfuserMG-style memo; H4-H6u);
 *   < 2^32  : compressed: v is a center iff hi32(mix64(v ^ K_c)) < center_a32
 *             (R9, alpha ~ center_a32 / 2^32); per sketch label[i], size[i]
 *             over centers only (H6c).
 * Also computes the initial gains gain0[v] = sum_{own r} |C_r(v)| (int64;
 * = R * Marginal(empty, v); H7).  EINVAL: R == 0,
 * shard_world == 0, shard_rank >= shard_world; ESTATE: no graph; ENOMEM if
 * the store does not fit. */
PACIM_API int pacim_build_sketches(pacim_ctx *ctx, uint32_t R, uint64_t hash_seed,
                         uint64_t center_a32, uint32_t shard_rank,
                         uint32_t shard_world);

/* ------------------------------------------------------------- selection */

/* Step 2 of Alg. 1 on a single ctx holding all R sketches
 * (shard_world == 1): k greedy steps, each picking the smallest-id vertex not
 * in S with maximal marginal gain (R5, R6), marking its CC
 * covered in every sketch (MarkSeed) and updating the gains of the
 * covered CCs' members (H8-H10).  HOST outputs (k entries each; sigma_out may
 * be NULL): seeds_out[i]; gain_num_out[i] = sum_r delta_r = R * Marginal(S_i, s_i)
 * (integer numerator, R7); sigma_num_out[i] = cumulative sum; sigma_out[i] =
 * sigma_num_out[i] / R.  Every call starts from S = empty (the store is
 * restored).  EINVAL: k == 0 or k > n or an output NULL; ESTATE: no sketches
 * or sharded build; ECHECK if sum_r delta_r != gain[s] (never expected). */
PACIM_API int pacim_select_seeds(pacim_ctx *ctx, uint32_t k, uint32_t *seeds_out,
                       int64_t *gain_num_out, int64_t *sigma_num_out,
                       double *sigma_out);

/* --------------------------------------------- multi-rank step primitives */
/* For sketches sharded over ranks (shard_world > 1) the host runs the greedy
 * loop and performs the collectives (paper_2311_07554_b200/dist.py); these
 * calls are this rank's part of a step.  All pointers are DEVICE pointers. */

/* Copy this rank's partial gain0 (n x int64) into d_out. ESTATE if no sketches. */
PACIM_API int pacim_gain0_to_device(pacim_ctx *ctx, int64_t *d_out);

/* Restore the covered flags of the store (start a new selection, S = empty). */
PACIM_API int pacim_select_reset(pacim_ctx *ctx);

/* MarkSeed(s) on this rank's sketches: for every own sketch where
 * C_r(s) is not yet covered, mark it covered and add -|C_r(s)| into d_delta[u]
 * for every member u (d_delta: n x int64, accumulated, not cleared).
 * *local_gain (host) receives sum over own sketches of delta_r. */
PACIM_API int pacim_cover_local(pacim_ctx *ctx, uint32_t s, int64_t *d_delta,
                      int64_t *local_gain);

/* pacim_cover_local plus the same updates as a sparse list (SURVEY §8(e)
 * sparse per-step deltas): every update d_delta[u] += -delta is also written
 * as d_list_v[i] = u, d_list_d[i] = -delta (u32 / int64 DEVICE arrays of
 * `cap` entries; duplicates of u are allowed and add up).  *count (host)
 * receives the number of updates; when *count > cap the list is incomplete
 * and the caller must use d_delta (dense fallback).  *local_gain as above. */
PACIM_API int pacim_cover_local_sparse(pacim_ctx *ctx, uint32_t s, int64_t *d_delta,
                                       uint32_t *d_list_v, int64_t *d_list_d, uint64_t cap,
                                       uint64_t *count, int64_t *local_gain);

/* d_gain[v[i]] += d[i] for i < count (the gathered lists of all ranks,
 * duplicates add up), then d_gain[s] = -1 (the seed leaves the candidates,
 * R6) unless s == 0xFFFFFFFF.  DEVICE arrays. */
PACIM_API int pacim_apply_deltas(pacim_ctx *ctx, int64_t *d_gain, const uint32_t *d_v,
                                 const int64_t *d_d, uint64_t count, uint32_t s);

/* Dense fallback: d_gain += d_delta, d_delta = 0 (n entries), then
 * d_gain[s] = -1 unless s == 0xFFFFFFFF.  DEVICE arrays. */
PACIM_API int pacim_apply_dense(pacim_ctx *ctx, int64_t *d_gain, int64_t *d_delta, uint32_t n,
                                uint32_t s);

/* d_delta[v[i]] = 0 for i < count: clears the dense delta after a sparse step. */
PACIM_API int pacim_clear_deltas(pacim_ctx *ctx, int64_t *d_delta, const uint32_t *d_v,
                                 uint64_t count);

/* NextSeed by full scan (H8): *s_out = smallest v with maximal d_gain[v]
 * (entries < 0 never win unless all are), *g_out = d_gain[*s_out]. */
PACIM_API int pacim_argmax_device(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n,
                        uint32_t *s_out, int64_t *g_out);

/* ------------------------------------------------------------ inspection */

/* gain0 (n x int64) to HOST. ESTATE if no sketches. */
PACIM_API int pacim_get_gain0(pacim_ctx *ctx, int64_t *out);

/* Canonical labels of sketch r (uncompressed store): out[v] = smallest vertex
 * id of v's CC in G'_r (R8); HOST out[n].  EINVAL if r is not held by this
 * ctx; ENOTIMPL in compressed mode. */
PACIM_API int pacim_get_labels(pacim_ctx *ctx, uint32_t r, uint32_t *out);

/* Compressed sketch r: label_out[i], size_out[i] for the rho centers in
 * vertex order; HOST arrays of rho entries (rho from
 * pacim_get_stats).  Sizes reflect covered CCs of the last selection. */
PACIM_API int pacim_get_center_sketch(pacim_ctx *ctx, uint32_t r, uint32_t *label_out,
                            uint32_t *size_out);

/* Counters and device timings of the last build/select (HOST *out). */
PACIM_API int pacim_get_stats(pacim_ctx *ctx, pacim_stats *out);

#ifdef __cplusplus
}
#endif

#endif /* PACIM_H */
