// pacim_internal.cuh — device helpers and the context of the B200 CUDA path.
//
// This is the PRODUCT path.  It shares nothing with oracle/ (its own hash,
// generator and graph code are written here, from the paper and DESIGN.md's
// readings).  Citation keys: P:n = PAPER.md line n; Hn = SURVEY.md §8(a) row;
// Rn = DESIGN.md reading n.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/pacim.h"

// Root-slot marker of the uncompressed store (DESIGN.md §Store layout):
//   slot(v, j) == v            v is a singleton in sketch j
//   slot(v, j) & PACIM_HIGH    v is the root (min id) of a non-singleton CC;
//                              low 31 bits = CC size (after compress_count) or
//                              compact component index ci (after compact)
//   otherwise                  slot(v, j) = root id of v's CC (< v)
#define PACIM_HIGH 0x80000000u
#define PACIM_LOW 0x7FFFFFFFu

// Slot epochs of the dense store (build.cu pc_build): the
// `mask` bits just below bit 30 (COV) of every slot hold the epoch of the
// build that last wrote it; a slot whose epoch differs from the current
// build's (`tag`) reads as a singleton root (HIGH | 1), so a build needs no
// pass that resets the store — one full reset per 2^bits builds.  Ep{}
// (mask 0) reads every slot as stored (stores reset in line).
struct Ep {
  uint32_t tag = 0, mask = 0;
};
__host__ __device__ __forceinline__ uint32_t ep_rd(uint32_t raw, Ep e) {
  return (raw & e.mask) == e.tag ? (raw & ~e.mask) : (PACIM_HIGH | 1u);
}
#define PACIM_TB 12  // bits of the sketch bucket table (R2 candidate enumeration)
#define PACIM_HUBF 0x80000000u  // hub flag of a row in ckeys
// Components of at least max(PACIM_BIG_MIN, n / PACIM_BIG_DIV) vertices are
// not put in the member index; MarkSeed covers them with one dense pass over
// the store (coff = PACIM_BIG marks them).
#define PACIM_BIG_MIN 4096u
#define PACIM_BIG_DIV 256u
#define PACIM_BIG 0xFFFFFFFFFFFFFFFFull

// ------------------------------------------------------------------ hash (R1)
__host__ __device__ __forceinline__ uint64_t pc_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// R19: Uniform U(lo, hi) threshold of edge key (min<<32 | max), packed = H<<32|L
#define PACIM_K_U_SEED 0x5EED0F0DDBA11E55ull
__host__ __device__ __forceinline__ uint64_t pc_t32_uniform(uint64_t packed, uint64_t key) {
  const uint64_t L = packed & 0xFFFFFFFFull, H = packed >> 32;
  const uint64_t x = pc_mix64(key ^ pc_mix64(PACIM_K_U_SEED)) >> 32;
  return L + (((H - L) * x) >> 32);
}

// ------------------------------------------------------------ error helpers
struct PacimError {
  int code;
  std::string msg;
};

#define PC_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      throw PacimError{e_ == cudaErrorMemoryAllocation ? PACIM_ENOMEM        \
                                                       : PACIM_ECUDA,        \
                       std::string(#call) + ": " + cudaGetErrorString(e_)};  \
  } while (0)

#define PC_CHECK_LAUNCH() PC_CUDA(cudaGetLastError())

#define PC_REQUIRE(cond, code, msg)                                           \
  do {                                                                        \
    if (!(cond)) throw PacimError{code, msg};                                 \
  } while (0)

// store address of (row, slot j) under the window layout (smap = d_smap)
__device__ __forceinline__ size_t pc_addr(const uint32_t *smap, uint32_t nr, uint32_t row,
                                          uint32_t j) {
  const uint32_t fc = smap[j], f = fc >> 16, c = fc & 0xFFFFu;
  return (size_t)nr * f + (size_t)row * c + (j - f);
}

// compact store (store_cs.cu): entry of (row, slot j) given the row's record
// words rec[row * MW + w] = {entries of the rows before + set bits of the row's
// words before w, live-slot mask word w}
__device__ __forceinline__ uint32_t pc_cs_pos(const uint2 *rec, uint32_t MW, uint32_t row,
                                              uint32_t j) {
  const uint2 r = rec[(size_t)row * MW + (j >> 5)];
  return r.x + __popc(r.y & ((1u << (j & 31)) - 1u));
}

// ------------------------------------------------------- device allocation
struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  template <typename T>
  T *as() const { return reinterpret_cast<T *>(p); }
};

// Sparse per-step deltas of a multi-rank greedy step: every
// gain update u -= delta of a cover step is also appended as (u, -delta)
// (duplicates allowed; their sum is the dense delta).  Entries past cap are
// dropped and counted, so cnt > cap tells the caller to use the dense vector.
struct DeltaList {
  uint32_t *v = nullptr;
  long long *d = nullptr;
  unsigned long long *cnt = nullptr;
  unsigned long long cap = 0;
  __device__ __forceinline__ void add(uint32_t u, long long delta) const {
    if (!v) return;
    const unsigned long long at = atomicAdd(cnt, 1ull);
    if (at < cap) {
      v[at] = u;
      d[at] = delta;
    }
  }
};

// a graph load in flight (pacim_load_graph_async): the host CSR copied into
// these buffers on the copy stream, committed by the next call needing the graph
struct StagedGraph {
  DevBuf off, nbr;  // the CSR as sent (upper: the upper CSR, symmetrized at commit)
  bool upper = false;
  cudaEvent_t done = nullptr;  // recorded on the copy stream after the copies
  bool pending = false;
  uint32_t n = 0;
  uint64_t nnz = 0;
  int pmodel = 0;
  uint64_t t32 = 0;
};

struct pacim_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // caller-owned workspace (pacim_create): every device buffer is carved
  // from it (first fit, 256-B aligned) instead of cudaMalloc
  void *ws_base = nullptr;
  size_t ws_bytes = 0;
  std::map<size_t, size_t> ws_free, ws_used;  // offset -> length
  std::string err;
  int sm_count = 148;
  uint64_t device_bytes = 0;
  uint64_t device_peak = 0;  // high-water mark since the last build started
  // cudaMemGetInfo, cached: on the B200 boxes one call took 4-18 ms with
  // ~100 GB allocated (c4), inside every build.  Free memory is re-queried at
  // graph loads / generation / failed allocations and tracked through this
  // ctx's own allocations in between (pc_mem_info)
  bool mi_valid = false;
  size_t mi_free = 0, mi_total = 0;
  uint64_t mi_dev_bytes = 0;

  // ---- multi-GPU (dist.cu): NCCL communicator of pacim_init_comm
  void *comm = nullptr;     // ncclComm_t
  int comm_rank = 0, comm_world = 1;
  bool dist_hot = false;    // dist_ghot holds the all-reduced hot sums
  DevBuf dist_ghot;         // i64[n]
  DevBuf dist_buf;          // fast sharded select: chunk cache, lists, messages, state
  DevBuf dist_cov_old;      // u64: covered root entries of the last fast select
  unsigned long long dist_cov_n = 0;
  bool dist_cov_valid = false;
  // the fast select's k-step loop captured once as a CUDA graph (per-step
  // launch overhead), replayed while its arguments are unchanged
  DevBuf ep_tab;            // edge-partitioned build: global slot table, owner map
  DevBuf ep_send;           // ... the pairs grouped by owner rank
  DevBuf ep_cnt;            // ... per-owner counts / cursors, all ranks' counts
  unsigned long long ep_hint = 0;  // list slots the last EP pass reserved (same graph, key)
  uint64_t ep_gen = ~0ull, ep_K = 0;
  cudaStream_t dist_cap_stream = nullptr;
  void *dist_graph = nullptr;              // cudaGraphExec_t
  std::vector<unsigned char> dist_graph_key;

  // ---- graph (H0/H1)
  bool has_graph = false;
  uint64_t graph_gen = 0;  // incremented by every graph load (derived-table caches)
  // strategy hints of the builds (store choice, slot epochs, list capacities)
  // are remembered per hint_gen: it changes only when a load brings a graph of
  // another shape (n, m, rows, edge model) — the same graph loaded again (the
  // e2e loop) keeps the measured choices
  uint64_t hint_gen = 0;
  uint64_t graph_sig = 0;
  uint32_t n = 0;
  uint64_t m = 0;        // undirected edges
  int pmodel = 0;        // PACIM_P_CONST / PACIM_P_WIC / PACIM_P_UNIFORM
  // per-edge thresholds (WIC, Uniform) are stored as T32 - toff in u32
  // (WIC: T32 in [1, 2^32], toff = 1; Uniform: T32 in [0, 2^32 - 1], toff = 0)
  uint32_t toff() const { return pmodel == PACIM_P_WIC ? 1u : 0u; }
  uint64_t t32 = 0;      // constant threshold (R3)
  DevBuf off;            // u64[n+1] full CSR offsets
  DevBuf nbr;            // u32[2m]  full CSR neighbours
  DevBuf keys;           // u64[m]   upper edge list min<<32|max, sorted
  DevBuf tm1;            // u32[m]   per-edge models: T32(e) - toff()
  DevBuf tcsr;           // u32[2m]  per-edge models: T32 - toff() per CSR entry (traversals)
  DevBuf ckeys;          // u64[m]   the same edges as store rows: row(min)<<32|row(max);
                         //          bit 31 of a half flags a hub row (PACIM_HUBF)
  DevBuf uoff;           // u64[n+1] exclusive prefix of the upper degrees (UpperCsr)
  DevBuf ucrow;          // u32      row of every 32nd upper edge (UpperCsr)
  DevBuf rk;             // uint2[n/32+1] rank map vertex -> store row (UpperCsr)
  DevBuf unbr;           // u32[m]   upper neighbours in upper-edge order (UpperCsr)
  DevBuf ud16;           // u16[m]   vertex / row deltas of upper edge e from chunk e >> 5
  DevBuf ucrowr;         // u32      store row of ucrow[c]
  DevBuf uvrow;          // u32[m]   store row of unbr[e] (PACIM_UCSR=2: from the rank map)
  DevBuf cid;            // u32[n]   store row of v, or 0xFFFFFFFF for isolated v
  DevBuf rmap;           // u32[nr]  vertex id of store row c
  uint32_t nr = 0;       // store rows = non-isolated vertices (order kept)
  bool lean = false;     // no keys / ckeys: rows = vertex ids, k_edges reads the CSR (c5)
  DevBuf vinfo;          // u64[n] degree << 32 | store row (+ hub flag), for the load's edge pass
  DevBuf crow;           // u32 row of the first CSR entry of each 32-entry chunk (lane-per-entry
                         // kernels; lean graphs: k_edges)
  uint32_t hub_row = 0xFFFFFFFFu;  // store row of the hub vertex
  uint64_t hub_degree = 0;         // its degree

  // hub rows (degree > hub_deg): index per row and the live hub adjacency of
  // the last build (HLA: per (hub, slot) the rows joined to the hub by a live
  // edge), used by the cover traversal instead of hashing the
  // hub's whole adjacency
  uint64_t hub_deg = 2048;
  uint32_t nhub = 0;
  uint64_t hub_entries = 0;  // CSR entries of the hub rows
  DevBuf hidx;           // u32[nr] hub index of a row or 0xFFFFFFFF
  DevBuf hub_tab;        // u64[hub_mask + 1] hash table (row << 32 | hub index), empty = ~0
  uint32_t hub_mask = 0;
  bool hla_ok = false;   // HLA built for the current store
  uint64_t hla_n = 0;    // live (hub, slot, row) entries
  DevBuf hla_off;        // u64[nhub * B + 1] segment offsets by (hub, slot)
  DevBuf hla_row;        // u32[hla_n] the other rows
  DevBuf hla_raw;        // u64 scratch: unsorted (key << 32 | row)

  // ---- sketches
  bool built = false;
  uint32_t R = 0, R_local = 0, rank = 0, world = 1;
  uint64_t hash_seed = 0, K = 0, a32 = 0;
  bool compressed = false;
  std::vector<uint32_t> slot_r;   // slot j -> sketch id r  (slots sorted by hash(r))
  std::vector<int32_t> r_slot;    // sketch id r -> slot j or -1
  std::vector<uint32_t> shr;      // hr32 of slot j (sorted ascending)
  std::vector<uint16_t> tab;      // bucket table, (1<<PACIM_TB)+1 entries
  std::vector<uint64_t> hr64;     // full hash(r) of slot j (R20 decorrelated rule)
  DevBuf d_shr, d_tab, d_hr64;
  int hash_rule = 0;              // 0: P:3-4 literal, 1: decorrelated (R20)
  int selector = 0;               // 0: incremental, 1: lazy (NEXT f2)
  DevBuf d_hot;        // u32[2*B]: per slot the hub's root and its component id
  uint32_t hub = 0;    // a maximum-degree vertex (most likely in the giant CC)

  // uncompressed store: slot windows: window w holds slots
  // [f_w, f_w + c_w) of every row at L + nr * f_w, row stride c_w, so
  // (row, j) lives at nr * f + row * c + (j - f).  One window [0, B) is the
  // plain vertex-major layout.  d_smap[j] = f << 16 | c of j's window.
  DevBuf L;
  DevBuf edge_work;  // k_edges' chunk counter (dynamic work distribution)
  // slot epochs of L (Ep above): the current build's, the epoch count and
  // bits, and the store they are valid for (a full reset otherwise)
  Ep ep;
  uint32_t ep_bits = 0, ep_cur = 0;
  bool ep_clean = false;
  const void *ep_store = nullptr;
  uint32_t ep_nr = 0, ep_B = 0;
  bool skip_init = false;  // pc_sketch_pass: the store needs no reset this build
  uint64_t ep_live_gen = ~0ull;  // live pairs per slot of the last dense build of graph_gen
  double ep_live_per_slot = 0;
  // hook list of epoch builds (k_edges -> k_compress_count<…, LIST>): capacity
  // from the non-root count of the last dense build of graph_gen (hk_gen)
  DevBuf sym[11];       // scratch of the upper-CSR symmetrization (graph.cu), kept across loads
  bool tcsr_ok = false;
  bool elist_ok = false;
  bool ucsr = false;      // the build streams the upper edges (UpperCsr), derive_edges
  bool ucsr_direct = false;  // ... without per-edge arrays (UpperCsr's CSR-direct form)
  // graphs loaded as an upper CSR (pacim_load_graph_upper[_async]): the upper
  // CSR stays in uoff / unbr, off holds the symmetric offsets (from the
  // degrees), and the symmetric neighbour lists nbr are built only when
  // something reads them (pc_ensure_sym: traversal selections, compressed
  // probes, Monte Carlo, lean builds, pacim_get_graph) — the dense store's
  // build and its Win-Tree selection read the upper edges only
  bool upper_src = false;
  bool sym_pending = false;  // keys / ckeys derived for the current graph (pc_ensure_edge_lists)  // tcsr derived for the current graph (pc_ensure_tcsr)
  DevBuf hk_list;
  uint64_t hk_hint = 0, hk_gen = ~0ull, hk_cap = 0;
  uint32_t hk_B = 0;
  std::vector<uint32_t> win_first;  // window starts, + B at the end
  DevBuf d_smap;
  std::vector<uint32_t> smap_of;   // the windows d_smap was filled for
  DevBuf pkeys;          // per-build edge partition by bucket: keys, ckeys, counts
  uint64_t ncomp = 0, nmember = 0, nnonsingle = 0;
  uint32_t big_t = 0;
  DevBuf csize;       // u32[ncomp] pristine CC sizes
  DevBuf csize_work;  // u32[ncomp] sizes zeroed on cover (MarkSeed)
  DevBuf coff;        // u64[ncomp] member-index offsets
  DevBuf cfill;       // u32[ncomp] scatter cursors
  DevBuf perm;        // u32[nmember] members grouped by component
  DevBuf gain0;       // i64[n]
  DevBuf gain;        // i64[n] working gains of a selection

  // compact uncompressed store (store_cs.cu): entries only for
  // the (row, slot) pairs whose vertex has a live edge in the slot's sketch
  bool cs = false;          // the current store is the compact one
  uint32_t cs_MW = 0;       // mask words per row (ceil(B / 32))
  uint64_t cs_total = 0;    // entries = non-singleton (vertex, sketch) pairs
  uint32_t cs_list_t = 0;   // CCs above it (or the hub's) are covered by the dense pass
  DevBuf cs_rec;            // uint2[nr][MW]: {entry prefix, live-slot mask word}
  DevBuf cs_soff;           // u32[nr + 1]: first entry of a row
  DevBuf cs_ecrow;          // u32[total / 32 + 1]: row of entry 32 c
  DevBuf cs_E;              // uint2[total]: {parent -> HIGH | size / root entry, next member}
  DevBuf cs_vid;            // u32[total]: vertex of an entry
  DevBuf cs_diag;           // u64 selection diagnostics
  DevBuf wt_buf;            // Win-Tree selector scratch (tree, wave lists; capacity reused)
  DevBuf cs_cnt;            // build scratch: row counts and their scan
  DevBuf cs_plist;          // build scratch: the mask pass's live (edge, slot) pairs
  double cs_live_rate = -1;      // its live pairs per (edge, slot)
  uint64_t cs_live_hint = 0;     // list slots of the last compact build of ...
  uint64_t cs_live_gen = ~0ull;  // ... graph_gen, with cs_live_B slots and key cs_live_K
  uint32_t cs_live_B = 0;
  uint64_t cs_live_K = 0;
  uint64_t cs_pref_gen = ~0ull;  // store decision of the last build of graph_gen ...
  uint32_t cs_pref_B = 0;        // ... with this many slots:
  bool cs_pref_dense = false;    // too dense for the compact store

  // compressed store (H6c)
  uint32_t rho = 0;
  DevBuf center_of;   // u32[n] center index or 0xFFFFFFFF
  DevBuf centers;     // u32[rho] center vertex ids in increasing order
  DevBuf clabel;      // u32[rho*B]  label of center i in slot j at i*B + j
  DevBuf csz;         // u32[rho*B]  pristine sizes
  DevBuf csz_work;    // u32[rho*B]  sizes zeroed by MarkSeed
  DevBuf Ltmp;        // u32[rows*Bb] parent arrays of one build batch
  uint32_t Bb = 0;    // slots per compressed build batch
  DevBuf is_seed;     // u8[n] seeds of the current selection (Get-center seed test)
  DevBuf cwork;       // per-step compressed cover scratch
  DevBuf cprobe;      // compressed cover: per-slot status / label / delta + sums
  DevBuf cseed;       // compressed cover: the seed's live neighbours per slot
  DevBuf hotsum;      // i64[n]: sizes of the hub's CCs of > 65536 vertices containing v
  DevBuf d_hot_size;  // u32[B]: the hub's CC size per slot
  std::vector<uint32_t> hot_size;
  uint32_t cbig_t = 65536;  // compressed: covered CCs above it go to the rebuild / hotsum
  bool hot_any = false;     // uncompressed: hotsum holds the giant hot CCs' sums (one window)
  uint32_t hot_big_t = 0;   // ... for this select dense threshold

  // scratch
  DevBuf counters;    // u64[64]
  DevBuf scratch;     // generic temporary
  DevBuf scratch2;
  unsigned long long *h_counters = nullptr;  // pinned host mirror (64)

  // selection outputs (device)
  DevBuf sel_seeds, sel_gain, sel_partial, sel_list, sel_flag, argmax_part;
  DevBuf bfs;                   // traversal state of the cover step (select.cu)
  uint32_t bfs_nr = 0, bfs_bw = 0;  // its layout (rows, mask words per row)
  bool bfs_ring_reset = false;  // the work-queue rings must be (re)initialised
  uint32_t sel_par = 0;         // parity of the next selection step (touched lists)
  uint32_t sel_k_cap = 128;     // covered-CC list capacity, in steps
  bool sel_list_valid = false;  // sel_list holds the covered list of this store

  DeltaList dlist;              // set only during pacim_cover_local_sparse

  pacim_stats stats{};
  uint32_t launches = 0;

  // asynchronous graph loads: two staging slots, filled in order on copy_stream
  StagedGraph stage[2];
  uint32_t stage_fill = 0, stage_commit = 0;  // next slot to fill / to commit
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t released = nullptr;  // main stream: the last commit's old buffers are free
};

// allocation with capacity reuse (cudaMalloc, or the caller's workspace)
void pc_ensure(pacim_ctx *ctx, DevBuf &b, size_t bytes);
void pc_free(pacim_ctx *ctx, DevBuf &b);
// free device bytes for sizing decisions: cudaMemGetInfo's free memory, or
// the largest hole of the workspace
size_t pc_mem_free(pacim_ctx *ctx);
void pc_mem_info(pacim_ctx *ctx, size_t *fr, size_t *tot);

// temporary device buffer released at scope exit (also on exceptions)
struct TmpBuf : DevBuf {
  pacim_ctx *c;
  explicit TmpBuf(pacim_ctx *c_) : c(c_) {}
  ~TmpBuf() { pc_free(c, *this); }
  TmpBuf(const TmpBuf &) = delete;
  TmpBuf &operator=(const TmpBuf &) = delete;
};

// ---------------------------------------------------------- host wrappers
// graph.cu
void pc_exclusive_scan_u64(pacim_ctx *ctx, const uint64_t *in, uint64_t *out,
                           size_t N);
void pc_graph_finish_load(pacim_ctx *ctx, int validate);
// upper CSR (each undirected edge once, neighbours > u, sorted; device arrays)
// -> the symmetric CSR in ctx->off / ctx->nbr (graph.cu)
void pc_validate_upper(pacim_ctx *ctx, const uint64_t *d_uoff, const uint32_t *d_unbr, uint32_t n);
void pc_symmetrize_upper(pacim_ctx *ctx, const uint64_t *d_uoff, const uint32_t *d_unbr,
                         uint32_t n, uint64_t m);
void pc_sym_free(pacim_ctx *ctx);
// the per-CSR-entry thresholds of per-edge models, derived on first use (graph.cu)
void pc_ensure_tcsr(pacim_ctx *ctx);
// after every graph load: graph_gen++, hint_gen++ if the shape changed (api.cu)
void pc_graph_loaded(pacim_ctx *ctx);
void pc_generate(pacim_ctx *ctx, int kind, const uint64_t *params, int nparams,
                 uint64_t gen_seed);
// build.cu
void pc_build(pacim_ctx *ctx);
void pc_cs_edges(pacim_ctx *ctx, uint32_t *P, const uint2 *rec, uint32_t MW,
                 unsigned long long *ctr);
void pc_cs_mask_edges(pacim_ctx *ctx, uint32_t *rec_words, uint32_t MW, unsigned long long *ctr,
                      unsigned long long *plist, unsigned long long *pcnt, unsigned long long cap);
void pc_ep_edges(pacim_ctx *ctx, uint64_t e0, uint64_t e1, const uint32_t *d_shr_all,
                 const uint16_t *d_tab_all, uint32_t R, unsigned long long *plist,
                 unsigned long long *pcnt, unsigned long long cap, unsigned long long *ctr);
// dist.cu: the edge-partitioned live pairs of a sharded compact build —
// this rank's edge range tested against all R sketches, routed to the
// sketches' owners (NCCL send/recv); the rank's pairs (local slots) land in
// ctx->cs_plist and their bits in the rec masks.  Returns their count, or
// ~0 if the build cannot take this path.
unsigned long long pc_cs_ep_pairs(pacim_ctx *ctx, uint32_t MW, unsigned long long *ctr);
void pc_cs_list_unite(pacim_ctx *ctx, uint32_t *E, const uint2 *rec, uint32_t MW,
                      const unsigned long long *plist, unsigned long long cnt,
                      unsigned long long *ctr, const unsigned long long *mask_live);
// dist.cu: NCCL sharding
void pc_nccl_unique_id(void *out);
void pc_init_comm(pacim_ctx *ctx, int rank, int world, const void *id);
void pc_free_comm(pacim_ctx *ctx);
bool pc_dist_active(const pacim_ctx *ctx);
void pc_dist_build_finish(pacim_ctx *ctx);
void pc_dist_restore(pacim_ctx *ctx);
void pc_dist_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num);
// store_cs.cu: the compact store (build, selection, inspection)
bool pc_cs_build(pacim_ctx *ctx);  // false: not eligible (dense store instead)
void pc_cs_free(pacim_ctx *ctx);
void pc_cs_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                  int64_t *sigma_num);
void pc_cs_select_reset(pacim_ctx *ctx);
void pc_cs_cover_local(pacim_ctx *ctx, uint32_t s, int64_t *d_delta, int64_t *local_gain);
void pc_cs_get_labels(pacim_ctx *ctx, uint32_t slot, uint32_t *host_out);
void pc_cs_lazy_eval(pacim_ctx *ctx, const uint32_t *cand, uint32_t b0, uint32_t b1,
                     long long *delta);
void pc_cs_lazy_mark(pacim_ctx *ctx, uint32_t s);
void pc_cs_select_wintree(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                          int64_t *sigma_num);
void pc_slot_table(pacim_ctx *ctx);
// Live hub adjacency (HLA) being recorded: raw (key << 32 | other row) with
// key = hub index * B + slot, appended in any order (grouped by key after the
// build: pc_hla_finish).  Entries past cap are dropped (the build then flags
// the HLA invalid and the selection hashes hubs' edges).
struct Hla {
  // hub row -> hub index: open addressing over (row << 32 | index), a few MB
  // and L2-resident (the per-row index hidx is not: one random DRAM read per entry)
  const unsigned long long *tab;
  uint32_t mask;
  unsigned long long *raw;   // [cap]
  unsigned long long *n;     // entries appended
  unsigned long long cap;
  uint32_t B;
  __device__ __forceinline__ uint32_t hub_of(uint32_t row) const {
    for (uint32_t h = (row * 2654435761u) & mask;; h = (h + 1) & mask) {
      const unsigned long long e = __ldg(tab + h);
      if ((uint32_t)(e >> 32) == row) return (uint32_t)e;
    }
  }
  // all 32 lanes call this together; lane i stages nu entries for hub row u
  // and nv for hub row v (live edge (u, v) in slot j) in the warp's shared
  // buffer buf (HLA_WBUF entries, bn of them used); a nearly full buffer is
  // flushed with one counter update (one global atomic per ~HLA_WBUF - 64
  // entries instead of one per round: the counter is a single address)
  static constexpr uint32_t HLA_WBUF = 128;
  __device__ __forceinline__ void stage(uint32_t u, uint32_t v, uint32_t j, uint32_t nu,
                                        uint32_t nv, unsigned long long *buf, uint32_t &bn) const {
    const uint32_t mine = nu + nv;
    if (!__ballot_sync(0xffffffffu, mine)) return;
    const uint32_t lane = threadIdx.x & 31;
    uint32_t pre = mine;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, pre, d);
      if (lane >= (uint32_t)d) pre += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
    uint32_t pos = bn + pre - mine;
    if (nu) buf[pos++] = ((unsigned long long)hub_of(u) * B + j) << 32 | v;
    if (nv) buf[pos] = ((unsigned long long)hub_of(v) * B + j) << 32 | u;
    bn += tot;
    if (bn > HLA_WBUF - 64) flush(buf, bn);
  }
  __device__ __forceinline__ void flush(unsigned long long *buf, uint32_t &bn) const {
    __syncwarp();
    if (!bn) return;
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(n, (unsigned long long)bn);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (uint32_t i = lane; i < bn; i += 32)
      if (base + i < cap) raw[base + i] = buf[i];
    __syncwarp();
    bn = 0;
  }
};

// edges of one sketch pass: the whole upper edge list (default) or one
// bucket of the per-build partition
struct EdgeSet {
  const uint64_t *keys = nullptr, *ckeys = nullptr;
  uint64_t m = 0;
};
// The upper edges as a compact stream (k_edges LEAN = 2, the dense store's
// one-window builds): upper edge e = (u, unbr[e]) with u = ucrow[c] + (ud16[e]
// & 255) and row(u) = ucrowr[c] + (ud16[e] >> 8), c = e >> 5 (ucrow[c] = the
// vertex of upper edge 32 c, ucrowr[c] its store row; a byte of 255: that
// far or more, the vertex then by the offsets walk from ucrow[c], the row by
// the rank map
// rk[u >> 5] = {row of the word's first non-isolated vertex, bitmap of its
// non-isolated vertices}: rk.x + popc(rk.y & below(u))); the neighbour's
// store row uvrow[e] (or, PACIM_UCSR=2, the rank map).  10 B per edge (+ 4 B
// tm1) instead of keys + ckeys' 16, and no load depends on another: a
// dependent rank-map gather in k_edges' front end cost 22.8 -> 31.5 ms at c4.
// CSR-direct form (k_edges LEAN = 4, `ucsr_direct`: graphs for which even
// the stream does not fit — c5): no per-edge array at all; the row by the
// chunk table and pc_row_of, the neighbour at the row's upper part of the
// symmetric CSR (off, nbr; or unbr[e] for an upper-loaded graph), both store
// rows by the rank map, the threshold t32 or tm1[e]
struct UpperCsr {
  uint32_t nv = 0;  // vertices
  const uint64_t *off = nullptr;  // LEAN = 4: the symmetric offsets
  const uint32_t *nbr = nullptr;  // LEAN = 4: the symmetric lists (null: unbr)
  const uint64_t *uoff = nullptr;
  const uint32_t *unbr = nullptr, *ucrow = nullptr, *uvrow = nullptr, *ucrowr = nullptr;
  const uint16_t *ud16 = nullptr;
  const uint2 *rk = nullptr;
};
// The row u in [lo, hi] of entry e of a CSR-like offsets array: off[lo] <=
// e, hi >= the row.  A few linear steps, then a binary search for the
// largest u with off[u] <= e (a linear walk over a run of empty rows — the
// top of an R-MAT id range has thousands of vertices without upper edges —
// kept one SM busy 24M cycles after the rest finished: c4 k_edges 22.8 ->
// 36 ms)
__device__ __forceinline__ uint32_t pc_row_of(const uint64_t *off, uint32_t lo, uint32_t hi,
                                              uint64_t e) {
#pragma unroll 1
  for (int i = 0; i < 4; i++) {
    if (e < off[lo + 1]) return lo;
    lo++;
  }
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo + 1) >> 1);
    if (off[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
// the symmetric neighbour lists of an upper-loaded graph (no-op otherwise)
void pc_ensure_sym(pacim_ctx *ctx);
// an upper CSR in uoff / unbr (n, m set): the symmetric offsets off from the
// degrees (lower degrees by a histogram of the targets), ucrow; nbr pending
void pc_upper_degrees(pacim_ctx *ctx);
// keys / ckeys of the current graph (derived on first use: the compact
// store, the edge-partitioned and bucketed builds, HLA recording)
void pc_ensure_edge_lists(pacim_ctx *ctx);
// HLA recording around the sketch passes of a build: begin sizes the raw
// buffer from the expected live hub entries E (false: not recorded — no hubs,
// a lean graph, E > max_per_edge * m, or it does not fit in a slice of the
// free memory); finish groups the entries by (hub, slot) and sets
// ctx->hla_ok (false on overflow).
bool pc_hla_begin(pacim_ctx *ctx, Hla *hla, double max_per_edge);
void pc_hla_finish(pacim_ctx *ctx, Hla *hla);
void pc_sketch_pass(pacim_ctx *ctx, uint32_t *Lb, uint32_t j0, uint32_t Bb,
                    unsigned long long *ctr, cudaEvent_t *ev, const Hla *hla = nullptr,
                    const EdgeSet *es = nullptr);
// compressed.cu (H6c, H11)
void pc_build_compressed(pacim_ctx *ctx);
void pc_select_compressed(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                          int64_t *sigma_num);
// dsel (optional): the argmax left on the device by pc_argmax_async — the seed
// is read from it by the kernels and returned in *s_out / *g_out after the
// step's one read-back (s is then ignored)
void pc_cover_compressed(pacim_ctx *ctx, uint32_t s, int64_t *target, int64_t *local_gain,
                         const void *dsel = nullptr, uint32_t *s_out = nullptr,
                         int64_t *g_out = nullptr);
void pc_select_reset_compressed(pacim_ctx *ctx);
// select.cu: device bytes of the selection's traversal state for nr rows, B slots
size_t pc_select_state_bytes(uint32_t nr, uint32_t B);
void pc_get_center_sketch(pacim_ctx *ctx, uint32_t slot, uint32_t *label, uint32_t *size);
// select.cu
void pc_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
               int64_t *sigma_num);
void pc_select_reset(pacim_ctx *ctx);
void pc_select_wintree_dense(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                             int64_t *sigma_num);
void pc_select_lazy(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                    int64_t *sigma_num);
void pc_cover_local(pacim_ctx *ctx, uint32_t s, int64_t *d_delta,
                    int64_t *local_gain);
const void *pc_argmax_async(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n);
void pc_argmax(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n, uint32_t *s,
               int64_t *g);
// mc.cu (NEXT f3)
void pc_simulate_ic(pacim_ctx *ctx, const uint32_t *seeds_host, uint32_t ns, uint32_t nsims,
                    uint64_t mc_seed, uint64_t *total_out);
void pc_apply_deltas(pacim_ctx *ctx, int64_t *d_gain, const uint32_t *v, const int64_t *d,
                     uint64_t count, uint32_t s);
void pc_apply_dense(pacim_ctx *ctx, int64_t *d_gain, int64_t *d_delta, uint32_t n, uint32_t s);
void pc_clear_deltas(pacim_ctx *ctx, int64_t *d_delta, const uint32_t *v, uint64_t count);
void pc_get_labels(pacim_ctx *ctx, uint32_t slot, uint32_t *host_out);
void pc_free_lalt(pacim_ctx *ctx);
void pc_reset_next(pacim_ctx *ctx);  // enqueue the due reset of the second store  // waits for a pending reset, frees the second store
// the cover traversal alone (no store): for every slot j with delta[j] > 0
// (HOST array of R_local), the members of C_j(s) lose delta[j] in target
void pc_traverse_slots(pacim_ctx *ctx, uint32_t s, int64_t *target, const uint32_t *delta);

// grid sizing: multiples of the SM count (148 on B200)
inline unsigned pc_grid(const pacim_ctx *ctx, size_t work, unsigned block,
                        unsigned per_sm = 8) {
  size_t need = (work + block - 1) / block;
  size_t cap = (size_t)ctx->sm_count * per_sm;
  if (need < 1) need = 1;
  return (unsigned)(need < cap ? need : cap);
}
// Grid of a grid-stride kernel: at most one full wave of resident blocks
// (the occupancy the kernel's registers and shared memory allow), so no block
// starts after the first ones finish — a partial second wave runs its share
// of the loop at a fraction of the occupancy (ncu: k_compress_count at 1.33
// waves spent up to half its time in the tail)
template <typename K>
inline unsigned pc_grid_occ(const pacim_ctx *ctx, K kern, size_t work, unsigned block,
                            size_t smem = 0) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, (int)block, smem) != cudaSuccess ||
      nb < 1)
    nb = 1;
  return pc_grid(ctx, work, block, (unsigned)nb);
}
