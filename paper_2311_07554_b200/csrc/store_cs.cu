// store_cs.cu — the COMPACT uncompressed store (H3-H7, H6u with its member
// lists) and the greedy loop over it (H8-H12).  DESIGN.md §5 / §6.
//
// Why: in the paper's workloads a vertex is a singleton in most sketches (c4:
// 9.8 % of the (row, sketch) pairs are in a CC of >= 2 vertices, c2: 23 %).
// The dense vertex-major store (build.cu) writes, compresses and re-reads
// every pair; the compact store keeps an entry only for the pairs (v, r) where
// v has a live edge in sketch r (exactly the non-singleton pairs), laid out
// row-major, so every streaming pass moves ~1/10 of the bytes at c4, and the
// members of every CC are linked so that covering a CC (MarkSeed + the
// member updates) costs O(|C|) with no traversal of the sampled graph.
//
// Layout (per build, B local sketch slots <= 256, MW = ceil(B/32) words):
//   rec[row][w]  {first entry of the row + set bits of the row's words < w,
//                 live-slot mask word w}: entry of (row, j) = pc_cs_pos (8 B)
//   soff[row]    first entry of a row; ecrow[c] row of entry 32 c
//   E[e] = {P, next}
//     P          union-find parent (an entry index: the entries of one slot are
//                in vertex order, so the minimum entry of a CC is its minimum
//                vertex, R8); after compression HIGH | |C| at the root entry,
//                the root entry elsewhere; bit 30 = covered during a selection
//     next       the CC's member list: root -> ... -> NONE (members inserted
//                right after the root by the compression pass)
//   vid[e]       the entry's vertex
// The hub's CCs (hot) and CCs above list_t have no list: covering them is one
// vector pass over the build's per-vertex hot sums (when a step covers
// exactly the hub's CCs) or one pass over the entries.
//
// Build: the mask pass (k_edges<…, 2> over the upper edges: every live (edge,
// sketch) sets the slot bit in both endpoints' row masks) -> counts, scan ->
// k_cs_rec -> E = {HIGH|1, NONE} ->
// k_edges<CS> (build.cu: the unions, on entries) -> k_cs_compress (full
// compression, CC sizes, member lists) -> k_cs_gain (gain0 = sum_r |C_r(v)|,
// hot sums, vid).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pacim_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t ROOT1 = PACIM_HIGH | 1u;
constexpr uint32_t COV = 0x40000000u;
constexpr uint32_t SIZE = 0x3FFFFFFFu;
constexpr uint32_t MAXW = 8;          // B <= 256
constexpr unsigned FULL = 0xffffffffu;
constexpr int CS_THREADS = 256;
constexpr int SEL_THREADS = 512;
constexpr uint32_t MAX_CHUNKS = 4096;
constexpr uint32_t LIST_T = 4096;     // longest member list walked in a cover step
constexpr uint32_t WBUF = 128;        // member entries a warp buffers per walk round

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t entry_row(const uint32_t *soff, const uint32_t *ecrow,
                                              uint64_t e) {
  uint32_t r = ecrow[e >> 5];
  while (e >= soff[r + 1]) r++;
  return r;
}

// union-find on the P words of E (stride 2)
__device__ __forceinline__ uint32_t find_halve(uint32_t *E, uint32_t x) {
  for (;;) {
    const uint32_t p = __ldcg(E + 2 * (size_t)x);
    if (p & PACIM_HIGH) return x;
    const uint32_t gp = __ldcg(E + 2 * (size_t)p);
    if (gp & PACIM_HIGH) return p;
    atomicMin(E + 2 * (size_t)x, gp);
    x = gp;
  }
}

__device__ __forceinline__ uint32_t find_ro(const uint32_t *E, uint32_t x) {
  for (;;) {
    const uint32_t p = __ldcg(E + 2 * (size_t)x);
    if (p & PACIM_HIGH) return x;
    x = p;
  }
}

__device__ __forceinline__ void add_count(unsigned long long *ctr, unsigned long long c) {
  for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(FULL, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(ctr, c);
}

// sum over the lanes of `peers` (same row) of a value < 2^31 per lane, in 64 bits
__device__ __forceinline__ unsigned long long peer_sum(unsigned peers, uint32_t x) {
  const uint32_t lo = __reduce_add_sync(peers, x & 0xFFFFu);
  const uint32_t hi = __reduce_add_sync(peers, x >> 16);
  return (unsigned long long)lo + ((unsigned long long)hi << 16);
}

// sorted copy of up to 256 root entries in shared memory (rank sort: each
// thread counts the smaller keys); NONE entries sort last.  Returns the count.
__device__ uint32_t load_sorted(const uint32_t *src, uint32_t B, uint32_t *dst) {
  __shared__ uint32_t tmp[256];
  __shared__ uint32_t nval;
  if (threadIdx.x == 0) nval = 0;
  for (uint32_t j = threadIdx.x; j < 256; j += blockDim.x) tmp[j] = j < B ? src[j] : NONE;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < 256; j += blockDim.x) {
    const uint32_t x = tmp[j];
    uint32_t r = 0;
    for (uint32_t i = 0; i < 256; i++) {
      const uint32_t y = tmp[i];
      r += (y < x) || (y == x && i < j);
    }
    dst[r] = x;
    if (x != NONE) atomicAdd(&nval, 1u);
  }
  __syncthreads();
  return nval;
}

// index of x in the sorted list (n entries), or -1
__device__ __forceinline__ int find_sorted(const uint32_t *a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && a[lo] == x) ? (int)lo : -1;
}

// entries per row (set bits), u64 for the scan; cnt[nr] = 0
__global__ void k_cs_count(const uint2 *rec, uint32_t nr, uint32_t MW, uint64_t *cnt) {
  for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r <= nr;
       r += (size_t)gridDim.x * blockDim.x) {
    uint64_t c = 0;
    if (r < nr)
      for (uint32_t q = 0; q < MW; q++) c += __popc(rec[r * MW + q].y);
    cnt[r] = c;
  }
}

// thread per row: word prefixes (rec[.].x), soff, and the chunk table (row of
// entry 32 c for every chunk starting in the row)
__global__ void k_cs_rec(uint2 *rec, uint32_t nr, uint32_t MW, const uint64_t *pos,
                         uint32_t *soff, uint32_t *ecrow) {
  for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr;
       r += (size_t)gridDim.x * blockDim.x) {
    const uint32_t base = (uint32_t)pos[r];
    uint32_t at = base;
    for (uint32_t q = 0; q < MW; q++) {
      uint2 x = rec[r * MW + q];
      x.x = at;
      at += __popc(x.y);
      rec[r * MW + q] = x;
    }
    soff[r] = base;
    if (r + 1 == nr) soff[nr] = at;
    for (uint32_t c = (base + 31) >> 5; (c << 5) < at; c++) ecrow[c] = (uint32_t)r;
  }
}

__global__ void k_cs_fill(uint2 *E, uint64_t N) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    E[i] = make_uint2(ROOT1, NONE);
}

// the hub row's root entry per slot (the hot CCs), NONE if the hub is a
// singleton there
__global__ void k_cs_hot(const uint2 *rec, uint32_t MW, const uint32_t *E, uint32_t hub_row,
                         uint32_t nr, uint32_t B, uint32_t *hot) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x) {
    uint32_t h = NONE;
    if (hub_row < nr && ((rec[(size_t)hub_row * MW + (j >> 5)].y >> (j & 31)) & 1u))
      h = find_ro(E, pc_cs_pos(rec, MW, hub_row, j));
    hot[j] = h;
  }
}

// full compression (H4), CC sizes into the root entries (H5) and the member
// lists (H6u): a non-root entry is linked in right after its root.  Members
// of the hub's CCs (hot roots; c2: ~500K per sketch) get no list and count in
// shared memory, one global increment per hot root per block at the end.
// ctr[1] += non-root entries.
__global__ void __launch_bounds__(CS_THREADS) k_cs_compress(uint32_t *E, uint64_t total,
                                                            const uint32_t *hot, uint32_t B,
                                                            unsigned long long *ctr) {
  __shared__ uint32_t hs[256], hcnt[256];
  const uint32_t nh = load_sorted(hot, B, hs);
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hcnt[i] = 0;
  __syncthreads();
  unsigned long long nnr = 0;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const uint32_t s = __ldcg(E + 2 * e);
    if (s & PACIM_HIGH) continue;
    nnr++;
    int h = nh ? find_sorted(hs, nh, s) : -1;
    uint32_t root = s;
    if (h < 0) {
      root = find_halve(E, s);
      if (root != s) {
        atomicMin(E + 2 * e, root);
        if (nh) h = find_sorted(hs, nh, root);
      }
    }
    if (h >= 0) {
      atomicAdd(hcnt + h, 1u);
    } else {
      atomicAdd(E + 2 * (size_t)root, 1u);                               // |C|
      E[2 * e + 1] = atomicExch(E + 2 * (size_t)root + 1, (uint32_t)e);  // link after the root
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nh; i += blockDim.x)
    if (hcnt[i]) atomicAdd(E + 2 * (size_t)hs[i], hcnt[i]);
  add_count(ctr + 1, nnr);
}

__global__ void k_cs_hot_sizes(const uint32_t *E, const uint32_t *hot, uint32_t B,
                               uint32_t *hot_size) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x)
    hot_size[j] = hot[j] != NONE ? (E[2 * (size_t)hot[j]] & PACIM_LOW) : 0u;
}

// gain0 before the entries: B - (entries of the row) singletons (size 1 each);
// isolated vertices B
__global__ void k_cs_gain_init(const uint32_t *cid, const uint32_t *soff, uint32_t n, uint32_t B,
                               int64_t *gain0, int64_t *hotsum) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    const uint32_t r = cid ? cid[v] : (uint32_t)v;
    gain0[v] = r == NONE ? (int64_t)B : (int64_t)B - (int64_t)(soff[r + 1] - soff[r]);
    if (hotsum) hotsum[v] = 0;
  }
}

// lane per entry: gain0[v] += |C_j(v)| (H7), hotsum[v] += |C| when the
// entry's CC is one of the hub's (HOT), vid[e] = v.  ctr[0] += roots.
template <bool HOT>
__global__ void __launch_bounds__(CS_THREADS) k_cs_gain(
    const uint32_t *__restrict__ E, uint64_t total, const uint32_t *__restrict__ soff,
    const uint32_t *__restrict__ ecrow, const uint32_t *__restrict__ rmap, uint32_t B,
    const uint32_t *hot, uint32_t *vid, int64_t *gain0, int64_t *hotsum,
    unsigned long long *ctr) {
  __shared__ uint32_t hs[256];
  uint32_t nh = 0;
  if (HOT) nh = load_sorted(hot, B, hs);
  const int lane = threadIdx.x & 31;
  unsigned long long nroot = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(size_t)31; base < total;
       base += stride) {
    const size_t e = base + lane;
    uint32_t row = NONE, size = 0, hsz = 0, v = 0;
    if (e < total) {
      const uint32_t s = E[2 * e];
      row = entry_row(soff, ecrow, e);
      const uint32_t root = (s & PACIM_HIGH) ? (uint32_t)e : s;
      const uint32_t rv = (s & PACIM_HIGH) ? s : __ldg(E + 2 * (size_t)s);
      v = rmap ? rmap[row] : row;
      vid[e] = v;
      size = rv & PACIM_LOW;
      nroot += (s & PACIM_HIGH) != 0;
      if (HOT && find_sorted(hs, nh, root) >= 0) hsz = size;
    }
    const unsigned peers = __match_any_sync(FULL, row);
    const unsigned long long g = peer_sum(peers, size);
    const unsigned long long h = HOT ? peer_sum(peers, hsz) : 0ull;
    if (lane == __ffs(peers) - 1 && row != NONE) {
      atomicAdd(reinterpret_cast<unsigned long long *>(gain0 + v), g);
      if (HOT && h) atomicAdd(reinterpret_cast<unsigned long long *>(hotsum + v), h);
    }
  }
  add_count(ctr, nroot);
}

// --------------------------------------------------------------- select
struct Best {
  long long g;
  uint32_t v;
};

__device__ __forceinline__ bool better(long long g1, uint32_t v1, long long g2, uint32_t v2) {
  return g1 > g2 || (g1 == g2 && v1 < v2);
}

__device__ __forceinline__ Best warp_best(Best b) {
  for (int d = 16; d; d >>= 1) {
    const long long g = __shfl_xor_sync(FULL, b.g, d);
    const uint32_t v = __shfl_xor_sync(FULL, b.v, d);
    if (better(g, v, b.g, b.v)) {
      b.g = g;
      b.v = v;
    }
  }
  return b;
}

__device__ Best block_best(Best b, Best *sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  b = warp_best(b);
  __syncthreads();
  if (lane == 0) sh[wid] = b;
  __syncthreads();
  if (wid == 0) {
    Best x = lane < (int)(blockDim.x >> 5) ? sh[lane] : Best{LLONG_MIN, NONE};
    x = warp_best(x);
    if (lane == 0) sh[32] = x;
  }
  __syncthreads();
  return sh[32];
}

// diagnostics (u64): steps, dense steps, hot-sum steps, member updates
enum { CD_STEPS = 0, CD_DENSE, CD_HOT, CD_UPD, CD_CELF, CD_WORDS = 8 };

struct CSel {
  const uint2 *rec;
  uint32_t MW;
  uint32_t *E;             // {P, next} words
  const uint32_t *vid, *soff, *rmap, *cid;
  uint32_t nr, B, nv;
  uint64_t total;
  uint32_t list_t;
  long long *target;       // gains (single rank) or the delta vector (multi-rank)
  uint32_t *cov_root, *cov_delta;  // [B] list-less CCs covered this step
  int *dense;              // [2] by step parity
  unsigned long long *cov_list, *cov_cnt;
  unsigned long long cov_cap;
  const int64_t *hotsum;
  const uint32_t *hot_root;  // [B] the hub's root entry per slot (NONE: singleton)
  Best *cmax;
  uint32_t *cdirty, *dlist, *dcnt;
  uint32_t csh, nchunks, par;
  int track;
  DeltaList dlst;
  unsigned long long *diag;
  long long *celf;         // CELF's stale scores (PACIM_CELF_COUNT) or null
};

struct CSelOut {
  uint32_t k;
  uint32_t given;          // NONE: argmax; else the seed of one multi-rank step
  uint32_t *seeds;
  long long *gain_num;     // k, zeroed
  long long *arg_gain;     // k
};

__device__ __forceinline__ void mark_dirty(const CSel &S, uint32_t c) {
  if (atomicExch(S.cdirty + c, 1u) == 0u)
    S.dlist[(size_t)S.par * S.nchunks + atomicAdd(S.dcnt + S.par, 1u)] = c;
}

__device__ __forceinline__ void sub_gain(const CSel &S, uint32_t u, long long d) {
  atomicAdd(reinterpret_cast<unsigned long long *>(&S.target[u]), (unsigned long long)(-d));
  S.dlst.add(u, -d);
  if (S.track) {
    const uint32_t c = u >> S.csh;
    if (__ldcg(&S.cmax[c].v) == u) mark_dirty(S, c);  // only the chunk's argmax matters
  }
}

// MarkSeed in slot j for the seed row srow (one thread): returns
// delta_j; *mroot: a newly covered CC whose member list is walked now
__device__ __forceinline__ uint32_t cs_cover(const CSel &S, uint32_t srow, uint32_t j,
                                             uint32_t *mroot) {
  *mroot = NONE;
  S.cov_root[j] = NONE;
  if (srow == NONE || !((S.rec[(size_t)srow * S.MW + (j >> 5)].y >> (j & 31)) & 1u))
    return 1;  // {s}: a singleton, uncovered while s is not a seed
  const uint32_t e = pc_cs_pos(S.rec, S.MW, srow, j);
  const uint32_t x0 = __ldcg(S.E + 2 * (size_t)e);
  const uint32_t root = (x0 & PACIM_HIGH) ? e : x0;
  const uint32_t x = atomicOr(S.E + 2 * (size_t)root, COV);
  if (x & COV) return 0;  // covered by an earlier seed
  const uint32_t delta = x & SIZE;
  const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
  if (at < S.cov_cap) S.cov_list[at] = root;
  if (delta > S.list_t || root == S.hot_root[j]) {  // no member list: the dense pass
    S.cov_root[j] = root;
    S.cov_delta[j] = delta;
    S.dense[S.par] = 1;
  } else {
    *mroot = root;
  }
  return delta;
}

__device__ void refresh_chunks(const CSel &S, uint32_t par, bool all, Best *sh) {
  const uint32_t nd = all ? S.nchunks : __ldcg(S.dcnt + par);
  for (uint32_t t = blockIdx.x; t < nd; t += gridDim.x) {
    const uint32_t c = all ? t : __ldcg(S.dlist + (size_t)par * S.nchunks + t);
    const size_t v0 = (size_t)c << S.csh, v1 = min((size_t)S.nv, v0 + ((size_t)1 << S.csh));
    Best b{LLONG_MIN, NONE};
    for (size_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
      const long long g = __ldcg(S.target + v);
      if (better(g, (uint32_t)v, b.g, b.v)) {
        b.g = g;
        b.v = (uint32_t)v;
      }
    }
    b = block_best(b, sh);
    if (threadIdx.x == 0) {
      S.cmax[c] = b;
      S.cdirty[c] = 0;
    }
  }
}

// the list-less CCs covered this step are exactly the hub's CCs (all of
// them, now) -> the build's hot sums are the member updates (one vector
// pass); block-collective, uniform result
__device__ bool dense_hot(const CSel &S, uint32_t s, size_t tid, size_t nth) {
  int ok = S.hotsum != nullptr;
  for (uint32_t j = threadIdx.x; j < S.B && ok; j += blockDim.x)
    if (__ldcg(S.cov_root + j) != S.hot_root[j]) ok = 0;
  if (!__syncthreads_and(ok)) return false;
  for (size_t v = tid; v < S.nv; v += nth) {
    const long long h = S.hotsum[v];
    if (h && v != s) sub_gain(S, (uint32_t)v, h);
  }
  return true;
}

// dense pass: thread per entry; an entry whose root is one of this step's
// covered list-less CCs (croot: sorted, nc of them, sizes in cdel) loses |C|
__device__ void dense_pass(const CSel &S, uint32_t s, const uint32_t *croot, const uint32_t *cdel,
                           uint32_t nc, size_t tid, size_t nth) {
  for (size_t e = tid; e < S.total; e += nth) {
    const uint32_t x = __ldcg(S.E + 2 * e);
    const uint32_t root = (x & PACIM_HIGH) ? (uint32_t)e : x;
    const int h = find_sorted(croot, nc, root);
    if (h < 0) continue;
    const uint32_t v = S.vid[e];
    if (v != s) sub_gain(S, v, cdel[h]);
  }
}

// Step (parity par): A argmax -> B MarkSeed + member-list walks -> (dense) ->
// E refresh of the chunk maxima; grid barriers after B, the dense pass and E.
__global__ void __launch_bounds__(SEL_THREADS, 1) k_cs_select(CSel S0, CSelOut O, uint32_t par0) {
  cg::grid_group grid = cg::this_grid();
  CSel S = S0;
  __shared__ Best sh[33];
  __shared__ uint32_t croot[256], cdel[256], csort[256], dsort[256];
  __shared__ uint32_t wbuf[SEL_THREADS / 32][WBUF];
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  const size_t gwarp = tid >> 5, nwarps = nth >> 5;
  const int lane = threadIdx.x & 31;
  if (S.track) refresh_chunks(S, 0, true, sh);
  if (tid == 0) {
    S.dcnt[par0 & 1] = 0;
    S.dense[par0 & 1] = 0;
  }
  grid.sync();
  for (uint32_t step = 0; step < O.k; step++) {
    S.par = (par0 + step) & 1;
    const uint32_t nxt = S.par ^ 1;
    // ---- A: NextSeed (gain desc, id asc; R5, R6)
    uint32_t s;
    long long sg = 0;
    if (O.given == NONE) {
      Best c{LLONG_MIN, NONE};
      for (uint32_t i = threadIdx.x; i < S.nchunks; i += blockDim.x) {
        Best x;
        x.g = __ldcg(&S.cmax[i].g);
        x.v = __ldcg(&S.cmax[i].v);
        if (better(x.g, x.v, c.g, c.v)) c = x;
      }
      c = block_best(c, sh);
      s = c.v;
      sg = c.g;
    } else {
      s = O.given;
    }
    const uint32_t srow = S.cid ? S.cid[s] : s;
    // ---- CELF's re-evaluations on the same gains (diagnostic):
    //      from step 2 on, every non-seed whose stale score ranks at or above
    //      the winner's fresh score (gain desc, id asc) is popped and
    //      re-evaluated before the winner surfaces fresh
    if (S.celf && O.given == NONE) {
      if (step > 0) {
        unsigned long long c = 0;
        for (size_t v = tid; v < S.nv; v += nth) {
          const long long kv = S.celf[v];
          if (v == s) {
            c++;
            S.celf[v] = sg;
            continue;
          }
          const long long gv = __ldcg(S.target + v);
          if (gv < 0) continue;  // a seed
          if (kv > sg || (kv == sg && v < s)) {
            c++;
            S.celf[v] = gv;
          }
        }
        for (int q = 16; q; q >>= 1) c += __shfl_xor_sync(FULL, c, q);
        if (lane == 0 && c) atomicAdd(S.diag + CD_CELF, c);
      }
      grid.sync();
    }
    if (tid == 0) {
      O.seeds[step] = s;
      O.arg_gain[step] = sg;
      if (O.given == NONE) {
        S.target[s] = -1;  // s leaves the candidate set (R6)
        mark_dirty(S, s >> S.csh);
      }
    }
    // ---- B: MarkSeed per slot (a warp per slot); the members of each newly
    //          covered CC lose |C|: lane 0 walks the CC's list (one dependent
    //          load per hop) into a shared buffer, the warp applies the updates
    {
      unsigned long long dsum = 0, upd = 0;
      uint32_t *buf = wbuf[threadIdx.x >> 5];
      for (size_t j = gwarp; j < S.B; j += nwarps) {
        uint32_t d = 0, mr = NONE;
        if (lane == 0) d = cs_cover(S, srow, (uint32_t)j, &mr);
        d = __shfl_sync(FULL, d, 0);
        mr = __shfl_sync(FULL, mr, 0);
        dsum += d;
        if (mr == NONE) continue;
        upd += d;
        uint32_t e = mr, left = d;
        while (left) {
          uint32_t cnt = 0;
          if (lane == 0) {
            for (; cnt < WBUF && left && e != NONE; cnt++, left--) {
              buf[cnt] = e;
              e = __ldcg(S.E + 2 * (size_t)e + 1);
            }
            if (e == NONE) left = 0;
          }
          cnt = __shfl_sync(FULL, cnt, 0);
          left = __shfl_sync(FULL, left, 0);
          __syncwarp();
          for (uint32_t t = lane; t < cnt; t += 32) {
            const uint32_t v = __ldg(S.vid + buf[t]);
            if (v != s) sub_gain(S, v, d);
          }
          __syncwarp();
        }
      }
      if (lane == 0) {
        if (dsum) atomicAdd(reinterpret_cast<unsigned long long *>(&O.gain_num[step]), dsum);
        if (upd) atomicAdd(S.diag + CD_UPD, upd);
      }
    }
    grid.sync();
    // ---- dense: list-less CCs covered this step
    if (__ldcg(S.dense + S.par)) {
      for (uint32_t j = threadIdx.x; j < 256; j += blockDim.x) {
        croot[j] = j < S.B ? __ldcg(S.cov_root + j) : NONE;
        cdel[j] = j < S.B ? __ldcg(S.cov_delta + j) : 0u;
      }
      __syncthreads();
      uint32_t nc = 0;
      for (uint32_t j = threadIdx.x; j < 256; j += blockDim.x) {
        const uint32_t x = croot[j], d = cdel[j];
        uint32_t r = 0;
        for (uint32_t i = 0; i < 256; i++) r += (croot[i] < x) || (croot[i] == x && i < j);
        csort[r] = x;
        dsort[r] = d;
      }
      for (uint32_t j = 0; j < 256; j++) nc += croot[j] != NONE;  // uniform
      __syncthreads();
      if (dense_hot(S, s, tid, nth)) {
        if (tid == 0) atomicAdd(S.diag + CD_HOT, 1ull);
      } else {
        dense_pass(S, s, csort, dsort, nc, tid, nth);
      }
      if (tid == 0) atomicAdd(S.diag + CD_DENSE, 1ull);
      grid.sync();
    }
    // ---- E: chunk maxima that lost their argmax; re-arm parity nxt
    if (S.track) refresh_chunks(S, S.par, false, sh);
    if (tid == 0) {
      S.dcnt[nxt] = 0;
      S.dense[nxt] = 0;
      atomicAdd(S.diag + CD_STEPS, 1ull);
    }
    grid.sync();
  }
}

__global__ void k_cs_uncover(uint32_t *E, const unsigned long long *list, unsigned long long cnt) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (size_t)gridDim.x * blockDim.x)
    atomicAnd(E + 2 * list[i], ~COV);
}

// ---------------------------------------------------- lazy selector (f2)
// fresh marginal gain of cand[t] (one warp per candidate): sum over the slots
// of |C_j(v)| unless covered; singleton slots count 1 (R17)
__global__ void k_cs_lazy_eval(CSel S, const uint32_t *cand, uint32_t b0, uint32_t b1,
                               long long *delta) {
  const int lane = threadIdx.x & 31;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t t = b0 + warp; t < b1; t += nw) {
    const uint32_t v = cand[t];
    if (__ldcg(delta + v) < 0) continue;  // a seed (R6)
    const uint32_t row = S.cid ? S.cid[v] : v;
    long long g = 0;
    if (row == NONE) {
      g = S.B;
    } else {
      for (uint32_t j = lane; j < S.B; j += 32) {
        const uint2 r = S.rec[(size_t)row * S.MW + (j >> 5)];
        if (!((r.y >> (j & 31)) & 1u)) {
          g += 1;
          continue;
        }
        const uint32_t e = r.x + __popc(r.y & ((1u << (j & 31)) - 1u));
        const uint32_t x = __ldcg(S.E + 2 * (size_t)e);
        const uint32_t rv = (x & PACIM_HIGH) ? x : __ldcg(S.E + 2 * (size_t)x);
        if (!(rv & COV)) g += rv & SIZE;
      }
      for (int d = 16; d; d >>= 1) g += __shfl_xor_sync(FULL, g, d);
    }
    if (lane == 0) delta[v] = g;
  }
}

__global__ void k_cs_lazy_mark(CSel S, uint32_t s) {
  const uint32_t srow = S.cid ? S.cid[s] : s;
  if (srow == NONE) return;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < S.B; j += gridDim.x * blockDim.x) {
    const uint2 r = S.rec[(size_t)srow * S.MW + (j >> 5)];
    if (!((r.y >> (j & 31)) & 1u)) continue;
    const uint32_t e = r.x + __popc(r.y & ((1u << (j & 31)) - 1u));
    const uint32_t x = S.E[2 * (size_t)e];
    const uint32_t root = (x & PACIM_HIGH) ? e : x;
    if (!(atomicOr(S.E + 2 * (size_t)root, COV) & COV)) {
      const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
      if (at < S.cov_cap) S.cov_list[at] = root;
    }
  }
}

// ---------------------------------------------- Win-Tree selector (f2)
// The paper's Win-Tree: an implicit winning tree T[1..2N-1]
// over the stale scores key[v] (N = 2^ceil(log2 n) leaves, T[N + v] = v),
// each internal node the id of its children's winner (key desc, id asc).
// NextSeed = FindMax from the root with Delta* the best fresh score so far:
// a node whose id is stale (not re-evaluated in this step) and cannot beat
// Delta* prunes its whole subtree; a stale id that can is re-evaluated
// (fresh marginal gain from the store, R17) and the search continues into
// both children; a fresh id (re-evaluated at an ancestor) is passed through.
// Level-synchronous in ONE block of 1024 threads (the frontier of the
// paper's parallel recursion one level at a time); then MarkSeed and the
// winners of the explored nodes recomputed bottom-up.  Evaluations counted.
constexpr int WT_THREADS = 1024;

__device__ __forceinline__ uint32_t wt_win(const long long *key, uint32_t a, uint32_t b) {
  if (a == NONE) return b;
  if (b == NONE) return a;
  const long long ka = key[a], kb = key[b];
  return (ka > kb || (ka == kb && a < b)) ? a : b;
}

// fresh marginal gain of v: sum over the slots of |C_j(v)| unless covered;
// a singleton slot counts 1 (one warp)
__device__ long long cs_eval(const CSel &S, uint32_t v) {
  const int lane = threadIdx.x & 31;
  const uint32_t row = S.cid ? S.cid[v] : v;
  long long g = 0;
  if (row == NONE) return S.B;
  for (uint32_t j = lane; j < S.B; j += 32) {
    const uint2 r = S.rec[(size_t)row * S.MW + (j >> 5)];
    if (!((r.y >> (j & 31)) & 1u)) {
      g += 1;
      continue;
    }
    const uint32_t e = r.x + __popc(r.y & ((1u << (j & 31)) - 1u));
    const uint32_t x = __ldcg(S.E + 2 * (size_t)e);
    const uint32_t rv = (x & PACIM_HIGH) ? x : __ldcg(S.E + 2 * (size_t)x);
    if (!(rv & COV)) g += rv & SIZE;
  }
  for (int d = 16; d; d >>= 1) g += __shfl_xor_sync(FULL, g, d);
  return g;
}

struct WTc {
  uint32_t *T;
  uint32_t N, D;        // leaves (2^D), tree depth
  long long *key;
  uint32_t *H0, *H1;    // hanging subtree roots of the current / next wave (2N each)
  uint32_t *Ev, *Et;    // the wave's re-evaluations: vertex, the hanging root it came from
  uint32_t *X;          // the step's re-evaluated vertices (the repaired paths)
  uint32_t *seeds;
  long long *gain_num;
  unsigned long long *evals;
};

// FindMax in waves (the same exploration as the paper's recursion, P:2690-
// 2700, scheduled by re-evaluation instead of by tree level): H = the roots of
// the subtrees hanging off the paths explored so far (initially the root).
// A wave takes every h in H whose (stale) winner can still beat Delta*,
// re-evaluates those winners, and replaces h by the siblings along the path
// from h down to the winner's leaf; it ends when no hanging winner can beat
// Delta*.  Each subtree root is pushed at most once per step (the subtrees of
// different hanging roots are disjoint).  Then MarkSeed and the winners on
// the re-evaluated vertices' paths recomputed bottom-up.
__global__ void __launch_bounds__(WT_THREADS, 1) k_cs_wintree(CSel S, WTc W, uint32_t k) {
  __shared__ uint32_t nh, nn, ne, nx;
  __shared__ Best sh[33];
  __shared__ Best best;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long evals = 0, nodes = 0;
  uint32_t *H = W.H0, *Hn = W.H1;
  for (uint32_t step = 0; step < k; step++) {
    if (threadIdx.x == 0) {
      H[0] = 1;
      nh = 1;
      nx = 0;
      best = Best{LLONG_MIN, NONE};
    }
    __syncthreads();
    for (;;) {
      if (threadIdx.x == 0) {
        ne = 0;
        nn = 0;
      }
      __syncthreads();
      // hanging winners that can beat Delta* (stale: none of them was
      // re-evaluated in this step, their subtrees being disjoint from the
      // explored paths)
      const Best cur = best;
      const uint32_t nhh = nh;
      for (uint32_t i = threadIdx.x; i < nhh; i += blockDim.x) {
        const uint32_t t = H[i];
        const uint32_t id = W.T[t];
        if (id == NONE || !better(W.key[id], id, cur.g, cur.v)) continue;
        const uint32_t at = atomicAdd(&ne, 1u);
        W.Ev[at] = id;
        W.Et[at] = t;
      }
      nodes += nhh;
      __syncthreads();
      const uint32_t nev = ne;
      if (nev == 0) break;
      Best mine{LLONG_MIN, NONE};
      for (uint32_t q = wid; q < nev; q += WT_THREADS / 32) {
        const uint32_t v = W.Ev[q];
        const long long g = cs_eval(S, v);
        if (lane == 0) W.key[v] = g;
        if (better(g, v, mine.g, mine.v)) mine = Best{g, v};
      }
      evals += nev;
      Best lb = block_best(mine, sh);
      if (threadIdx.x == 0 && better(lb.g, lb.v, best.g, best.v)) best = lb;
      __syncthreads();
      // the siblings along each re-evaluated path, from its hanging root down
      const Best nb = best;
      for (uint32_t q = threadIdx.x; q < nev * W.D; q += blockDim.x) {
        const uint32_t e = q / W.D, l = q % W.D;
        const uint32_t t = W.Et[e], leaf = W.N + W.Ev[e];
        const uint32_t p = leaf >> l;
        if (p <= t) continue;  // at or above the hanging root
        const uint32_t sib = p ^ 1u, sid = W.T[sib];
        if (sid != NONE && better(W.key[sid], sid, nb.g, nb.v)) Hn[atomicAdd(&nn, 1u)] = sib;
      }
      for (uint32_t q = threadIdx.x; q < nev; q += blockDim.x) W.X[nx + q] = W.Ev[q];
      __syncthreads();
      if (threadIdx.x == 0) {
        nx += nev;
        nh = nn;
      }
      uint32_t *tmp = H;
      H = Hn;
      Hn = tmp;
      __syncthreads();
    }
    const uint32_t s = best.v;
    const long long g = best.g;
    // MarkSeed(s) (covered bits; the lazy selector updates no member)
    const uint32_t srow = S.cid ? S.cid[s] : s;
    if (srow != NONE)
      for (uint32_t j = threadIdx.x; j < S.B; j += blockDim.x) {
        const uint2 r = S.rec[(size_t)srow * S.MW + (j >> 5)];
        if (!((r.y >> (j & 31)) & 1u)) continue;
        const uint32_t e = r.x + __popc(r.y & ((1u << (j & 31)) - 1u));
        const uint32_t x = S.E[2 * (size_t)e];
        const uint32_t root = (x & PACIM_HIGH) ? e : x;
        if (!(atomicOr(S.E + 2 * (size_t)root, COV) & COV)) {
          const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
          if (at < S.cov_cap) S.cov_list[at] = root;
        }
      }
    if (threadIdx.x == 0) {
      W.key[s] = -1;  // s leaves the candidate set (R6); s is one of X
      W.seeds[step] = s;
      W.gain_num[step] = g;
    }
    __syncthreads();
    // the winners on the re-evaluated vertices' paths, bottom-up (a level at
    // a time: the children of a level are final before it is recomputed)
    const uint32_t nxx = nx;
    for (uint32_t l = 1; l <= W.D; l++) {
      for (uint32_t q = threadIdx.x; q < nxx; q += blockDim.x) {
        const uint32_t t = (W.N + W.X[q]) >> l;
        W.T[t] = wt_win(W.key, W.T[2 * t], W.T[2 * t + 1]);
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    W.evals[0] = evals;
    W.evals[1] = nodes;
  }
}

// leaves and one level of internal winners of the initial Win-Tree
__global__ void k_wt_leaves(uint32_t *T, uint32_t N, uint32_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    T[N + i] = i < n ? (uint32_t)i : NONE;
}

__global__ void k_wt_level(uint32_t *T, const long long *key, uint32_t lo, uint32_t hi) {
  for (size_t t = lo + (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < hi;
       t += (size_t)gridDim.x * blockDim.x)
    T[t] = wt_win(key, T[2 * t], T[2 * t + 1]);
}

// ------------------------------------------------------------- labels
__global__ void k_cs_labels(const CSel S, uint32_t j, uint32_t *out) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < S.nv;
       v += (size_t)gridDim.x * blockDim.x) {
    const uint32_t row = S.cid ? S.cid[v] : (uint32_t)v;
    uint32_t lab = (uint32_t)v;
    if (row != NONE) {
      const uint2 r = S.rec[(size_t)row * S.MW + (j >> 5)];
      if ((r.y >> (j & 31)) & 1u) {
        const uint32_t e = r.x + __popc(r.y & ((1u << (j & 31)) - 1u));
        const uint32_t x = S.E[2 * (size_t)e];
        lab = S.vid[(x & PACIM_HIGH) ? e : x];  // the root entry's vertex (R8: min id)
      }
    }
    out[v] = lab;
  }
}

}  // namespace

// ------------------------------------------------------------------ host
static float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

void pc_cs_free(pacim_ctx *ctx) {
  for (DevBuf *d : {&ctx->cs_rec, &ctx->cs_soff, &ctx->cs_ecrow, &ctx->cs_E, &ctx->cs_vid,
                    &ctx->cs_diag, &ctx->cs_cnt, &ctx->cs_plist})
    pc_free(ctx, *d);
  ctx->cs = false;
}

// The compact build.  Returns false (nothing changed but the scratch) when the
// store would not be compact: more than half of the (row, slot) pairs are
// non-singletons (c3: p = 1/2 on a grid), or 2^31 entries or more.
bool pc_cs_build(pacim_ctx *ctx) {
  const uint32_t nr = ctx->nr, B = ctx->R_local, n = ctx->n;
  bool force = false;
  if (const char *e = getenv("PACIM_STORE")) {
    if (std::string(e) == "dense") return false;
    force = std::string(e) == "compact";
  } else if (getenv("PACIM_L2_BUDGET")) {
    return false;  // the slot-window layout is a dense-store experiment
  }
  if (B > 256 || nr == 0 || ctx->compressed) return false;
  // The store: one GPU -> the dense vertex-major store (its build is faster:
  // the compact store adds a mask pass and an indirection per union, c4 r02:
  // 81 vs 58 ms) unless it does not fit; a sharded build -> the compact store
  // (the fast NCCL select walks its member lists; the dense store would need a
  // dense all-reduce per step).  PACIM_STORE = compact | dense forces one.
  if (!force && ctx->world == 1 && !pc_dist_active(ctx)) {
    size_t fr = 0, tot = 0;
    pc_mem_info(ctx, &fr, &tot);
    fr += ctx->L.bytes;  // an earlier dense store is reused
    if ((size_t)nr * B * 4 <= fr / 2) return false;
  }
  // an earlier build of this graph with these many slots found the sketches
  // too dense for the compact store (the mask pass is not repeated)
  if (!force && ctx->cs_pref_gen == ctx->hint_gen && ctx->cs_pref_B == B && ctx->cs_pref_dense)
    return false;
  const uint32_t MW = (B + 31) / 32;
  pc_slot_table(ctx);
  pc_ensure(ctx, ctx->counters, 64 * sizeof(uint64_t));
  unsigned long long *ctr = ctx->counters.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(ctr, 0, 64 * sizeof(uint64_t), ctx->stream));
  ctx->launches = 0;
  // phase events: named marks after each kernel (PACIM_BUILD_TIMES=1 prints them)
  std::vector<std::pair<const char *, cudaEvent_t>> marks;
  auto mark = [&](const char *name) {
    cudaEvent_t e;
    PC_CUDA(cudaEventCreate(&e));
    PC_CUDA(cudaEventRecord(e, ctx->stream));
    marks.push_back({name, e});
  };
  struct Cleanup {
    std::vector<std::pair<const char *, cudaEvent_t>> &m;
    ~Cleanup() {
      for (auto &x : m) cudaEventDestroy(x.second);
    }
  } cleanup{marks};
  const uint64_t nnz = 2 * ctx->m;
  mark("start");
  // ---- masks (the rec array, .y words)
  pc_ensure(ctx, ctx->cs_rec, (size_t)nr * MW * 8);
  PC_CUDA(cudaMemsetAsync(ctx->cs_rec.p, 0, (size_t)nr * MW * 8, ctx->stream));
  // the pair list: the union pass reads the mask pass's live pairs instead of
  // hashing every edge again (c4 shard of 32 sketches: 14 ms per edge pass);
  // sized by the last build of this graph / slot count / key, else a quarter
  // of the free memory; an overflow falls back to the full union pass
  // (PACIM_CS_PAIRLIST = 0: no list; > 1: that capacity, for tests)
  unsigned long long pcap = 0;
  const long long pl_env = getenv("PACIM_CS_PAIRLIST") ? atoll(getenv("PACIM_CS_PAIRLIST")) : 1;
  // the list pays when live pairs are rare per edge: its union pass costs
  // ~60 ps per pair, the full pass ~9 ps per edge plus the unions (c4 builds
  // of one rank's shard: 256 slots, 0.34 pairs per edge: 90 vs 83 ms; 128
  // slots: 58 vs 56; 64: 38 vs 42; 32: 25.5 vs 33.6); the rate of the last
  // build of this graph and key decides, else the slot count
  const bool same = ctx->cs_live_gen == ctx->hint_gen && ctx->cs_live_K == ctx->K &&
                    ctx->cs_live_rate >= 0;
  const bool want_list = pl_env > 1 || (same ? ctx->cs_live_rate * B < 0.12 : B <= 64);
  if (nr < (1u << 28) && B <= 256 && pl_env != 0 && want_list) {
    if (pl_env > 1) {
      pcap = (unsigned long long)pl_env;
    } else if (same && ctx->cs_live_B == B) {
      pcap = ctx->cs_live_hint + ctx->cs_live_hint / 16 + (1ull << 22);  // + chunk holes
    } else {
      size_t fr = 0, tot = 0;
      pc_mem_info(ctx, &fr, &tot);
      fr += ctx->cs_plist.bytes;
      pcap = std::min<unsigned long long>(fr / 4 / 8, 1ull << 33);
    }
    if (ctx->cs_plist.bytes < pcap * 8 || ctx->cs_plist.bytes > 2 * pcap * 8 + (64ull << 20)) {
      pc_free(ctx, ctx->cs_plist);
      pc_ensure(ctx, ctx->cs_plist, pcap * 8);
    }
  }
  // a sharded build with a communicator: the edge-partitioned pairs (each
  // rank tests 1/P of the edges against all sketches, NCCL routes the pairs
  // to the sketches' owners; dist.cu) instead of every rank's full mask pass
  const unsigned long long ep = nnz ? pc_cs_ep_pairs(ctx, MW, ctr) : ~0ull;
  if (ep != ~0ull) {
    pcap = std::max<unsigned long long>(ep, 1);  // the union pass reads the received pairs
    const unsigned long long two[1] = {ep};
    PC_CUDA(cudaMemcpyAsync(ctr + 13, two, 8, cudaMemcpyHostToDevice, ctx->stream));  // live
    PC_CUDA(cudaMemcpyAsync(ctr + 16, two, 8, cudaMemcpyHostToDevice, ctx->stream));  // list
  } else if (nnz) {  // the upper edges (the k_edges scheme): both endpoints' bits per live pair
    pc_cs_mask_edges(ctx, ctx->cs_rec.as<uint32_t>(), MW, ctr + 8,
                     pcap ? ctx->cs_plist.as<unsigned long long>() : nullptr, ctr + 16, pcap);
  }
  mark("mask");
  // ---- counts -> entry offsets (build scratch kept by the ctx)
  pc_ensure(ctx, ctx->cs_cnt, 2 * ((size_t)nr + 1) * 8);
  uint64_t *c64 = ctx->cs_cnt.as<uint64_t>(), *pos = c64 + nr + 1;
  k_cs_count<<<pc_grid(ctx, nr + 1, 256), 256, 0, ctx->stream>>>(ctx->cs_rec.as<uint2>(), nr, MW, c64);
  PC_CHECK_LAUNCH();
  pc_exclusive_scan_u64(ctx, c64, pos, (size_t)nr + 1);
  uint64_t total = 0;
  unsigned long long npairs = 0, nlive = 0;
  PC_CUDA(cudaMemcpyAsync(&total, pos + nr, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(&npairs, ctr + 16, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(&nlive, ctr + 13, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->cs_live_gen = ctx->hint_gen;
  ctx->cs_live_K = ctx->K;
  ctx->cs_live_rate = ctx->m ? (double)nlive / ((double)ctx->m * B) : 0.0;
  ctx->cs_live_B = pcap ? B : 0;
  ctx->cs_live_hint = npairs;
  ctx->launches += 2;
  mark("scan");
  // above half non-singleton pairs (c3: p = 1/2 on a grid) the compact store
  // is larger than the dense one
  const double dmax = getenv("PACIM_CS_DENSITY") ? atof(getenv("PACIM_CS_DENSITY")) : 0.5;
  const bool dense = total >= (1ull << 31) || (double)total > dmax * (double)nr * B;
  ctx->cs_pref_gen = ctx->hint_gen;
  ctx->cs_pref_B = B;
  ctx->cs_pref_dense = dense;
  if (dense) {
    pc_free(ctx, ctx->cs_rec);
    return false;  // dense: the vertex-major store is the better layout
  }
  // the dense store of an earlier build and the compressed store go first
  for (DevBuf *d : {&ctx->L, &ctx->clabel, &ctx->csz, &ctx->csz_work, &ctx->Ltmp, &ctx->cwork,
                    &ctx->hla_off, &ctx->hla_row, &ctx->hla_raw, &ctx->pkeys})
    pc_free(ctx, *d);
  ctx->hla_ok = false;
  ctx->cs_MW = MW;
  ctx->cs_total = total;
  const uint64_t T1 = std::max<uint64_t>(total, 1);
  pc_ensure(ctx, ctx->cs_soff, ((size_t)nr + 1) * 4);
  pc_ensure(ctx, ctx->cs_ecrow, (T1 / 32 + 2) * 4);
  pc_ensure(ctx, ctx->cs_E, T1 * 8);
  pc_ensure(ctx, ctx->cs_vid, T1 * 4);
  k_cs_rec<<<pc_grid(ctx, nr, 256), 256, 0, ctx->stream>>>(
      ctx->cs_rec.as<uint2>(), nr, MW, pos, ctx->cs_soff.as<uint32_t>(), ctx->cs_ecrow.as<uint32_t>());
  PC_CHECK_LAUNCH();
  mark("rec");
  uint2 *E = ctx->cs_E.as<uint2>();
  uint32_t *Ew = ctx->cs_E.as<uint32_t>();
  k_cs_fill<<<pc_grid(ctx, total, 256), 256, 0, ctx->stream>>>(E, total);
  PC_CHECK_LAUNCH();
  ctx->launches += 2;
  mark("init");
  // ---- unions (H2, H3) on the P words (stride 2): from the pair list, or
  // (none, or it overflowed) over every edge again
  if (pcap && npairs <= pcap) {
    if (npairs)
      pc_cs_list_unite(ctx, Ew, ctx->cs_rec.as<uint2>(), MW, ctx->cs_plist.as<unsigned long long>(),
                       npairs, ctr, ctr + 13);  // the mask pass's live count (ctr + 8 + 1 + 4)
  } else {
    pc_cs_edges(ctx, Ew, ctx->cs_rec.as<uint2>(), MW, ctr);
  }
  mark("edges");
  // ---- compression, sizes, member lists (H4, H5, H6u)
  pc_ensure(ctx, ctx->d_hot, 2 * (size_t)B * 4);
  uint32_t *hot = ctx->d_hot.as<uint32_t>();
  // the hub's CCs are "hot" (counted in shared memory, covered by the hot sums)
  // when they are expected to be giant: its expected live degree (deg * p)
  // is large (c2: 163K * 0.02; never under WIC, whose hub edges have p ~ 1/deg)
  double pm = (double)ctx->t32 / 4294967296.0;
  if (ctx->pmodel == PACIM_P_UNIFORM)
    pm = 0.5 * ((double)(ctx->t32 >> 32) + (double)(ctx->t32 & 0xFFFFFFFFull)) / 4294967296.0;
  const bool hot_on = ctx->pmodel != PACIM_P_WIC && (double)ctx->hub_degree * pm >= 64.0 &&
                      !getenv("PACIM_NO_HOT");
  k_cs_hot<<<(B + 255) / 256, 256, 0, ctx->stream>>>(ctx->cs_rec.as<uint2>(), MW, Ew,
                                                     hot_on ? ctx->hub_row : NONE, nr, B, hot);
  PC_CHECK_LAUNCH();
  k_cs_compress<<<pc_grid(ctx, total, CS_THREADS, 8), CS_THREADS, 0, ctx->stream>>>(Ew, total, hot,
                                                                                   B, ctr);
  PC_CHECK_LAUNCH();
  pc_ensure(ctx, ctx->d_hot_size, (size_t)B * 4);
  k_cs_hot_sizes<<<(B + 255) / 256, 256, 0, ctx->stream>>>(Ew, hot, B, ctx->d_hot_size.as<uint32_t>());
  PC_CHECK_LAUNCH();
  ctx->launches += 3;
  mark("compress");
  // ---- gain0 (H7), hot sums, vertex of each entry
  ctx->cs_list_t = getenv("PACIM_BIG_T") ? (uint32_t)std::max(1LL, atoll(getenv("PACIM_BIG_T")))
                                         : LIST_T;
  ctx->hot_size.resize(B);
  PC_CUDA(cudaMemcpyAsync(ctx->hot_size.data(), ctx->d_hot_size.p, (size_t)B * 4,
                          cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  bool any = false;
  for (uint32_t j = 0; j < B; j++) any |= ctx->hot_size[j] > 0;
  ctx->hot_any = any;
  ctx->hot_big_t = 0;
  if (any) pc_ensure(ctx, ctx->hotsum, (size_t)n * 8);
  pc_ensure(ctx, ctx->gain0, (size_t)n * 8);
  k_cs_gain_init<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(
      ctx->lean ? nullptr : ctx->cid.as<uint32_t>(), ctx->cs_soff.as<uint32_t>(), n, B,
      ctx->gain0.as<int64_t>(), any ? ctx->hotsum.as<int64_t>() : nullptr);
  PC_CHECK_LAUNCH();
  {
    auto kern = any ? k_cs_gain<true> : k_cs_gain<false>;
    kern<<<pc_grid(ctx, total, CS_THREADS, 8), CS_THREADS, 0, ctx->stream>>>(
        Ew, total, ctx->cs_soff.as<uint32_t>(), ctx->cs_ecrow.as<uint32_t>(),
        ctx->lean ? nullptr : ctx->rmap.as<uint32_t>(), B, hot, ctx->cs_vid.as<uint32_t>(),
        ctx->gain0.as<int64_t>(), any ? ctx->hotsum.as<int64_t>() : nullptr, ctr);
    PC_CHECK_LAUNCH();
  }
  ctx->launches += 2;
  mark("gain");
  unsigned long long h[6];
  PC_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->cs = true;
  ctx->ncomp = h[0];
  ctx->nnonsingle = total;
  ctx->nmember = total;
  ctx->stats.live_pairs = h[4];
  PC_REQUIRE(h[0] + h[1] == total, PACIM_ECHECK, "compact store: roots + non-roots != entries");
  auto span = [&](const char *a, const char *b) {
    cudaEvent_t ea = nullptr, eb = nullptr;
    for (auto &x : marks) {
      if (!strcmp(x.first, a)) ea = x.second;
      if (!strcmp(x.first, b)) eb = x.second;
    }
    return ev_ms(ea, eb);
  };
  ctx->stats.t_init_ms = span("start", "init");      // masks, offsets, records, E
  ctx->stats.t_edges_ms = span("init", "edges");
  ctx->stats.t_compress_ms = span("edges", "compress");
  ctx->stats.t_compact_ms = 0;
  ctx->stats.t_gain_ms = span("compress", "gain");
  ctx->stats.t_centers_ms = 0;
  ctx->stats.t_build_ms = span("start", "gain");
  ctx->stats.kernel_launches_build = ctx->launches;
  if (getenv("PACIM_BUILD_TIMES")) {
    fprintf(stderr, "cs build ms:");
    for (size_t i = 1; i < marks.size(); i++)
      fprintf(stderr, " %s %.3f", marks[i].first, ev_ms(marks[i - 1].second, marks[i].second));
    fprintf(stderr, " | total %.3f entries %llu\n", ctx->stats.t_build_ms,
            (unsigned long long)total);
  }
  ctx->sel_list_valid = false;
  return true;
}

// ------------------------------------------------------------ selection
static CSel make_csel(pacim_ctx *ctx, long long *target) {
  const uint32_t B = ctx->R_local, n = ctx->n;
  CSel S;
  S.rec = ctx->cs_rec.as<uint2>();
  S.MW = ctx->cs_MW;
  S.E = ctx->cs_E.as<uint32_t>();
  S.vid = ctx->cs_vid.as<uint32_t>();
  S.soff = ctx->cs_soff.as<uint32_t>();
  S.rmap = ctx->lean ? nullptr : ctx->rmap.as<uint32_t>();
  S.cid = ctx->lean ? nullptr : ctx->cid.as<uint32_t>();
  S.nr = ctx->nr;
  S.B = B;
  S.nv = n;
  S.total = ctx->cs_total;
  S.list_t = ctx->cs_list_t;
  S.target = target;
  S.hotsum = ctx->hot_any ? ctx->hotsum.as<int64_t>() : nullptr;
  S.hot_root = ctx->d_hot.as<uint32_t>();
  uint32_t csh = 10;
  while (((uint64_t)n + (1ull << csh) - 1) >> csh > MAX_CHUNKS) csh++;
  S.csh = csh;
  S.nchunks = (uint32_t)(((uint64_t)n + (1ull << csh) - 1) >> csh);
  S.cov_cap = (uint64_t)std::max<uint32_t>(ctx->sel_k_cap, 128) * B;
  // sel_list: cov_root[B], cov_delta[B], dense[2], pad | cov_cnt, cov_list[cap]
  const size_t head_words = (2 * (size_t)B + 2 + 1) & ~(size_t)1;
  pc_ensure(ctx, ctx->sel_list, head_words * 4 + 8 + 8 * S.cov_cap + 64);
  uint32_t *base = ctx->sel_list.as<uint32_t>();
  S.cov_root = base;
  S.cov_delta = base + B;
  S.dense = reinterpret_cast<int *>(base + 2 * (size_t)B);
  S.cov_cnt = reinterpret_cast<unsigned long long *>(base + head_words);
  S.cov_list = S.cov_cnt + 1;
  pc_ensure(ctx, ctx->sel_partial, (size_t)S.nchunks * (sizeof(Best) + 12) + 64);
  S.cmax = ctx->sel_partial.as<Best>();
  S.cdirty = reinterpret_cast<uint32_t *>(S.cmax + S.nchunks);
  S.dlist = S.cdirty + S.nchunks;
  S.dcnt = S.dlist + 2 * (size_t)S.nchunks;
  pc_ensure(ctx, ctx->cs_diag, CD_WORDS * 8);
  S.diag = ctx->cs_diag.as<unsigned long long>();
  S.par = 0;
  S.track = 0;
  S.dlst = ctx->dlist;
  S.celf = nullptr;
  return S;
}

static void cs_uncover(pacim_ctx *ctx, const CSel &S) {
  unsigned long long cnt = 0;
  if (ctx->sel_list_valid) {
    PC_CUDA(cudaMemcpyAsync(&cnt, S.cov_cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  PC_REQUIRE(cnt <= S.cov_cap, PACIM_ECHECK, "covered-CC list overflowed");
  if (cnt) k_cs_uncover<<<pc_grid(ctx, cnt, 256), 256, 0, ctx->stream>>>(S.E, S.cov_list, cnt);
  PC_CUDA(cudaMemsetAsync(S.cov_cnt, 0, 8, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.dense, 0, 8, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.cov_root, 0xFF, (size_t)S.B * 4, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.diag, 0, CD_WORDS * 8, ctx->stream));
  ctx->sel_list_valid = true;
}

static void cs_grow_list(pacim_ctx *ctx, uint32_t k) {
  if (k > ctx->sel_k_cap) {
    if (ctx->sel_list_valid) {
      CSel old = make_csel(ctx, nullptr);
      cs_uncover(ctx, old);
    }
    ctx->sel_k_cap = k;
    ctx->sel_list_valid = false;
  }
}

void pc_cs_select_reset(pacim_ctx *ctx) {
  pc_dist_restore(ctx);
  CSel S = make_csel(ctx, nullptr);
  cs_uncover(ctx, S);
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

static unsigned cs_sel_grid(pacim_ctx *ctx) {
  int occ = 0;
  PC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cs_select, SEL_THREADS, 0));
  PC_REQUIRE(occ >= 1, PACIM_ECUDA, "k_cs_select cannot be resident");
  return (unsigned)ctx->sm_count;
}

void pc_cs_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                  int64_t *sigma_num) {
  const uint32_t n = ctx->n;
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  cs_grow_list(ctx, k);
  pc_dist_restore(ctx);
  CSel S = make_csel(ctx, ctx->gain.as<long long>());
  S.track = 1;
  pc_ensure(ctx, ctx->sel_gain, (size_t)k * 16 + 64);
  pc_ensure(ctx, ctx->sel_seeds, (size_t)k * 4);
  CSelOut O;
  O.k = k;
  O.given = NONE;
  O.seeds = ctx->sel_seeds.as<uint32_t>();
  O.gain_num = ctx->sel_gain.as<long long>();
  O.arg_gain = O.gain_num + k;
  const unsigned grid = cs_sel_grid(ctx);
  cudaEvent_t e0, e1;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  cs_uncover(ctx, S);
  PC_CUDA(cudaMemcpyAsync(ctx->gain.p, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  PC_CUDA(cudaMemsetAsync(ctx->sel_gain.p, 0, (size_t)k * 16 + 64, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.cdirty, 0, (size_t)S.nchunks * 4, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.dcnt, 0, 8, ctx->stream));
  TmpBuf celf(ctx);
  if (getenv("PACIM_CELF_COUNT")) {  // CELF's evaluation count on the same gains (f2)
    pc_ensure(ctx, celf, (size_t)n * 8);
    PC_CUDA(cudaMemcpyAsync(celf.p, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice,
                            ctx->stream));
    S.celf = celf.as<long long>();
  }
  uint32_t par0 = ctx->sel_par;
  void *args[] = {&S, &O, &par0};
  PC_CUDA(cudaLaunchCooperativeKernel((void *)k_cs_select, grid, SEL_THREADS, args, 0, ctx->stream));
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  std::vector<long long> hg(2 * (size_t)k);
  unsigned long long d[CD_WORDS];
  PC_CUDA(cudaMemcpyAsync(seeds, O.seeds, (size_t)k * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(hg.data(), O.gain_num, (2 * (size_t)k) * 8, cudaMemcpyDeviceToHost,
                          ctx->stream));
  PC_CUDA(cudaMemcpyAsync(d, S.diag, sizeof(d), cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms = ms;
  ctx->stats.kernel_launches_select = 2;
  ctx->stats.select_member_updates = d[CD_UPD];
  ctx->stats.select_dense_steps = d[CD_DENSE];
  ctx->stats.select_hotsum_steps = d[CD_HOT];
  ctx->stats.select_celf_evaluations = d[CD_CELF];
  ctx->stats.select_evaluations = 0;  // the lazy selectors' counters
  ctx->stats.select_eval_rounds = 0;
  ctx->stats.select_bfs_visits = 0;
  ctx->stats.select_warp_slots = ctx->stats.select_deferred_slots = 0;
  ctx->stats.select_row_items = ctx->stats.select_chunk_items = 0;
  ctx->stats.select_inline_rows = ctx->stats.select_edges = 0;
  ctx->sel_par = (par0 + k) & 1;
  long long run = 0;
  bool ok = true;
  for (uint32_t i = 0; i < k; i++) {
    gain_num[i] = hg[i];
    ok &= hg[i] == hg[k + i];
    run += hg[i];
    sigma_num[i] = run;
  }
  PC_REQUIRE(ok, PACIM_ECHECK, "select: sum_r delta_r differs from the argmax gain");
}

void pc_cs_cover_local(pacim_ctx *ctx, uint32_t s, int64_t *d_delta, int64_t *local_gain) {
  PC_REQUIRE(ctx->sel_list_valid, PACIM_ESTATE, "pacim_select_reset first");
  CSel S = make_csel(ctx, reinterpret_cast<long long *>(d_delta));
  pc_ensure(ctx, ctx->sel_gain, 64);
  pc_ensure(ctx, ctx->sel_seeds, 16);
  CSelOut O;
  O.k = 1;
  O.given = s;
  O.seeds = ctx->sel_seeds.as<uint32_t>();
  O.gain_num = ctx->sel_gain.as<long long>();
  O.arg_gain = O.gain_num + 1;
  PC_CUDA(cudaMemsetAsync(O.gain_num, 0, 16, ctx->stream));
  const unsigned grid = cs_sel_grid(ctx);
  uint32_t par0 = ctx->sel_par;
  void *args[] = {&S, &O, &par0};
  PC_CUDA(cudaLaunchCooperativeKernel((void *)k_cs_select, grid, SEL_THREADS, args, 0, ctx->stream));
  ctx->sel_par ^= 1;
  long long h = 0;
  PC_CUDA(cudaMemcpyAsync(&h, O.gain_num, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  *local_gain = (int64_t)h;
}

void pc_cs_get_labels(pacim_ctx *ctx, uint32_t slot, uint32_t *host_out) {
  CSel S = make_csel(ctx, nullptr);
  TmpBuf t(ctx);
  pc_ensure(ctx, t, (size_t)ctx->n * 4);
  k_cs_labels<<<pc_grid(ctx, ctx->n, 256), 256, 0, ctx->stream>>>(S, slot, t.as<uint32_t>());
  PC_CHECK_LAUNCH();
  PC_CUDA(cudaMemcpyAsync(host_out, t.p, (size_t)ctx->n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

void pc_cs_lazy_eval(pacim_ctx *ctx, const uint32_t *cand, uint32_t b0, uint32_t b1,
                     long long *delta) {
  CSel S = make_csel(ctx, delta);
  k_cs_lazy_eval<<<pc_grid(ctx, (size_t)(b1 - b0) * 32, 256, 8), 256, 0, ctx->stream>>>(S, cand, b0,
                                                                                        b1, delta);
  PC_CHECK_LAUNCH();
}

void pc_cs_lazy_mark(pacim_ctx *ctx, uint32_t s) {
  CSel S = make_csel(ctx, nullptr);
  k_cs_lazy_mark<<<(S.B + 255) / 256, 256, 0, ctx->stream>>>(S, s);
  PC_CHECK_LAUNCH();
}

// NEXT f2: the Win-Tree selector (selector 2).  One single-block kernel runs
// all k steps; the tree and the stale scores live in device memory.
void pc_cs_select_wintree(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                          int64_t *sigma_num) {
  const uint32_t n = ctx->n;
  uint32_t N = 1, depth = 0;
  while (N < n) {
    N <<= 1;
    depth++;
  }
  cs_grow_list(ctx, k);
  pc_dist_restore(ctx);
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  CSel S = make_csel(ctx, ctx->gain.as<long long>());
  // persistent scratch (capacity reused): T[2N], H0[2N], H1[2N], Ev[N], Et[N], X[N], outputs
  DevBuf &wb = ctx->wt_buf;
  pc_ensure(ctx, wb, (size_t)9 * N * 4 + (size_t)k * 12 + 64);
  WTc W;
  W.T = wb.as<uint32_t>();
  W.H0 = W.T + 2 * (size_t)N;
  W.H1 = W.H0 + 2 * (size_t)N;
  W.Ev = W.H1 + 2 * (size_t)N;
  W.Et = W.Ev + N;
  W.X = W.Et + N;
  W.gain_num = reinterpret_cast<long long *>(
      (reinterpret_cast<uintptr_t>(W.X + N) + 7) & ~(uintptr_t)7);
  W.seeds = reinterpret_cast<uint32_t *>(W.gain_num + k);
  W.evals = reinterpret_cast<unsigned long long *>(
      (reinterpret_cast<uintptr_t>(W.seeds + k) + 7) & ~(uintptr_t)7);
  W.N = N;
  W.D = depth;
  W.key = ctx->gain.as<long long>();
  cudaEvent_t e0, e1;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  cs_uncover(ctx, S);
  PC_CUDA(cudaMemcpyAsync(W.key, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  k_wt_leaves<<<pc_grid(ctx, N, 256), 256, 0, ctx->stream>>>(W.T, N, n);
  for (uint32_t lo = N >> 1; lo >= 1; lo >>= 1)
    k_wt_level<<<pc_grid(ctx, lo, 256), 256, 0, ctx->stream>>>(W.T, W.key, lo, 2 * lo);
  PC_CHECK_LAUNCH();
  k_cs_wintree<<<1, WT_THREADS, 0, ctx->stream>>>(S, W, k);
  PC_CHECK_LAUNCH();
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  std::vector<long long> hg(k);
  unsigned long long ev[2];
  PC_CUDA(cudaMemcpyAsync(seeds, W.seeds, (size_t)k * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(hg.data(), W.gain_num, (size_t)k * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(ev, W.evals, 16, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms = ms;
  ctx->stats.select_evaluations = ev[0];
  ctx->stats.select_eval_rounds = ev[1];  // Win-Tree nodes explored
  ctx->stats.kernel_launches_select = depth + 2;
  long long run = 0;
  for (uint32_t i = 0; i < k; i++) {
    gain_num[i] = hg[i];
    run += hg[i];
    sigma_num[i] = run;
  }
}
