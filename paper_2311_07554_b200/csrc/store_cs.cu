// store_cs.cu — the COMPACT uncompressed store (H3-H7, H6u with its member
// index) and the greedy loop over it (H8-H12).  DESIGN.md §5 / §6.
//
// Why: in the paper's workloads a vertex is a singleton in most sketches (c4:
// 9.8 % of the (row, sketch) pairs are in a CC of >= 2 vertices, c2: 23 %).
// The dense vertex-major store (build.cu) writes, compresses and re-reads
// every pair; the compact store keeps an entry only for the pairs (v, r) where
// v has a live edge in sketch r (exactly the non-singleton pairs), laid out
// row-major, so every streaming pass moves ~1/10 of the bytes at c4.
//
// Layout (per build, B local sketch slots <= 256, MW = ceil(B/32) words):
//   rec[row][w]  = {first entry of the row + set bits of words < w, live-slot
//                   mask word w}: entry of (row, j) = pc_cs_pos (one 8-B read)
//   soff[row]    first entry of a row; sl[e] slot of entry e; ecrow[c] row of
//                entry 32c (lane-per-entry kernels find their row from it)
//   P[e]         union-find parent (an entry index: entries of one slot are in
//                vertex order, so the minimum entry of a CC is its minimum
//                vertex, R8), after compression: HIGH | |C| at the root entry,
//                the root entry elsewhere; bit 30 = covered during a selection
//   moff, memb   member index: the vertices of every CC of <= big_t vertices,
//                grouped by root entry (moff[root] = end of its group)
//
// Build: k_cs_mask (lane per CSR entry: live slots of the entry's edge, OR-ed
// into the row's mask) -> counts, scan -> k_cs_rec (prefixes, slot ids, chunk
// rows) -> P = HIGH|1 -> k_edges<CS> (build.cu: the unions, on entries) ->
// k_cs_compress (full compression, CC sizes) -> member offsets (scan) ->
// k_cs_gain (gain0 = sum_r |C_r(v)|, hot sums, member scatter).
//
// Selection (one persistent cooperative kernel, k steps): argmax over cached
// chunk maxima (Win-Tree layout), MarkSeed per slot,
// the members of each newly covered CC lose its size (from the member index,
// O(members) per step); CCs above big_t by the build's hot sums or one pass
// over the entries.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

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

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t csr_row(const uint64_t *off, const uint32_t *crow, uint64_t e) {
  uint32_t u = crow[e >> 5];
  while (e >= off[u + 1]) u++;
  return u;
}

__device__ __forceinline__ uint32_t entry_row(const uint32_t *soff, const uint32_t *ecrow,
                                              uint64_t e) {
  uint32_t r = ecrow[e >> 5];
  while (e >= soff[r + 1]) r++;
  return r;
}

// candidate slots [lo, hi) of an edge (R2 candidate enumeration, exact: the
// top clz(T-1) bits of hash(r) and hash(e) agree for every live slot; the
// same table lookup as k_edges so both passes see the same live sets)
__device__ __forceinline__ void cand_range(uint32_t he, uint64_t T, const uint16_t *tab,
                                           uint32_t B, bool decor, uint32_t &lo, uint32_t &hi) {
  lo = hi = 0;
  if (T == 0) return;
  if (decor) {
    hi = B;
    return;
  }
  const uint32_t w = __clz((uint32_t)(T - 1));
  if (w >= PACIM_TB) {
    const uint32_t p = he >> (32 - PACIM_TB);
    lo = tab[p];
    hi = tab[p + 1];
  } else if (w == 0) {
    hi = B;
  } else {
    const uint32_t p = (he >> (32 - w)) << (PACIM_TB - w);
    lo = tab[p];
    hi = tab[p + (1u << (PACIM_TB - w))];
  }
}

__device__ __forceinline__ uint32_t find_halve(uint32_t *P, uint32_t x) {
  for (;;) {
    const uint32_t p = __ldcg(P + x);
    if (p & PACIM_HIGH) return x;
    const uint32_t gp = __ldcg(P + p);
    if (gp & PACIM_HIGH) return p;
    atomicMin(P + x, gp);
    x = gp;
  }
}

__device__ __forceinline__ uint32_t find_ro(const uint32_t *P, uint32_t x) {
  for (;;) {
    const uint32_t p = __ldcg(P + x);
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

// ------------------------------------------------------------ k_cs_mask
// Lane per CSR entry (u, w) (balanced whatever the degrees): the live slots
// of edge {u, w} (P:3-4 / R3; per-edge T32 for WIC / Uniform, R4 / R19; R20)
// OR-ed into u's row mask.  Lanes of one row combine with one redux per word.
template <bool PERE, bool DECOR>
__global__ void __launch_bounds__(CS_THREADS) k_cs_mask(
    const uint64_t *__restrict__ off, const uint32_t *__restrict__ nbr,
    const uint32_t *__restrict__ crow, uint64_t nnz, const uint32_t *__restrict__ cid,
    const uint32_t *__restrict__ tcsr, uint32_t toff, uint64_t t32, uint64_t K,
    const uint32_t *__restrict__ g_shr, const uint16_t *__restrict__ g_tab,
    const uint64_t *__restrict__ hr64, uint32_t B, uint32_t MW, uint32_t *rec) {
  extern __shared__ uint32_t sm[];
  uint32_t *shr = sm;
  uint16_t *tab = reinterpret_cast<uint16_t *>(sm + B);
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) shr[i] = g_shr[i];
  for (uint32_t i = threadIdx.x; i <= (1u << PACIM_TB); i += blockDim.x) tab[i] = g_tab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(size_t)31; base < nnz;
       base += stride) {
    const uint64_t e = base + lane;
    uint32_t row = NONE;
    uint32_t bits[MAXW];
#pragma unroll
    for (int q = 0; q < (int)MAXW; q++) bits[q] = 0;
    if (e < nnz) {
      const uint32_t u = csr_row(off, crow, e), w = nbr[e];
      row = cid ? cid[u] : u;
      const uint64_t T = PERE ? (uint64_t)tcsr[e] + toff : t32;
      const uint64_t a = u < w ? u : w, b = u < w ? w : u;
      const uint64_t he64 = pc_mix64(((a << 32) | b) ^ K);
      const uint32_t he = (uint32_t)(he64 >> 32);
      uint32_t lo, hi;
      cand_range(he, T, tab, B, DECOR, lo, hi);
#pragma unroll
      for (int q = 0; q < (int)MAXW; q++) {
        const uint32_t j0 = max(lo, 32u * q), j1 = min(hi, 32u * q + 32);
        uint32_t x = 0;
        for (uint32_t j = j0; j < j1; j++) {
          const bool lv = DECOR ? (T >= (1ull << 32) || (pc_mix64(__ldg(hr64 + j) ^ he64) >> 32) < T)
                                : (uint64_t)(shr[j] ^ he) < T;
          x |= (uint32_t)lv << (j & 31);
        }
        bits[q] = x;
      }
    }
    const unsigned peers = __match_any_sync(FULL, row);
    const int leader = __ffs(peers) - 1;
#pragma unroll
    for (int q = 0; q < (int)MAXW; q++) {
      if ((uint32_t)q >= MW) break;
      if (!__any_sync(FULL, bits[q])) continue;
      const uint32_t x = __reduce_or_sync(peers, bits[q]);
      if (lane == leader && x && row != NONE) atomicOr(rec + ((size_t)row * MW + q) * 2 + 1, x);
    }
  }
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

// thread per row: word prefixes, soff, slot ids of the row's entries, and
// the chunk table (row of entry 32 c for every chunk starting in the row)
__global__ void k_cs_rec(uint2 *rec, uint32_t nr, uint32_t MW, const uint64_t *pos,
                         uint32_t *soff, uint8_t *sl, uint32_t *ecrow) {
  for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr;
       r += (size_t)gridDim.x * blockDim.x) {
    const uint32_t base = (uint32_t)pos[r];
    uint32_t at = base;
    for (uint32_t q = 0; q < MW; q++) {
      uint2 x = rec[r * MW + q];
      x.x = at;
      rec[r * MW + q] = x;
      for (uint32_t t = x.y; t; t &= t - 1) sl[at++] = (uint8_t)(q * 32 + __ffs(t) - 1);
    }
    soff[r] = base;
    if (r + 1 == nr) soff[nr] = at;
    for (uint32_t c = (base + 31) >> 5; (c << 5) < at; c++) ecrow[c] = (uint32_t)r;
  }
}

__global__ void k_cs_fill(uint32_t *a, uint64_t N, uint32_t x) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    a[i] = x;
}

// the hub row's root entry per slot (the hot, typically giant, CCs), NONE if
// the hub is a singleton there
__global__ void k_cs_hot(const uint2 *rec, uint32_t MW, const uint32_t *P, uint32_t hub_row,
                         uint32_t nr, uint32_t B, uint32_t *hot) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x) {
    uint32_t h = NONE;
    if (hub_row < nr && ((rec[(size_t)hub_row * MW + (j >> 5)].y >> (j & 31)) & 1u))
      h = find_ro(P, pc_cs_pos(rec, MW, hub_row, j));
    hot[j] = h;
  }
}

// full compression (H4) and CC sizes into the root entries (H5): lane per
// entry; members of a slot's hot CC counted per block in shared memory.
// ctr[1] += non-root entries.
__global__ void __launch_bounds__(CS_THREADS) k_cs_compress(uint32_t *P, uint64_t total,
                                                            const uint8_t *sl, uint32_t B,
                                                            const uint32_t *hot,
                                                            unsigned long long *ctr) {
  __shared__ uint32_t hroot[256], hcnt[256];
  for (uint32_t j = threadIdx.x; j < 256; j += blockDim.x) {
    hroot[j] = j < B ? hot[j] : NONE;
    hcnt[j] = 0;
  }
  __syncthreads();
  unsigned long long nnr = 0;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const uint32_t s = __ldcg(P + e);
    if (s & PACIM_HIGH) continue;
    nnr++;
    const uint32_t j = sl[e];
    uint32_t root = s;
    if (s != hroot[j]) {
      root = find_halve(P, s);
      if (root != s) atomicMin(P + e, root);
    }
    if (root == hroot[j])
      atomicAdd(hcnt + j, 1u);
    else
      atomicAdd(P + root, 1u);
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < B; j += blockDim.x)
    if (hcnt[j]) atomicAdd(P + hroot[j], hcnt[j]);
  add_count(ctr + 1, nnr);
}

__global__ void k_cs_hot_sizes(const uint32_t *P, const uint32_t *hot, uint32_t B,
                               uint32_t *hot_size) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x)
    hot_size[j] = hot[j] != NONE ? (P[hot[j]] & PACIM_LOW) : 0u;
}

// member-index sizes: |C| at a root entry of a CC of <= big_t vertices, else 0
struct MembSize {
  const uint32_t *P;
  uint64_t total;
  uint32_t big_t;
  __host__ __device__ __forceinline__ uint32_t operator()(uint64_t e) const {
    if (e >= total) return 0;
    const uint32_t s = P[e];
    return ((s & PACIM_HIGH) && (s & PACIM_LOW) <= big_t) ? (s & PACIM_LOW) : 0u;
  }
};

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

// lane per entry: gain0[v] += |C_j(v)| (H7), hotsum[v] += |hot C_j| when v is
// in slot j's giant hot CC, and the member scatter (H6u).  ctr[0] += roots.
template <bool HOT>
__global__ void __launch_bounds__(CS_THREADS) k_cs_gain(
    const uint32_t *__restrict__ P, uint64_t total, const uint8_t *__restrict__ sl,
    const uint32_t *__restrict__ soff, const uint32_t *__restrict__ ecrow,
    const uint32_t *__restrict__ rmap, uint32_t B, const uint32_t *hot, const uint32_t *hot_size,
    uint32_t big_t, uint32_t *moff, uint32_t *memb, int64_t *gain0, int64_t *hotsum,
    unsigned long long *ctr) {
  __shared__ uint32_t hroot[256], hsz[256];
  if (HOT) {
    for (uint32_t j = threadIdx.x; j < 256; j += blockDim.x) {
      const bool giant = j < B && hot_size[j] > big_t;
      hroot[j] = giant ? hot[j] : NONE;
      hsz[j] = giant ? hot_size[j] : 0u;
    }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  unsigned long long nroot = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(size_t)31; base < total;
       base += stride) {
    const size_t e = base + lane;
    uint32_t row = NONE, size = 0, hs = 0, v = 0;
    if (e < total) {
      row = entry_row(soff, ecrow, e);
      v = rmap ? rmap[row] : row;
      const uint32_t s = P[e];
      const uint32_t root = (s & PACIM_HIGH) ? (uint32_t)e : s;
      const uint32_t rv = (s & PACIM_HIGH) ? s : __ldg(P + s);
      size = rv & PACIM_LOW;
      nroot += (s & PACIM_HIGH) != 0;
      if (HOT) {
        const uint32_t j = sl[e];
        if (root == hroot[j]) hs = hsz[j];
      }
      if (size <= big_t) memb[atomicAdd(moff + root, 1u)] = v;
    }
    const unsigned peers = __match_any_sync(FULL, row);
    const unsigned long long g = peer_sum(peers, size);
    const unsigned long long h = HOT ? peer_sum(peers, hs) : 0ull;
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
enum { CD_STEPS = 0, CD_DENSE, CD_HOT, CD_UPD, CD_WORDS = 8 };

struct CSel {
  const uint2 *rec;
  uint32_t MW;
  uint32_t *P;
  const uint32_t *moff, *memb;
  const uint8_t *sl;
  const uint32_t *soff, *ecrow, *rmap, *cid;
  uint32_t nr, B, nv;
  uint64_t total;
  uint32_t big_t;
  long long *target;       // gains (single rank) or the delta vector (multi-rank)
  uint32_t *cov_root, *cov_delta;  // [B] big CCs covered this step
  int *dense;              // [2] by step parity
  unsigned long long *cov_list, *cov_cnt;
  unsigned long long cov_cap;
  const int64_t *hotsum;
  const uint32_t *hot_root, *hot_size;
  Best *cmax;
  uint32_t *cdirty, *dlist, *dcnt;
  uint32_t csh, nchunks, par;
  int track;
  DeltaList dlst;
  unsigned long long *diag;
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

// MarkSeed in slot j for the seed row srow (one thread):
// returns delta_j; *mroot / *msize: a newly covered CC with a member list
__device__ __forceinline__ uint32_t cs_cover(const CSel &S, uint32_t srow, uint32_t j,
                                             uint32_t *mroot) {
  *mroot = NONE;
  S.cov_root[j] = NONE;
  if (srow == NONE || !((S.rec[(size_t)srow * S.MW + (j >> 5)].y >> (j & 31)) & 1u))
    return 1;  // {s}: a singleton, uncovered while s is not a seed
  const uint32_t e = pc_cs_pos(S.rec, S.MW, srow, j);
  const uint32_t x0 = __ldcg(S.P + e);
  const uint32_t root = (x0 & PACIM_HIGH) ? e : x0;
  const uint32_t x = atomicOr(S.P + root, COV);
  if (x & COV) return 0;  // covered by an earlier seed
  const uint32_t delta = x & SIZE;
  const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
  if (at < S.cov_cap) S.cov_list[at] = root;
  if (delta > S.big_t) {
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

// the covered big CCs of this step: exactly the hub's giant CCs -> hot sums
// (one vector pass); block-collective, uniform result
__device__ bool dense_hot(const CSel &S, uint32_t s, size_t tid, size_t nth) {
  int ok = S.hotsum != nullptr;
  for (uint32_t j = threadIdx.x; j < S.B && ok; j += blockDim.x) {
    const uint32_t cr = __ldcg(S.cov_root + j);
    const bool big = S.hot_size[j] > S.big_t;
    if (big != (cr != NONE) || (big && cr != S.hot_root[j])) ok = 0;
  }
  if (!__syncthreads_and(ok)) return false;
  for (size_t v = tid; v < S.nv; v += nth) {
    const long long h = S.hotsum[v];
    if (h && v != s) sub_gain(S, (uint32_t)v, h);
  }
  return true;
}

// dense pass: lane per entry; an entry of slot j whose root is slot j's
// covered big CC loses cov_delta[j] at its vertex
__device__ void dense_pass(const CSel &S, uint32_t s, const uint32_t *croot, const uint32_t *cdel,
                           size_t tid, size_t nth) {
  for (size_t e = tid; e < S.total; e += nth) {
    const uint32_t j = S.sl[e];
    const uint32_t cr = croot[j];
    if (cr == NONE) continue;
    const uint32_t x = __ldcg(S.P + e);
    const uint32_t root = (x & PACIM_HIGH) ? (uint32_t)e : x;
    if (root != cr) continue;
    const uint32_t row = entry_row(S.soff, S.ecrow, e);
    const uint32_t v = S.rmap ? S.rmap[row] : row;
    if (v != s) sub_gain(S, v, cdel[j]);
  }
}

// Step (parity par): A argmax -> B MarkSeed + member updates -> (dense) ->
// E refresh of the chunk maxima; grid barriers after B, the dense pass and E.
__global__ void __launch_bounds__(SEL_THREADS, 1) k_cs_select(CSel S0, CSelOut O, uint32_t par0) {
  cg::grid_group grid = cg::this_grid();
  CSel S = S0;
  __shared__ Best sh[33];
  __shared__ uint32_t croot[256], cdel[256];
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
    if (tid == 0) {
      O.seeds[step] = s;
      O.arg_gain[step] = sg;
      if (O.given == NONE) {
        S.target[s] = -1;  // s leaves the candidate set (R6)
        mark_dirty(S, s >> S.csh);
      }
    }
    // ---- B: MarkSeed per slot; members of the newly covered CCs lose |C|
    {
      unsigned long long dsum = 0, upd = 0;
      for (size_t j = gwarp; j < S.B; j += nwarps) {
        uint32_t d = 0, mr = NONE;
        if (lane == 0) d = cs_cover(S, srow, (uint32_t)j, &mr);
        d = __shfl_sync(FULL, d, 0);
        mr = __shfl_sync(FULL, mr, 0);
        dsum += d;
        if (mr != NONE && d > 1) {
          const uint32_t end = __ldg(S.moff + mr);
          for (uint32_t t = end - d + lane; t < end; t += 32) {
            const uint32_t v = __ldg(S.memb + t);
            if (v != s) sub_gain(S, v, d);
          }
          upd += d;
        }
      }
      if (lane == 0) {
        if (dsum) atomicAdd(reinterpret_cast<unsigned long long *>(&O.gain_num[step]), dsum);
        if (upd) atomicAdd(S.diag + CD_UPD, upd);
      }
    }
    grid.sync();
    // ---- dense: CCs above big_t covered this step
    if (__ldcg(S.dense + S.par)) {
      for (uint32_t j = threadIdx.x; j < 256; j += blockDim.x) {
        croot[j] = j < S.B ? __ldcg(S.cov_root + j) : NONE;
        cdel[j] = j < S.B ? __ldcg(S.cov_delta + j) : 0u;
      }
      __syncthreads();
      if (dense_hot(S, s, tid, nth)) {
        if (tid == 0) atomicAdd(S.diag + CD_HOT, 1ull);
      } else {
        dense_pass(S, s, croot, cdel, tid, nth);
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

__global__ void k_cs_uncover(uint32_t *P, const unsigned long long *list, unsigned long long cnt) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (size_t)gridDim.x * blockDim.x)
    atomicAnd(P + list[i], ~COV);
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
        const uint32_t x = __ldcg(S.P + r.x + __popc(r.y & ((1u << (j & 31)) - 1u)));
        const uint32_t rv = (x & PACIM_HIGH) ? x : __ldcg(S.P + x);
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
    const uint32_t x = S.P[e];
    const uint32_t root = (x & PACIM_HIGH) ? e : x;
    if (!(atomicOr(S.P + root, COV) & COV)) {
      const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
      if (at < S.cov_cap) S.cov_list[at] = root;
    }
  }
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
        const uint32_t x = S.P[e];
        const uint32_t root = (x & PACIM_HIGH) ? e : x;
        // row of the root entry: the last row whose first entry is <= root
        uint32_t lo = 0, hi = S.nr;  // soff[lo] <= root < soff[hi]
        while (hi - lo > 1) {
          const uint32_t mid = lo + (hi - lo) / 2;
          if (S.soff[mid] <= root) lo = mid;
          else hi = mid;
        }
        lab = S.rmap ? S.rmap[lo] : lo;
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

static uint32_t cs_big_t(pacim_ctx *ctx) {
  const char *e = getenv("PACIM_BIG_T");
  return (uint32_t)(e ? std::max(1LL, atoll(e)) : std::max<uint64_t>(65536, ctx->nr / 8));
}

void pc_cs_free(pacim_ctx *ctx) {
  for (DevBuf *d : {&ctx->cs_rec, &ctx->cs_soff, &ctx->cs_sl, &ctx->cs_ecrow, &ctx->cs_P,
                    &ctx->cs_moff, &ctx->cs_memb, &ctx->cs_diag})
    pc_free(ctx, *d);
  ctx->cs = false;
}

// The compact build.  Returns false (nothing changed but the scratch) when the
// store would not be compact: more than half of the (row, slot) pairs are
// non-singletons (c3: p = 1/2 on a grid), or 2^31 entries or more.
bool pc_cs_build(pacim_ctx *ctx) {
  const uint32_t nr = ctx->nr, B = ctx->R_local, n = ctx->n;
  if (const char *e = getenv("PACIM_STORE")) {
    if (std::string(e) == "dense") return false;
  } else if (getenv("PACIM_L2_BUDGET")) {
    return false;  // the slot-window layout is a dense-store experiment
  }
  if (B > 256 || nr == 0 || ctx->compressed) return false;
  const uint32_t MW = (B + 31) / 32;
  pc_slot_table(ctx);
  pc_ensure(ctx, ctx->counters, 64 * sizeof(uint64_t));
  unsigned long long *ctr = ctx->counters.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(ctr, 0, 64 * sizeof(uint64_t), ctx->stream));
  ctx->launches = 0;
  cudaEvent_t ev[8];
  for (auto &e : ev) PC_CUDA(cudaEventCreate(&e));
  PC_CUDA(cudaEventRecord(ev[0], ctx->stream));
  // ---- masks (the rec array, .y words)
  pc_ensure(ctx, ctx->cs_rec, (size_t)nr * MW * 8);
  PC_CUDA(cudaMemsetAsync(ctx->cs_rec.p, 0, (size_t)nr * MW * 8, ctx->stream));
  const uint64_t nnz = 2 * ctx->m;
  if (nnz) {
    const size_t smem = B * 4 + ((1u << PACIM_TB) + 1) * 2;
    const bool pe = ctx->pmodel != PACIM_P_CONST;
    auto kern = pe ? (ctx->hash_rule ? k_cs_mask<true, true> : k_cs_mask<true, false>)
                   : (ctx->hash_rule ? k_cs_mask<false, true> : k_cs_mask<false, false>);
    PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<pc_grid(ctx, (nnz + 31) / 32 * 32, CS_THREADS, 8), CS_THREADS, smem, ctx->stream>>>(
        ctx->off.as<uint64_t>(), ctx->nbr.as<uint32_t>(), ctx->crow.as<uint32_t>(), nnz,
        ctx->lean ? nullptr : ctx->cid.as<uint32_t>(), pe ? ctx->tcsr.as<uint32_t>() : nullptr,
        ctx->toff(), ctx->t32, ctx->K, ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(),
        ctx->d_hr64.as<uint64_t>(), B, MW, ctx->cs_rec.as<uint32_t>());
    PC_CHECK_LAUNCH();
    ctx->launches++;
  }
  // ---- counts -> entry offsets
  TmpBuf cnt(ctx);
  pc_ensure(ctx, cnt, 2 * ((size_t)nr + 1) * 8);
  uint64_t *c64 = cnt.as<uint64_t>(), *pos = c64 + nr + 1;
  k_cs_count<<<pc_grid(ctx, nr + 1, 256), 256, 0, ctx->stream>>>(ctx->cs_rec.as<uint2>(), nr, MW, c64);
  PC_CHECK_LAUNCH();
  pc_exclusive_scan_u64(ctx, c64, pos, (size_t)nr + 1);
  uint64_t total = 0;
  PC_CUDA(cudaMemcpyAsync(&total, pos + nr, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->launches += 2;
  if (total >= (1ull << 31) || 2 * total > (uint64_t)nr * B) {
    for (auto &e : ev) cudaEventDestroy(e);
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
  pc_ensure(ctx, ctx->cs_sl, T1);
  pc_ensure(ctx, ctx->cs_ecrow, (T1 / 32 + 2) * 4);
  pc_ensure(ctx, ctx->cs_P, T1 * 4);
  pc_ensure(ctx, ctx->cs_moff, (T1 + 1) * 4);
  k_cs_rec<<<pc_grid(ctx, nr, 256), 256, 0, ctx->stream>>>(
      ctx->cs_rec.as<uint2>(), nr, MW, pos, ctx->cs_soff.as<uint32_t>(), ctx->cs_sl.as<uint8_t>(),
      ctx->cs_ecrow.as<uint32_t>());
  PC_CHECK_LAUNCH();
  uint32_t *P = ctx->cs_P.as<uint32_t>();
  k_cs_fill<<<pc_grid(ctx, total, 256), 256, 0, ctx->stream>>>(P, total, ROOT1);
  PC_CHECK_LAUNCH();
  ctx->launches += 2;
  PC_CUDA(cudaEventRecord(ev[1], ctx->stream));
  // ---- unions (H2, H3)
  pc_cs_edges(ctx, P, ctx->cs_rec.as<uint2>(), MW, ctr);
  PC_CUDA(cudaEventRecord(ev[2], ctx->stream));
  // ---- compression + sizes (H4, H5)
  pc_ensure(ctx, ctx->d_hot, 2 * (size_t)B * 4);
  uint32_t *hot = ctx->d_hot.as<uint32_t>();
  k_cs_hot<<<(B + 255) / 256, 256, 0, ctx->stream>>>(ctx->cs_rec.as<uint2>(), MW, P, ctx->hub_row,
                                                     nr, B, hot);
  PC_CHECK_LAUNCH();
  k_cs_compress<<<pc_grid(ctx, total, CS_THREADS, 8), CS_THREADS, 0, ctx->stream>>>(
      P, total, ctx->cs_sl.as<uint8_t>(), B, hot, ctr);
  PC_CHECK_LAUNCH();
  pc_ensure(ctx, ctx->d_hot_size, (size_t)B * 4);
  k_cs_hot_sizes<<<(B + 255) / 256, 256, 0, ctx->stream>>>(P, hot, B, ctx->d_hot_size.as<uint32_t>());
  PC_CHECK_LAUNCH();
  ctx->launches += 3;
  PC_CUDA(cudaEventRecord(ev[3], ctx->stream));
  // ---- member offsets: exclusive scan of the member-list sizes (H6u)
  const uint32_t big_t = cs_big_t(ctx);
  ctx->cs_big_t = big_t;
  {
    cub::CountingInputIterator<uint64_t> it(0);
    cub::TransformInputIterator<uint32_t, MembSize, cub::CountingInputIterator<uint64_t>> in(
        it, MembSize{P, total, big_t});
    size_t tb = 0;
    PC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, ctx->cs_moff.as<uint32_t>(),
                                          (int64_t)total + 1, ctx->stream));
    TmpBuf tmp(ctx);
    pc_ensure(ctx, tmp, std::max<size_t>(tb, 16));
    PC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, ctx->cs_moff.as<uint32_t>(),
                                          (int64_t)total + 1, ctx->stream));
    uint32_t nm = 0;
    PC_CUDA(cudaMemcpyAsync(&nm, ctx->cs_moff.as<uint32_t>() + total, 4, cudaMemcpyDeviceToHost,
                            ctx->stream));
    ctx->hot_size.resize(B);
    PC_CUDA(cudaMemcpyAsync(ctx->hot_size.data(), ctx->d_hot_size.p, (size_t)B * 4,
                            cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->cs_nmemb = nm;
    ctx->launches++;
  }
  pc_ensure(ctx, ctx->cs_memb, std::max<size_t>(ctx->cs_nmemb, 1) * 4);
  PC_CUDA(cudaEventRecord(ev[4], ctx->stream));
  // ---- gain0 (H7), hot sums, member scatter
  bool any = false;
  for (uint32_t j = 0; j < B; j++) any |= ctx->hot_size[j] > big_t;
  ctx->hot_any = any;
  ctx->hot_big_t = big_t;
  if (any) pc_ensure(ctx, ctx->hotsum, (size_t)n * 8);
  pc_ensure(ctx, ctx->gain0, (size_t)n * 8);
  k_cs_gain_init<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(
      ctx->lean ? nullptr : ctx->cid.as<uint32_t>(), ctx->cs_soff.as<uint32_t>(), n, B,
      ctx->gain0.as<int64_t>(), any ? ctx->hotsum.as<int64_t>() : nullptr);
  PC_CHECK_LAUNCH();
  {
    auto kern = any ? k_cs_gain<true> : k_cs_gain<false>;
    kern<<<pc_grid(ctx, total, CS_THREADS, 8), CS_THREADS, 0, ctx->stream>>>(
        P, total, ctx->cs_sl.as<uint8_t>(), ctx->cs_soff.as<uint32_t>(), ctx->cs_ecrow.as<uint32_t>(),
        ctx->lean ? nullptr : ctx->rmap.as<uint32_t>(), B, hot, ctx->d_hot_size.as<uint32_t>(), big_t,
        ctx->cs_moff.as<uint32_t>(), ctx->cs_memb.as<uint32_t>(), ctx->gain0.as<int64_t>(),
        any ? ctx->hotsum.as<int64_t>() : nullptr, ctr);
    PC_CHECK_LAUNCH();
  }
  ctx->launches += 2;
  PC_CUDA(cudaEventRecord(ev[5], ctx->stream));
  unsigned long long h[6];
  PC_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->cs = true;
  ctx->ncomp = h[0];
  ctx->nnonsingle = total;
  ctx->nmember = ctx->cs_nmemb;
  ctx->stats.live_pairs = h[4];
  PC_REQUIRE(h[0] + h[1] == total, PACIM_ECHECK, "compact store: roots + non-roots != entries");
  ctx->stats.t_init_ms = ev_ms(ev[0], ev[1]);      // masks, offsets, P = HIGH | 1
  ctx->stats.t_edges_ms = ev_ms(ev[1], ev[2]);
  ctx->stats.t_compress_ms = ev_ms(ev[2], ev[3]);
  ctx->stats.t_compact_ms = ev_ms(ev[3], ev[4]);   // member offsets
  ctx->stats.t_gain_ms = ev_ms(ev[4], ev[5]);
  ctx->stats.t_centers_ms = 0;
  ctx->stats.t_build_ms = ev_ms(ev[0], ev[5]);
  ctx->stats.kernel_launches_build = ctx->launches;
  for (auto &e : ev) cudaEventDestroy(e);
  ctx->sel_list_valid = false;
  return true;
}

// ------------------------------------------------------------ selection
static CSel make_csel(pacim_ctx *ctx, long long *target) {
  const uint32_t B = ctx->R_local, n = ctx->n;
  CSel S;
  S.rec = ctx->cs_rec.as<uint2>();
  S.MW = ctx->cs_MW;
  S.P = ctx->cs_P.as<uint32_t>();
  S.moff = ctx->cs_moff.as<uint32_t>();
  S.memb = ctx->cs_memb.as<uint32_t>();
  S.sl = ctx->cs_sl.as<uint8_t>();
  S.soff = ctx->cs_soff.as<uint32_t>();
  S.ecrow = ctx->cs_ecrow.as<uint32_t>();
  S.rmap = ctx->lean ? nullptr : ctx->rmap.as<uint32_t>();
  S.cid = ctx->lean ? nullptr : ctx->cid.as<uint32_t>();
  S.nr = ctx->nr;
  S.B = B;
  S.nv = n;
  S.total = ctx->cs_total;
  S.big_t = ctx->cs_big_t;
  S.target = target;
  S.hotsum = ctx->hot_any ? ctx->hotsum.as<int64_t>() : nullptr;
  S.hot_root = ctx->d_hot.as<uint32_t>();
  S.hot_size = ctx->d_hot_size.as<uint32_t>();
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
  return S;
}

static void cs_uncover(pacim_ctx *ctx, const CSel &S) {
  unsigned long long cnt = 0;
  if (ctx->sel_list_valid) {
    PC_CUDA(cudaMemcpyAsync(&cnt, S.cov_cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  PC_REQUIRE(cnt <= S.cov_cap, PACIM_ECHECK, "covered-CC list overflowed");
  if (cnt) k_cs_uncover<<<pc_grid(ctx, cnt, 256), 256, 0, ctx->stream>>>(S.P, S.cov_list, cnt);
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
