// select.cu — Step 2 of Alg. 1: the device-resident greedy loop
// over the uncompressed store (H8-H12).
//
// One persistent cooperative kernel runs all k steps:
//   A  NextSeed: argmax of (gain desc, id asc) over v (R5, R6) through a
//      two-level tournament array (the Win-Tree layout of P:2658-2664,
//      flattened): per-chunk maxima, recomputed only for chunks whose gains
//      changed, reduced by every block.
//   B  MarkSeed: one warp per sketch slot j reads the seed's CC
//      from its root slot (HIGH | size): delta_j = size unless the CC is
//      already covered (bit 30), then marks it covered.
//   C  incremental gain update (R17): the members of every newly covered CC
//      lose delta_j.  Small CCs (<= big_t vertices) are enumerated by ONE
//      breadth-first search over the live edges shared by all slots: a
//      frontier vertex carries the set of slots it was reached in, its
//      adjacency is read once and each edge's hash is computed once, and only
//      the candidate slots of the edge (the same bucket table as the build)
//      are tested — hubs are expanded once, not once per sketch.  Big CCs are
//      handled by one dense pass over the store (slot == covered root).
// The covered bits are cleared before the next selection (the list of
// covered root slots is kept).  gain_num[i] = sum_j delta_j; the host checks
// it against the argmax gain.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "pacim_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int SEL_THREADS = 512;
constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t COV = 0x40000000u;   // covered bit of a root slot
constexpr uint32_t SIZE = 0x3FFFFFFFu;  // CC size bits of a root slot
constexpr uint32_t MAX_CHUNKS = 4096;   // argmax cache: chunk maxima per step
constexpr uint32_t BIG_DEFAULT = 4096;  // CCs larger than this: dense pass

struct Best {
  long long g;
  uint32_t v;
};

__device__ __forceinline__ bool better(long long g1, uint32_t v1, long long g2, uint32_t v2) {
  return g1 > g2 || (g1 == g2 && v1 < v2);
}

__device__ __forceinline__ Best warp_best(Best b) {
  for (int d = 16; d; d >>= 1) {
    long long g = __shfl_xor_sync(0xffffffffu, b.g, d);
    uint32_t v = __shfl_xor_sync(0xffffffffu, b.v, d);
    if (better(g, v, b.g, b.v)) {
      b.g = g;
      b.v = v;
    }
  }
  return b;
}

// block-wide (g desc, v asc) reduction; result valid in all threads
__device__ Best block_best(Best b, Best *sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  b = warp_best(b);
  __syncthreads();
  if (lane == 0) sh[wid] = b;
  __syncthreads();
  if (wid == 0) {
    Best x = lane < (int)(blockDim.x >> 5) ? sh[lane] : Best{LLONG_MIN, 0xFFFFFFFFu};
    x = warp_best(x);
    if (lane == 0) sh[32] = x;
  }
  __syncthreads();
  return sh[32];
}

struct Sel {
  // graph (BFS over live edges)
  const uint64_t *off;
  const uint32_t *nbr;
  uint64_t K, t32;
  const uint32_t *tcsr;  // WIC: T32 - 1 per CSR entry
  int wic;
  const uint32_t *g_shr;   // hi32(hash(r)) of slot j (sorted)
  const uint16_t *g_tab;   // candidate bucket table of the sorted slots
  // store
  uint32_t *L;
  uint32_t nr, B, BW, nv;  // rows, slots, bitmap words per row, vertices
  const uint32_t *cid, *rmap;
  // per step
  long long *target;       // gain vector (single rank) or delta vector (multi-rank)
  uint32_t *dl;            // B: delta_j of a CC to enumerate by BFS (0: none)
  uint32_t *cov_root;      // B: root row of a big CC covered in slot j, or NONE
  uint32_t *cov_delta;     // B
  int *dense;              // [2] by step parity: a big CC was covered
  unsigned long long *cov_list, *cov_cnt;  // covered root-slot indices (restored later)
  unsigned long long cov_cap;
  uint32_t big_t;
  // multi-slot BFS
  uint32_t *vis;           // rows x BW: slot bits of visited (row, slot)
  uint32_t *fmask;         // [2][rows x BW]: slots a frontier row was newly reached in
  uint32_t *inl;           // [2][rows]: row is in the frontier list
  uint32_t *flist;         // [2][rows] light frontier rows
  uint32_t *hlist;         // [2][rows] heavy frontier rows
  uint32_t *fcnt;          // [0..2] light / [4..6] heavy list sizes by level % 3,
                           // [8 + par] touched count of a step of parity par
  uint32_t *touched;       // [2][rows]: rows visited in a step of parity par (each once)
  uint32_t *tflag;         // [rows]: row is in a touched list
  uint64_t heavy_deg;      // rows of higher degree are expanded by the whole grid
  // argmax cache (single rank): marks of step i go to buffer i & 1, consumed
  // by step i + 1 which resets buffer i - 1 (no reset races with a mark)
  Best *cmax;
  uint32_t *cdirty, *dlist, *dcnt;  // dlist[2][nchunks], dcnt[2]
  int *alldirty;                    // [2]
  uint32_t par, csh, nchunks;
  int track;
};

__device__ __forceinline__ void mark_dirty(const Sel &S, uint32_t u) {
  const uint32_t c = u >> S.csh;
  if (atomicExch(S.cdirty + c, 1u) == 0u)
    S.dlist[(size_t)S.par * S.nchunks + atomicAdd(S.dcnt + S.par, 1u)] = c;
}

// remember a row whose visited bits must be cleared before the next step
__device__ __forceinline__ void touch(const Sel &S, uint32_t row) {
  if (atomicExch(S.tflag + row, 1u) == 0u)
    S.touched[(size_t)S.par * S.nr + atomicAdd(S.fcnt + 8 + S.par, 1u)] = row;
}

__device__ __forceinline__ void sub_gain(const Sel &S, uint32_t u, long long d) {
  atomicAdd((unsigned long long *)&S.target[u], (unsigned long long)(-d));
  if (S.track) mark_dirty(S, u);
}

// Phase B for slot j (one thread): MarkSeed and classification.
__device__ __forceinline__ uint32_t cover_slot(const Sel &S, uint32_t srow, uint32_t j) {
  uint32_t delta = 1;
  S.dl[j] = 0;
  S.cov_root[j] = NONE;
  if (srow == NONE) return delta;  // isolated seed: singleton in every sketch
  const uint32_t sl = S.L[(size_t)srow * S.B + j];
  if (sl == srow) return delta;    // singleton {s}
  const uint32_t root = (sl & PACIM_HIGH) ? srow : sl;
  uint32_t *rs = S.L + (size_t)root * S.B + j;
  const uint32_t x = atomicOr(rs, COV);  // covered from now on
  if (x & COV) return 0;                 // covered by an earlier seed
  delta = x & SIZE;
  const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
  if (at < S.cov_cap) S.cov_list[at] = (size_t)root * S.B + j;
  if (delta > S.big_t) {
    S.cov_root[j] = root;
    S.cov_delta[j] = delta;
    S.dense[S.par] = 1;
  } else {
    S.dl[j] = delta;
    atomicOr(S.vis + (size_t)srow * S.BW + (j >> 5), 1u << (j & 31));
    touch(S, srow);
  }
  return delta;
}

// hand slot j of the seed's small CC to the grid-wide multi-slot BFS
__device__ __forceinline__ void defer_slot(const Sel &S, uint32_t s, uint32_t srow, uint32_t j) {
  atomicOr(S.fmask + (size_t)srow * S.BW + (j >> 5), 1u << (j & 31));
  if (atomicExch(S.inl + srow, 1u) == 0u) {  // level-0 list (parity 0)
    if (S.off[s + 1] - S.off[s] > S.heavy_deg)
      S.hlist[atomicAdd(S.fcnt + 4, 1u)] = srow;
    else
      S.flist[atomicAdd(S.fcnt + 0, 1u)] = srow;
  }
}

// Warp-local BFS of the seed's CC in slot j (<= QCAP vertices) with a
// shared-memory queue and visited set; applies the gain updates.  Returns
// false, before updating anything, if it meets a vertex of degree > WARP_DEG
// (the grid-wide BFS then takes the slot and reads that adjacency once for
// all slots).
constexpr uint32_t QCAP = 512;
constexpr uint32_t HCAP = 1024;
constexpr uint64_t WARP_DEG = 1024;
constexpr uint32_t WARP_WORDS = QCAP + HCAP + 1;

// shared-memory words of the slot tables (shr[B] + tab[2^TB + 1] u16), 16-B aligned
__host__ __device__ __forceinline__ uint32_t table_words(uint32_t B) {
  return (((uint32_t)B * 4 + ((1u << PACIM_TB) + 1) * 2 + 15) & ~15u) / 4;
}

__device__ bool warp_bfs(const Sel &S, uint32_t s, uint32_t j, uint32_t delta, uint32_t *q,
                         uint32_t *hs, uint32_t *tail, const uint32_t *shr) {
  const int lane = threadIdx.x & 31;
  const uint32_t hr = shr[j];
  for (uint32_t i = lane; i < HCAP; i += 32) hs[i] = NONE;
  __syncwarp();
  if (lane == 0) {
    q[0] = s;
    hs[(s * 2654435761u) & (HCAP - 1)] = s;
    *tail = 1;
  }
  __syncwarp();
  for (uint32_t head = 0; head < *tail;) {
    const uint32_t x = q[head++];
    const uint64_t e0 = S.off[x], e1 = S.off[x + 1];
    if (e1 - e0 > WARP_DEG) return false;  // uniform: same x in every lane
    for (uint64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t w = S.nbr[e];
      const uint64_t a = x < w ? x : w, b = x < w ? w : x;
      const uint32_t he = (uint32_t)(pc_mix64(((a << 32) | b) ^ S.K) >> 32);
      const uint64_t T = S.wic ? (uint64_t)S.tcsr[e] + 1 : S.t32;  // R4
      if ((uint64_t)(hr ^ he) >= T) continue;                        // R3
      uint32_t h = (w * 2654435761u) & (HCAP - 1);
      for (;;) {
        const uint32_t old = atomicCAS(hs + h, NONE, w);
        if (old == NONE) {
          const uint32_t pos = atomicAdd(tail, 1u);
          if (pos < QCAP) q[pos] = w;
          break;
        }
        if (old == w) break;
        h = (h + 1) & (HCAP - 1);
      }
    }
    __syncwarp();
    if (*tail > QCAP) return false;  // cannot happen for a CC of delta <= QCAP
  }
  const uint32_t cnt = *tail;
  for (uint32_t i = lane; i < cnt; i += 32) {
    const uint32_t u = q[i];
    if (u != s) sub_gain(S, u, delta);
  }
  __syncwarp();
  return true;
}

// One BFS level: every frontier row is expanded by one block; its adjacency
// is read once, each edge hashed once, and only the edge's candidate slots
// that the row was newly reached in are tested (R3 live test).
// Frontier lists alternate by level parity; their sizes live in fcnt[lvl % 3]
// so that the counter of level + 2 can be reset during level (nobody reads
// or appends to it then).
// Expand frontier row u (vertex x) over adjacency entries [e0, e1) taken with
// stride `stride` from offset `first` (a block or the whole grid).
__device__ void expand_row(const Sel &S, uint32_t lvl, uint32_t u, const uint32_t *shr,
                           const uint16_t *tab, uint32_t s, uint64_t first, uint64_t stride) {
  const uint32_t cur = lvl & 1, nxt = cur ^ 1;
  uint32_t *ncnt = S.fcnt + (lvl + 1) % 3;      // light list of level + 1
  uint32_t *nhcnt = S.fcnt + 4 + (lvl + 1) % 3; // heavy list of level + 1
  const uint32_t *M = S.fmask + ((size_t)cur * S.nr + u) * S.BW;
  uint32_t *fm_nxt = S.fmask + (size_t)nxt * S.nr * S.BW;
  const uint32_t x = S.rmap[u];
  const uint64_t e1 = S.off[x + 1];
  {
    for (uint64_t e = S.off[x] + first; e < e1; e += stride) {
      const uint32_t w = S.nbr[e];
      const uint64_t a = x < w ? x : w, b = x < w ? w : x;
      const uint32_t he = (uint32_t)(pc_mix64(((a << 32) | b) ^ S.K) >> 32);
      const uint64_t T = S.wic ? (uint64_t)S.tcsr[e] + 1 : S.t32;  // R3 / R4
      if (T == 0) continue;
      const uint32_t wb = __clz((uint32_t)(T - 1));
      uint32_t lo, hi;
      if (wb >= PACIM_TB) {
        const uint32_t p = he >> (32 - PACIM_TB);
        lo = tab[p];
        hi = tab[p + 1];
      } else if (wb == 0) {
        lo = 0;
        hi = S.B;
      } else {
        const uint32_t p = (he >> (32 - wb)) << (PACIM_TB - wb);
        lo = tab[p];
        hi = tab[p + (1u << (PACIM_TB - wb))];
      }
      uint32_t wr = NONE;
      for (uint32_t j = lo; j < hi; j++) {
        if (!((__ldcg(M + (j >> 5)) >> (j & 31)) & 1u)) continue;
        if ((uint64_t)(shr[j] ^ he) >= T) continue;
        if (wr == NONE) wr = S.cid[w];
        const uint32_t bit = 1u << (j & 31);
        const uint32_t old = atomicOr(S.vis + (size_t)wr * S.BW + (j >> 5), bit);
        if (old & bit) continue;  // already in this slot's CC walk
        if (w != s) sub_gain(S, w, __ldcg(S.dl + j));
        atomicOr(fm_nxt + (size_t)wr * S.BW + (j >> 5), bit);
        if (atomicExch(S.inl + (size_t)nxt * S.nr + wr, 1u) == 0u) {
          const bool heavy = S.off[w + 1] - S.off[w] > S.heavy_deg;
          if (heavy)
            S.hlist[(size_t)nxt * S.nr + atomicAdd(nhcnt, 1u)] = wr;
          else
            S.flist[(size_t)nxt * S.nr + atomicAdd(ncnt, 1u)] = wr;
        }
        // a row can enter several levels' lists (reached at different depths
        // in different slots) but is listed for the vis clean-up only once
        touch(S, wr);
      }
    }
  }
}

// One BFS level.  Light frontier rows are expanded by one block each (which
// then clears the row's frontier mask and list flag); heavy rows (degree >
// heavy_deg, e.g. hubs) by the whole grid, their masks cleared after the
// level barrier (clear_heavy).  Frontier lists alternate by level parity;
// their sizes live in fcnt[lvl % 3] (light) and fcnt[4 + lvl % 3] (heavy) so
// that the counters of level + 2 can be reset during the level.
__device__ void bfs_level(const Sel &S, uint32_t lvl, const uint32_t *shr, const uint16_t *tab,
                          uint32_t s) {
  const uint32_t cur = lvl & 1;
  const uint32_t cnt = __ldcg(S.fcnt + lvl % 3);
  const uint32_t hcnt = __ldcg(S.fcnt + 4 + lvl % 3);
  for (uint32_t i = blockIdx.x; i < cnt; i += gridDim.x) {
    const uint32_t u = __ldcg(S.flist + (size_t)cur * S.nr + i);
    expand_row(S, lvl, u, shr, tab, s, threadIdx.x, blockDim.x);
    __syncthreads();
    uint32_t *fm = S.fmask + ((size_t)cur * S.nr + u) * S.BW;
    for (uint32_t q = threadIdx.x; q < S.BW; q += blockDim.x) fm[q] = 0;
    if (threadIdx.x == 0) S.inl[(size_t)cur * S.nr + u] = 0;
  }
  const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t gn = (uint64_t)gridDim.x * blockDim.x;
  for (uint32_t i = 0; i < hcnt; i++) {
    const uint32_t u = __ldcg(S.hlist + (size_t)cur * S.nr + i);
    expand_row(S, lvl, u, shr, tab, s, gt, gn);
  }
}

// after the level barrier: clear the heavy rows' frontier masks and flags
__device__ void clear_heavy(const Sel &S, uint32_t lvl, uint64_t gt, uint64_t gn) {
  const uint32_t cur = lvl & 1;
  const uint32_t hcnt = __ldcg(S.fcnt + 4 + lvl % 3);
  for (uint64_t t = gt; t < (uint64_t)hcnt * S.BW; t += gn) {
    const uint32_t u = __ldcg(S.hlist + (size_t)cur * S.nr + t / S.BW);
    S.fmask[((size_t)cur * S.nr + u) * S.BW + t % S.BW] = 0;
    if (t % S.BW == 0) S.inl[(size_t)cur * S.nr + u] = 0;
  }
}

// dense pass for the big CCs covered this step: v is a member of slot j's
// covered CC iff its slot holds that root, or v is the root.  8 slots per
// lane kept in registers, rows streamed.
__device__ void apply_dense(const Sel &S, uint32_t s, size_t warp0, size_t nwarps) {
  const int lane = threadIdx.x & 31;
  for (uint32_t j0 = 0; j0 < S.B; j0 += 256) {
    uint32_t cr[8], cd[8];
    bool any = false;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const uint32_t j = j0 + lane + 32 * i;
      cr[i] = j < S.B ? __ldcg(S.cov_root + j) : NONE;
      cd[i] = j < S.B ? __ldcg(S.cov_delta + j) : 0;
      any |= cr[i] != NONE;
    }
    if (!__any_sync(0xffffffffu, any)) continue;
    for (size_t v = warp0; v < S.nr; v += nwarps) {
      uint32_t x[8];
#pragma unroll
      for (int i = 0; i < 8; i++)
        x[i] = cr[i] != NONE ? __ldcs(S.L + v * S.B + j0 + lane + 32 * i) : NONE;
      long long d = 0;
#pragma unroll
      for (int i = 0; i < 8; i++)
        if (cr[i] != NONE && (x[i] == cr[i] || (uint32_t)v == cr[i])) d += cd[i];
      for (int q = 16; q; q >>= 1) d += __shfl_xor_sync(0xffffffffu, d, q);
      if (lane == 0 && d) {
        const uint32_t vid = S.rmap[v];
        if (vid != s) atomicAdd((unsigned long long *)&S.target[vid], (unsigned long long)(-d));
      }
    }
  }
}

__device__ void load_tables(const Sel &S, uint32_t *shr, uint16_t *tab) {
  for (uint32_t i = threadIdx.x; i < S.B; i += blockDim.x) shr[i] = S.g_shr[i];
  for (uint32_t i = threadIdx.x; i <= (1u << PACIM_TB); i += blockDim.x) tab[i] = S.g_tab[i];
  __syncthreads();
}

struct SelOut {
  uint32_t k;
  uint32_t *seeds;
  long long *gain_num;   // k, zeroed
  long long *arg_gain;   // k
  unsigned long long *levels;
};

__global__ void __launch_bounds__(SEL_THREADS) k_select(Sel S0, SelOut O) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint32_t dsm[];
  Sel S = S0;
  uint32_t *shr = dsm;
  uint16_t *tab = reinterpret_cast<uint16_t *>(dsm + S.B);
  // per-warp queue / visited set / tail of warp_bfs, after the tables
  uint32_t *wbase = dsm + (table_words(S.B)) + (size_t)(threadIdx.x >> 5) * WARP_WORDS;
  uint32_t *wq = wbase, *whs = wbase + QCAP, *wtail = wbase + QCAP + HCAP;
  __shared__ Best sh[33];
  load_tables(S, shr, tab);
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  const size_t gwarp = tid >> 5, nwarps = nth >> 5;
  unsigned long long lvls = 0;
  for (uint32_t step = 0; step < O.k; step++) {
    S.par = step & 1;
    const uint32_t prev = S.par ^ 1;
    // ---- A1: refresh the chunk maxima whose gains changed; clear the
    //          previous step's visited bits
    const bool all = ((volatile int *)S.alldirty)[prev];
    const uint32_t nd = all ? S.nchunks : ((volatile uint32_t *)S.dcnt)[prev];
    for (uint32_t t = blockIdx.x; t < nd; t += gridDim.x) {
      const uint32_t c = all ? t : __ldcg(S.dlist + (size_t)prev * S.nchunks + t);
      const size_t v0 = (size_t)c << S.csh, v1 = min((size_t)S.nv, v0 + ((size_t)1 << S.csh));
      Best b{LLONG_MIN, 0xFFFFFFFFu};
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
    {  // rows visited by the previous step: clear their visited bits and flags
      const uint32_t nt = ((volatile uint32_t *)S.fcnt)[8 + prev];
      for (size_t t = tid; t < (size_t)nt * S.BW; t += nth) {
        const uint32_t r = __ldcg(S.touched + (size_t)prev * S.nr + t / S.BW);
        S.vis[(size_t)r * S.BW + (t % S.BW)] = 0;
        if (t % S.BW == 0) S.tflag[r] = 0;
      }
    }
    // level-0/1 list sizes for this step's BFS (nobody reads them before the
    // barrier; the previous step's loop exit only read zero ones)
    if (tid == 0) S.fcnt[0] = S.fcnt[1] = S.fcnt[4] = S.fcnt[5] = 0;
    grid.sync();
    // ---- A2: every block reduces the chunk maxima -> s
    Best c{LLONG_MIN, 0xFFFFFFFFu};
    for (uint32_t i = threadIdx.x; i < S.nchunks; i += blockDim.x) {
      Best x;
      x.g = __ldcg(&S.cmax[i].g);
      x.v = __ldcg(&S.cmax[i].v);
      if (better(x.g, x.v, c.g, c.v)) c = x;
    }
    c = block_best(c, sh);
    const uint32_t s = c.v;
    const uint32_t srow = S.cid[s];
    if (tid == 0) {
      S.alldirty[prev] = 0;
      S.dcnt[prev] = 0;
      S.dense[prev] = 0;
      S.fcnt[8 + prev] = 0;  // the previous step's touched rows were cleared in A1
      O.seeds[step] = s;
      O.arg_gain[step] = c.g;
      S.target[s] = -1;  // s leaves the candidate set (R6)
      mark_dirty(S, s);
    }
    // ---- B: MarkSeed, one warp per slot; small newly covered CCs are
    //          enumerated right here by the warp (warp_bfs) unless they are
    //          larger than its queue or reach a high-degree vertex, which
    //          defers them to the grid-wide BFS below
    {
      const int lane = threadIdx.x & 31;
      unsigned long long dsum = 0;
      for (size_t j = gwarp; j < S.B; j += nwarps) {
        uint32_t d = 0;
        if (lane == 0) d = cover_slot(S, srow, (uint32_t)j);
        d = __shfl_sync(0xffffffffu, d, 0);
        __syncwarp();
        dsum += d;
        const uint32_t small = __shfl_sync(0xffffffffu, lane == 0 ? __ldcg(S.dl + j) : 0u, 0);
        if (small) {
          bool done = false;
          if (small <= QCAP) done = warp_bfs(S, s, (uint32_t)j, small, wq, whs, wtail, shr);
          if (!done && lane == 0) defer_slot(S, s, srow, (uint32_t)j);
          __syncwarp();
        }
      }
      if (lane == 0 && dsum) atomicAdd((unsigned long long *)&O.gain_num[step], dsum);
    }
    grid.sync();
    // ---- C1: multi-slot BFS over the small newly covered CCs
    for (uint32_t lvl = 0;; lvl++) {
      // uniform decisions: counts read after a barrier
      const uint32_t nl = __ldcg(S.fcnt + lvl % 3), nh = __ldcg(S.fcnt + 4 + lvl % 3);
      if (nl == 0 && nh == 0) break;
      if (tid == 0) S.fcnt[(lvl + 2) % 3] = S.fcnt[4 + (lvl + 2) % 3] = 0;  // level + 2
      bfs_level(S, lvl, shr, tab, s);
      grid.sync();
      if (nh) {
        clear_heavy(S, lvl, tid, nth);
        grid.sync();
      }
      lvls++;
    }
    // ---- C2: dense pass for big CCs (uniform decision after the barrier)
    if (__ldcg(S.dense + S.par)) {
      apply_dense(S, s, gwarp, nwarps);
      if (tid == 0) S.alldirty[S.par] = 1;
      grid.sync();
    }
  }
  if (tid == 0) *O.levels = lvls;
}

// ------------------------------------------------ multi-rank step kernels
__global__ void k_cover_slots(Sel S, uint32_t s, unsigned long long *sum) {
  const uint32_t srow = S.cid[s];
  unsigned long long d = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < S.B; j += gridDim.x * blockDim.x) {
    d += cover_slot(S, srow, j);
    if (S.dl[j]) defer_slot(S, s, srow, j);  // all small CCs: grid BFS
  }
  if (d) atomicAdd(sum, d);
}

__global__ void __launch_bounds__(SEL_THREADS) k_bfs_level(Sel S, uint32_t lvl, uint32_t s) {
  extern __shared__ uint32_t dsm[];
  uint32_t *shr = dsm;
  uint16_t *tab = reinterpret_cast<uint16_t *>(dsm + S.B);
  load_tables(S, shr, tab);
  bfs_level(S, lvl, shr, tab, s);
}

__global__ void __launch_bounds__(256) k_dense(Sel S, uint32_t s) {
  if (!((volatile int *)S.dense)[S.par]) return;
  apply_dense(S, s, ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
              ((size_t)gridDim.x * blockDim.x) >> 5);
}

__global__ void k_clear_heavy(Sel S, uint32_t lvl) {
  clear_heavy(S, lvl, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
              (uint64_t)gridDim.x * blockDim.x);
}

__global__ void k_clear_touched(Sel S) {  // multi-rank calls use parity 0
  const uint32_t nt = S.fcnt[8];
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < (size_t)nt * S.BW;
       t += (size_t)gridDim.x * blockDim.x)
  {
    const uint32_t r = S.touched[t / S.BW];
    S.vis[(size_t)r * S.BW + (t % S.BW)] = 0;
    if (t % S.BW == 0) S.tflag[r] = 0;
  }
}

// restore: clear the covered bits set by the previous selection
__global__ void k_uncover(uint32_t *L, const unsigned long long *list, unsigned long long cnt) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (size_t)gridDim.x * blockDim.x)
    atomicAnd(L + list[i], ~COV);
}

__global__ void __launch_bounds__(SEL_THREADS) k_argmax_part(const long long *gain, uint32_t n,
                                                             Best *partial) {
  __shared__ Best sh[33];
  Best b{LLONG_MIN, 0xFFFFFFFFu};
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    long long g = gain[v];
    if (better(g, (uint32_t)v, b.g, b.v)) {
      b.g = g;
      b.v = (uint32_t)v;
    }
  }
  b = block_best(b, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = b;
}

__global__ void __launch_bounds__(SEL_THREADS) k_argmax_final(const Best *partial, uint32_t np,
                                                              Best *out) {
  __shared__ Best sh[33];
  Best c{LLONG_MIN, 0xFFFFFFFFu};
  for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
    Best x = partial[i];
    if (better(x.g, x.v, c.g, c.v)) c = x;
  }
  c = block_best(c, sh);
  if (threadIdx.x == 0) *out = c;
}

}  // namespace

// ------------------------------------------------------------------ host
static size_t table_smem(uint32_t B) {
  return ((size_t)B * 4 + ((1u << PACIM_TB) + 1) * 2 + 15) & ~(size_t)15;
}

// Device state shared by the single-rank kernel and the multi-rank calls.
static Sel make_sel(pacim_ctx *ctx, long long *target) {
  const uint32_t B = ctx->R_local, n = ctx->n, nr = ctx->nr;
  Sel S;
  S.off = ctx->off.as<uint64_t>();
  S.nbr = ctx->nbr.as<uint32_t>();
  S.K = ctx->K;
  S.t32 = ctx->t32;
  S.tcsr = ctx->tcsr.as<uint32_t>();
  S.wic = ctx->pmodel == PACIM_P_WIC;
  S.g_shr = ctx->d_shr.as<uint32_t>();
  S.g_tab = ctx->d_tab.as<uint16_t>();
  S.L = ctx->L.as<uint32_t>();
  S.nr = nr;
  S.B = B;
  S.BW = (B + 31) / 32;
  S.nv = n;
  S.cid = ctx->cid.as<uint32_t>();
  S.rmap = ctx->rmap.as<uint32_t>();
  S.target = target;
  S.big_t = BIG_DEFAULT;
  if (const char *e = getenv("PACIM_BIG_T"))  // tests: force the dense path
    S.big_t = (uint32_t)std::max(1L, atol(e));
  // argmax cache geometry: <= MAX_CHUNKS chunks of 2^csh vertices
  uint32_t csh = 12;
  while (((uint64_t)n + (1ull << csh) - 1) >> csh > MAX_CHUNKS) csh++;
  S.csh = csh;
  S.nchunks = (uint32_t)(((uint64_t)n + (1ull << csh) - 1) >> csh);
  // sel_list: dl[B], cov_root[B], cov_delta[B], dense[2], pad, cov_cnt, cov_list
  S.cov_cap = (uint64_t)std::max<uint32_t>(ctx->sel_k_cap, 128) * B;
  const size_t head_words = (3 * (size_t)B + 2 + 1) & ~(size_t)1;
  pc_ensure(ctx, ctx->sel_list, head_words * 4 + 8 + 8 * S.cov_cap + 64);
  uint32_t *base = ctx->sel_list.as<uint32_t>();
  S.dl = base;
  S.cov_root = base + B;
  S.cov_delta = base + 2 * (size_t)B;
  S.dense = reinterpret_cast<int *>(base + 3 * (size_t)B);
  S.cov_cnt = reinterpret_cast<unsigned long long *>(base + head_words);
  S.cov_list = S.cov_cnt + 1;
  // argmax cache: cmax[nchunks], cdirty[nchunks], dlist[2][nchunks], dcnt[2], alldirty[2]
  pc_ensure(ctx, ctx->sel_partial, (size_t)S.nchunks * (sizeof(Best) + 12) + 64);
  S.cmax = ctx->sel_partial.as<Best>();
  S.cdirty = reinterpret_cast<uint32_t *>(S.cmax + S.nchunks);
  S.dlist = S.cdirty + S.nchunks;
  S.dcnt = S.dlist + 2 * (size_t)S.nchunks;
  S.alldirty = reinterpret_cast<int *>(S.dcnt + 2);
  // BFS state: vis, fmask[2], inl[2], flist[2], touched, fcnt[3]
  const size_t bw = (size_t)nr * S.BW;
  // words: vis, fmask[2], inl[2], flist[2], hlist[2], touched[2], tflag, fcnt[16]
  const size_t words = 3 * bw + 9 * (size_t)nr + 16;
  if (ctx->bfs.bytes < words * 4 || ctx->bfs_nr != nr || ctx->bfs_bw != S.BW) {
    // new layout: every mask, flag and counter starts at zero
    pc_ensure(ctx, ctx->bfs, words * 4);
    PC_CUDA(cudaMemsetAsync(ctx->bfs.p, 0, words * 4, ctx->stream));
    ctx->bfs_nr = nr;
    ctx->bfs_bw = S.BW;
  }
  uint32_t *q = ctx->bfs.as<uint32_t>();
  S.vis = q;
  S.fmask = q + bw;
  S.inl = q + 3 * bw;
  S.flist = S.inl + 2 * (size_t)nr;
  S.hlist = S.flist + 2 * (size_t)nr;
  S.touched = S.hlist + 2 * (size_t)nr;
  S.tflag = S.touched + 2 * (size_t)nr;
  S.fcnt = S.tflag + nr;
  S.heavy_deg = 4096;
  S.par = 0;
  S.track = 0;
  return S;
}

// clear covered bits of the previous selection and the BFS bookkeeping
static void uncover(pacim_ctx *ctx, const Sel &S) {
  unsigned long long cnt = 0;
  if (ctx->sel_list_valid) {
    PC_CUDA(cudaMemcpyAsync(&cnt, S.cov_cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  PC_REQUIRE(cnt <= S.cov_cap, PACIM_ECHECK, "covered-CC list overflowed");
  if (cnt)
    k_uncover<<<pc_grid(ctx, cnt, 256), 256, 0, ctx->stream>>>(S.L, S.cov_list, cnt);
  PC_CUDA(cudaMemsetAsync(S.cov_cnt, 0, 8, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.dense, 0, 8, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.cov_root, 0xFF, (size_t)S.B * 4, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.vis, 0, (size_t)S.nr * S.BW * 4, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.tflag, 0, (size_t)S.nr * 4, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.fcnt, 0, 64, ctx->stream));
  ctx->sel_list_valid = true;
}

void pc_select_reset(pacim_ctx *ctx) {
  Sel S = make_sel(ctx, nullptr);
  uncover(ctx, S);
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

void pc_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
               int64_t *sigma_num) {
  const uint32_t n = ctx->n;
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  if (k > ctx->sel_k_cap) {
    // growing the covered list: clear the previous selection's bits first
    if (ctx->sel_list_valid) {
      Sel old = make_sel(ctx, nullptr);
      uncover(ctx, old);
    }
    ctx->sel_k_cap = k;
    ctx->sel_list_valid = false;
  }
  Sel S = make_sel(ctx, ctx->gain.as<long long>());
  S.track = 1;
  pc_ensure(ctx, ctx->sel_gain, (size_t)k * 16 + 64);
  pc_ensure(ctx, ctx->sel_seeds, (size_t)k * 4);
  SelOut O;
  O.k = k;
  O.seeds = ctx->sel_seeds.as<uint32_t>();
  O.gain_num = ctx->sel_gain.as<long long>();
  O.arg_gain = O.gain_num + k;
  O.levels = reinterpret_cast<unsigned long long *>(O.gain_num + 2 * k);
  const size_t smem = (size_t)table_words(S.B) * 4 + (SEL_THREADS / 32) * WARP_WORDS * 4;
  PC_REQUIRE(smem <= 200 * 1024, PACIM_ENOTIMPL, "too many sketch slots for k_select");
  PC_CUDA(cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  PC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_select, SEL_THREADS, smem));
  PC_REQUIRE(occ >= 1, PACIM_ECUDA, "k_select cannot be resident");
  const unsigned grid = (unsigned)ctx->sm_count * (unsigned)std::min(occ, 2);
  cudaEvent_t e0, e1;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  uncover(ctx, S);
  PC_CUDA(cudaMemcpyAsync(ctx->gain.p, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  PC_CUDA(cudaMemsetAsync(ctx->sel_gain.p, 0, (size_t)k * 16 + 64, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.cdirty, 0, (size_t)S.nchunks * 4, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.dcnt, 0, 8, ctx->stream));
  // step 0 reads the buffer of "step -1" (parity 1): everything dirty
  static const int init_all[2] = {0, 1};
  PC_CUDA(cudaMemcpyAsync(S.alldirty, init_all, 8, cudaMemcpyHostToDevice, ctx->stream));
  void *args[] = {&S, &O};
  PC_CUDA(cudaLaunchCooperativeKernel((void *)k_select, grid, SEL_THREADS, args, smem, ctx->stream));
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  std::vector<long long> hg(2 * (size_t)k + 1);
  PC_CUDA(cudaMemcpyAsync(seeds, O.seeds, (size_t)k * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(hg.data(), O.gain_num, (2 * (size_t)k + 1) * 8, cudaMemcpyDeviceToHost,
                          ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms = ms;
  ctx->stats.kernel_launches_select = 2;
  ctx->stats.select_member_updates = (uint64_t)hg[2 * (size_t)k];  // BFS levels run
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

void pc_cover_local(pacim_ctx *ctx, uint32_t s, int64_t *d_delta, int64_t *local_gain) {
  PC_REQUIRE(ctx->sel_list_valid, PACIM_ESTATE, "pacim_select_reset first");
  Sel S = make_sel(ctx, reinterpret_cast<long long *>(d_delta));
  pc_ensure(ctx, ctx->sel_flag, 64);
  unsigned long long *sum = ctx->sel_flag.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(sum, 0, 8, ctx->stream));
  PC_CUDA(cudaMemsetAsync(S.dense, 0, 8, ctx->stream));
  // previous call's visited rows, then the seed's row as the BFS start
  k_clear_touched<<<pc_grid(ctx, (size_t)S.nr, 256), 256, 0, ctx->stream>>>(S);
  // list and touched counters start empty; k_cover_slots defers the small
  // CCs (seed row into the level-0 list) and records touched rows
  PC_CUDA(cudaMemsetAsync(S.fcnt, 0, 64, ctx->stream));
  k_cover_slots<<<(S.B + 255) / 256, 256, 0, ctx->stream>>>(S, s, sum);
  PC_CHECK_LAUNCH();
  const size_t smem = table_smem(S.B);
  PC_CUDA(cudaFuncSetAttribute(k_bfs_level, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (uint32_t lvl = 0;; lvl++) {
    uint32_t c[7];
    PC_CUDA(cudaMemcpyAsync(c, S.fcnt, 28, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint32_t nl = c[lvl % 3], nh = c[4 + lvl % 3];
    if (!nl && !nh) break;
    PC_CUDA(cudaMemsetAsync(S.fcnt + (lvl + 2) % 3, 0, 4, ctx->stream));
    PC_CUDA(cudaMemsetAsync(S.fcnt + 4 + (lvl + 2) % 3, 0, 4, ctx->stream));
    k_bfs_level<<<ctx->sm_count * 2, SEL_THREADS, smem, ctx->stream>>>(S, lvl, s);
    PC_CHECK_LAUNCH();
    if (nh) {
      k_clear_heavy<<<pc_grid(ctx, (size_t)nh * S.BW, 256), 256, 0, ctx->stream>>>(S, lvl);
      PC_CHECK_LAUNCH();
    }

  }
  k_dense<<<pc_grid(ctx, (size_t)S.nr * 32, 256, 8), 256, 0, ctx->stream>>>(S, s);
  PC_CHECK_LAUNCH();
  unsigned long long h = 0;
  PC_CUDA(cudaMemcpyAsync(&h, sum, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  *local_gain = (int64_t)h;
}

void pc_argmax(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n, uint32_t *s, int64_t *g) {
  unsigned grid = pc_grid(ctx, n, SEL_THREADS, 2);
  DevBuf &part = ctx->argmax_part;  // persistent: no allocation per step
  pc_ensure(ctx, part, (size_t)(grid + 1) * sizeof(Best));
  k_argmax_part<<<grid, SEL_THREADS, 0, ctx->stream>>>(reinterpret_cast<const long long *>(d_gain),
                                                       n, part.as<Best>());
  PC_CHECK_LAUNCH();
  k_argmax_final<<<1, SEL_THREADS, 0, ctx->stream>>>(part.as<Best>(), grid,
                                                     part.as<Best>() + grid);
  PC_CHECK_LAUNCH();
  Best h;
  PC_CUDA(cudaMemcpyAsync(&h, part.as<Best>() + grid, sizeof(Best), cudaMemcpyDeviceToHost,
                          ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  *s = h.v;
  *g = h.g;
}
