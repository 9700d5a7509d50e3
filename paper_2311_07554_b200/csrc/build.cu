// build.cu — Step 1 of Alg. 1: Sketch(r) for every local sketch.
//
// Store layout (DESIGN.md §Store layout): the uncompressed store is ONE u32
// array L[v*B + j] (vertex-major; slot j = local sketch, slots sorted by
// hash(r) so that correlated sketches are adjacent in a row).
// During the build it is the union-find parent array of all B sketches; after
// compress_count / compact it is the per-vertex CC memo of P:597-601.
//
// Kernels (one pass each over L):
//   k_init            L[v][j] = v                                   (H3 setup)
//   k_edges           per upper edge: hash, candidate sketches, live test,
//                     lock-free hook-larger-root-under-smaller union (H2, H3);
//                     a warp flattens the candidate (edge, slot) pairs of 32
//                     edges and unites 32 pairs per round (adjacent slots of
//                     one edge -> coalesced row accesses, no idle lanes)
//   k_hot_roots       per slot the root of the hub vertex (hot component)
//   k_compress_count  full path compression to the min-id root (H4) and CC
//                     sizes counted into the root slot (H5); the hot root's
//                     count is aggregated per block in shared memory
//   k_compact         root slots -> compact component ids, member-index
//                     ranges allocated per tile                    (H6u)
//   k_gain_scatter    gain0[v] = sum_j |C_j(v)| (H7) and the member index
//                     perm grouped by component (H6u); hot-component cursor
//                     reservations aggregated per tile in shared memory
#include <type_traits>
#include <chrono>
#include <algorithm>
#include <cstdlib>

#include <cub/cub.cuh>

#include "pacim_internal.cuh"

namespace {

constexpr uint32_t HOT_MAX = 1024;  // slots with a shared-memory hot-root cache
// windows narrower than this use the (row, slot) lane map (measured: the
// warp-per-row kernels win from ~16 slots up, e.g. c4's 23-slot batch)
constexpr uint32_t NARROW_W = 16;
constexpr uint32_t NONE = 0xFFFFFFFFu;
#ifndef PACIM_UF_KEEP
#define PACIM_UF_KEEP 1  // uf_unite keeps the unmoved side's word (A/B: -DPACIM_UF_KEEP=0)
#endif

__device__ __forceinline__ uint32_t ld_cg(const uint32_t *p) { return __ldcg(p); }

// ---------------------------------------------------------------- k_init
// A root slot holds HIGH | size (size 1 until k_compress_count counts the
// members), a non-root slot its parent row: the union-find reads a HIGH value
// as "parent = itself", and counting a member is a single atomicAdd.
constexpr uint32_t ROOT1 = PACIM_HIGH | 1u;

__global__ void k_init(uint32_t *L, uint32_t n, uint32_t B) {
  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  // every slot starts as the root of a singleton: HIGH | 1 (R8 store form)
  if ((B & 3) == 0 && (reinterpret_cast<uintptr_t>(L) & 15) == 0) {
    const uint32_t B4 = B >> 2;
    const uint4 x = make_uint4(ROOT1, ROOT1, ROOT1, ROOT1);
    for (size_t v = warp; v < n; v += nw) {
      uint4 *row = reinterpret_cast<uint4 *>(L + v * B);
      for (uint32_t j = lane; j < B4; j += 32) row[j] = x;
    }
  } else {
    for (size_t v = warp; v < n; v += nw)
      for (uint32_t j = lane; j < B; j += 32) L[v * B + j] = ROOT1;
  }
}

// ------------------------------------------------------------- union-find
// Rem's union with splicing, lock-free (the UniteRemCAS variant of ConnectIt
// the paper uses, P:8 / P:1328): walk both paths one step at a time from the
// side with the larger parent; hook a root under the other side's parent, or
// splice the non-root's pointer over to the other side's (smaller) parent.
// Parents stay strictly smaller than children, so the final root of every
// CC is its minimum id (R8).  Two independent loads per step; the walk stops
// as soon as the two paths meet.  A root slot holds ROOT1 (read as itself).
// *hu / *hp (optional): the row hooked and the parent it was hooked under —
// every non-root slot of a build is hooked exactly once (a CAS from its root
// state; splices only move non-roots), so these pairs are the hook list
__device__ __forceinline__ void uf_unite(uint32_t *L, uint32_t B, uint32_t j, uint32_t u,
                                         uint32_t v, Ep ep = Ep{}, uint32_t *hu = nullptr,
                                         uint32_t *hp = nullptr) {
  // ep: slot epochs (a stale slot is a root; every write carries ep.tag and
  // every CAS expects the raw word it read)
  uint32_t *Lj = L + j;
#if PACIM_UF_KEEP
  // the side that did not move keeps the word it read: parents only
  // decrease, so a stale word names an ancestor (same set, smaller id) and
  // every hook is still a CAS against the word read; a failed CAS returns
  // the current word, which replaces the re-read
  uint32_t ru = ld_cg(Lj + (size_t)u * B), rv = ld_cg(Lj + (size_t)v * B);
  for (;;) {
    uint32_t pu = ep_rd(ru, ep), pv = ep_rd(rv, ep);
    if (pu & PACIM_HIGH) pu = u;
    if (pv & PACIM_HIGH) pv = v;
    if (pu == pv) return;
    if (pu < pv) {
      uint32_t t = u;
      u = v;
      v = t;
      t = pu;
      pu = pv;
      pv = t;
      t = ru;
      ru = rv;
      rv = t;
    }
    if (u == pu) {
      const uint32_t got = atomicCAS(Lj + (size_t)u * B, ru, pv | ep.tag);
      if (got == ru) {  // hooked root u under pv
        if (hu) {
          *hu = u;
          *hp = pv;
        }
        return;
      }
      ru = got;
    } else {
      atomicCAS(Lj + (size_t)u * B, ru, pv | ep.tag);  // splice (may lose a race harmlessly)
      u = pu;
      ru = ld_cg(Lj + (size_t)u * B);
    }
  }
#endif
  for (;;) {
    const uint32_t ru = ld_cg(Lj + (size_t)u * B), rv = ld_cg(Lj + (size_t)v * B);
    uint32_t pu = ep_rd(ru, ep), pv = ep_rd(rv, ep);
    if (pu & PACIM_HIGH) pu = u;
    if (pv & PACIM_HIGH) pv = v;
    if (pu == pv) return;
    uint32_t raw = ru;  // the word of the side that moves (u after the swap)
    if (pu < pv) {
      uint32_t t = u;
      u = v;
      v = t;
      t = pu;
      pu = pv;
      pv = t;
      raw = rv;
    }
    // now pu > pv
    if (u == pu) {
      if (atomicCAS(Lj + (size_t)u * B, raw, pv | ep.tag) == raw) {  // hook root u under pv
        if (hu) {
          *hu = u;
          *hp = pv;
        }
        return;
      }
    } else {
      atomicCAS(Lj + (size_t)u * B, raw, pv | ep.tag);  // splice (may lose a race harmlessly)
      u = pu;
    }
  }
}

// --------------------------------------------------------------- k_edges
// Sketch slot table in shared memory: shr[j] = hi32(hash(r_j)) ascending and
// tab[p] = #{j : shr[j] >> (32-TB) < p}.  live(e, j) <=> (shr[j] ^ he) < T
// implies the top w = clz(T-1) bits of shr[j] and he agree, so the candidate
// slots of an edge are one contiguous range of the sorted table (exact; R2
// candidate enumeration, SURVEY §8(a) note).
constexpr int EDGE_THREADS = 256;
constexpr int EDGE_WARPS = EDGE_THREADS / 32;
#ifndef PACIM_EDGE_BLOCKS
#define PACIM_EDGE_BLOCKS 8  // resident blocks per SM (32 registers)
#endif

// The live (edge, slot) pairs of the compact store's mask pass (CS = 2), for
// its union pass to read instead of hashing every edge again: entry =
// u_row << 36 | v_row << 8 | slot (rows < 2^28, slots < 256).  Each warp
// reserves PL_CHUNK entries at a time (*cnt += PL_CHUNK; unused ones = ~0);
// entries at or past cap are dropped (*cnt > cap: the host runs the full pass)
constexpr uint32_t PL_CHUNK = 512;  // list entries reserved per warp at a time
// Dynamic work distribution of k_edges: warps take chunks of `citer`
// 32-edge iterations from *ctr (zeroed before the launch) instead of a fixed
// grid stride, so warps whose unions hit contended roots do not leave the
// rest of their block idle at the end (c3: 23 % of the warp samples waited
// at the final barrier with the fixed stride)
struct EdgeWork {
  unsigned long long *ctr = nullptr;
  uint32_t citer = 1;
};
struct PairList {
  unsigned long long *p = nullptr;
  unsigned long long *cnt = nullptr;
  unsigned long long cap = 0;
};
// warp-wide (every lane calls it): the lanes with `has` append `val` to the
// warp's reserved chunk [base, base + PL_CHUNK) of `pl`, `used` of it filled
// (warp-uniform); a chunk that cannot take them is closed (holes: ~0) and
// the next one reserved with one counter add
__device__ __forceinline__ void pl_append(const PairList &pl, unsigned long long &base,
                                          uint32_t &used, bool has, unsigned long long val,
                                          int lane) {
  const uint32_t lm = __ballot_sync(0xffffffffu, has);
  const uint32_t nl = __popc(lm);
  if (!nl) return;
  if (used + nl > PL_CHUNK) {
    for (uint32_t q = used + lane; q < PL_CHUNK; q += 32)
      if (base + q < pl.cap) pl.p[base + q] = ~0ull;
    unsigned long long b0 = 0;
    if (lane == 0) b0 = atomicAdd(pl.cnt, (unsigned long long)PL_CHUNK);
    base = __shfl_sync(0xffffffffu, b0, 0);
    used = 0;
  }
  const unsigned long long at = base + used + __popc(lm & ((1u << lane) - 1));
  if (has && at < pl.cap) pl.p[at] = val;
  used += nl;
}

// LEAN: no edge list — the warp reads 32 consecutive CSR entries (chunk c),
// their rows from the chunk table (the row of the first entry, advanced while
// an entry lies past the row's end), and keeps the upper ones (v > u); rows
// are the vertex ids.  `keys` = CSR offsets, `ckeys` = neighbours (as u32),
// `tm1` = chunk rows, m = CSR entries (2m).
// CS: the compact store (store_cs.cu), j0 = 0, Bb = B.  CS = 1: the unions,
// L = the {P, next} words of the entries, (row, slot) = entry
// pc_cs_pos(rec, MW, row, slot); CS = 2: the mask pass, every live (edge,
// slot) sets bit slot of both endpoints' row masks (L = the rec words)
// LEAN = 2 (UpperCsr, the dense store, no HLA): upper edge e from the
// symmetric CSR (row by the chunk table ucrow, neighbour nbr[off[u+1] -
// (uoff[u+1] - e)]), the threshold tm1[e] (per-edge models), the store rows
// from the rank map — 8 B streamed per edge instead of keys + ckeys + tm1's 20
template <bool WIC, bool REC, bool DECOR, int LEAN, int CS = 0, bool EP = false>
__global__ void __launch_bounds__(EDGE_THREADS, PACIM_EDGE_BLOCKS) k_edges(const uint64_t *__restrict__ keys,
                                                        const uint64_t *__restrict__ ckeys,
                                                        const uint32_t *__restrict__ tm1,
                                                        uint64_t m, uint64_t K, uint64_t t32,
                                                        const uint32_t *__restrict__ g_shr,
                                                        const uint16_t *__restrict__ g_tab,
                                                        uint32_t B, uint32_t j0, uint32_t Bb,
                                                        uint32_t *L,
                                                        unsigned long long *live_ctr, Hla hla,
                                                        const uint64_t *__restrict__ hr64,
                                                        const uint2 *__restrict__ rec,
                                                        uint32_t MW, PairList pl, Ep ep,
                                                        EdgeWork ew, UpperCsr uc = UpperCsr{}) {
  // slots [j0, j0 + Bb) of the B sorted slots go to L (row stride Bb)
  extern __shared__ uint32_t sm[];
  uint32_t *shr = sm;
  uint16_t *tab = reinterpret_cast<uint16_t *>(sm + B);
  __shared__ uint32_t w_u[EDGE_WARPS][32], w_v[EDGE_WARPS][32], w_he[EDGE_WARPS][32];
  __shared__ uint32_t w_lo[EDGE_WARPS][32];
  __shared__ uint64_t w_T[EDGE_WARPS][32];
  __shared__ uint64_t w_he64[DECOR ? EDGE_WARPS : 1][32];  // R20: the full hash(e)
  __shared__ unsigned long long w_hla[REC ? EDGE_WARPS : 1][REC ? Hla::HLA_WBUF : 1];
  uint32_t hla_n = 0;  // entries staged in w_hla[wid] (warp-uniform)
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) shr[i] = g_shr[i];
  for (uint32_t i = threadIdx.x; i <= (1u << PACIM_TB); i += blockDim.x) tab[i] = g_tab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long live = 0;
  // pair list (CS = 2): the warp's current chunk [pl_base, pl_base + PL_CHUNK)
  // of the list, pl_used of it filled (warp-uniform; one counter add per chunk)
  unsigned long long pl_base = 0;
  uint32_t pl_used = PL_CHUNK;
  const uint64_t niter = (m + 31) / 32;
  uint64_t it = 0, it_end = 0;
  for (;;) {
    if (it >= it_end) {  // the warp's next chunk of iterations
      unsigned long long c0 = 0;
      if (lane == 0) c0 = atomicAdd(ew.ctr, (unsigned long long)ew.citer);
      it = __shfl_sync(0xffffffffu, c0, 0);
      if (it >= niter) break;
      it_end = min(it + ew.citer, niter);
    }
    const size_t base = it++ * 32;
    // ---- one edge per lane: hash and candidate slot range
    const size_t e = base + lane;
    uint32_t cnt = 0, eu = 0, ev = 0, ehe = 0, elo = 0;
    uint64_t eT = 0, ehe64 = 0;
    uint64_t lkey = 0, lrow = 0;
    bool upper = e < m;
    if (LEAN == 2 && upper) {
      const uint32_t v = uc.unbr[e], d = uc.ud16[e];
      uint32_t u = uc.ucrow[base >> 5], ru = uc.ucrowr[base >> 5] + (d >> 8);
      if ((d & 255u) != 255u)
        u += d & 255u;
      else  // the offsets search from the chunk's first row to the next chunk's
        u = pc_row_of(uc.uoff, u, (base >> 5) + 1 < niter ? uc.ucrow[(base >> 5) + 1] : uc.nv - 1, e);
      if ((d >> 8) == 255u) {
        const uint2 a = uc.rk[u >> 5];
        ru = a.x + __popc(a.y & ((1u << (u & 31)) - 1));
      }
      lkey = ((uint64_t)u << 32) | v;
      uint32_t rv;
      if (uc.uvrow) {
        rv = uc.uvrow[e];
      } else {
        const uint2 b = uc.rk[v >> 5];
        rv = b.x + __popc(b.y & ((1u << (v & 31)) - 1));
      }
      lrow = ((uint64_t)ru << 32) | rv;
    } else if (LEAN == 4 && upper) {
      const uint64_t c = base >> 5;
      const uint32_t u = pc_row_of(uc.uoff, uc.ucrow[c], c + 1 < niter ? uc.ucrow[c + 1] : uc.nv - 1, e);
      const uint32_t v = uc.nbr ? uc.nbr[uc.off[u + 1] - (uc.uoff[u + 1] - e)] : uc.unbr[e];
      lkey = ((uint64_t)u << 32) | v;
      const uint2 a = uc.rk[u >> 5], b = uc.rk[v >> 5];
      lrow = ((uint64_t)(a.x + __popc(a.y & ((1u << (u & 31)) - 1))) << 32) |
             (b.x + __popc(b.y & ((1u << (v & 31)) - 1)));
    } else if (LEAN == 3 && upper) {
      // lean graphs, upper entries only: e = upper edge index, the row by
      // the upper chunk table (tm1) and the upper offsets, the neighbour at
      // the row's upper part of the symmetric CSR (rows are [lower ++ upper])
      const uint64_t c = base >> 5;
      const uint32_t u = pc_row_of(uc.uoff, tm1[c], c + 1 < niter ? tm1[c + 1] : uc.nv - 1, e);
      const uint32_t v = reinterpret_cast<const uint32_t *>(ckeys)[keys[u + 1] - (uc.uoff[u + 1] - e)];
      lkey = ((uint64_t)u << 32) | v;
    } else if (LEAN && upper) {
      const uint32_t u = pc_row_of(keys, tm1[base >> 5],
                                   (base >> 5) + 1 < niter ? tm1[(base >> 5) + 1] : uc.nv - 1, e);
      const uint32_t v = reinterpret_cast<const uint32_t *>(ckeys)[e];
      upper = v > u;
      lkey = ((uint64_t)u << 32) | v;
    }
    if (upper) {
      const uint64_t key = LEAN ? lkey : keys[e];
      const uint64_t T = (WIC && LEAN != 1) ? (uint64_t)tm1[e] + t32 : t32;  // per-edge: t32 = toff
      const uint64_t he64 = pc_mix64(key ^ K);
      const uint32_t he = (uint32_t)(he64 >> 32);
      uint32_t lo = 0, hi = 0;
      if (DECOR) {  // R20: no leading-bit structure, every slot is a candidate
        if (T != 0) hi = B;
        ehe64 = he64;
      } else if (T != 0) {
        const uint32_t w = __clz((uint32_t)(T - 1));
        if (w >= PACIM_TB) {
          uint32_t p = he >> (32 - PACIM_TB);
          lo = tab[p];
          hi = tab[p + 1];
        } else if (w == 0) {
          lo = 0;
          hi = B;
        } else {
          uint32_t p = (he >> (32 - w)) << (PACIM_TB - w);
          lo = tab[p];
          hi = tab[p + (1u << (PACIM_TB - w))];
        }
      }
      lo = max(lo, j0);  // clip to the batch window
      hi = min(hi, j0 + Bb);
      if (hi < lo) hi = lo;
      cnt = hi - lo;
      const uint64_t ck = (LEAN == 2 || LEAN == 4) ? lrow : LEAN ? lkey : ckeys[e];  // the endpoints' store rows (+ hub flags)
      eu = (uint32_t)(ck >> 32);
      ev = (uint32_t)ck;
      ehe = he;
      eT = T;
      elo = lo;
    }
    // ---- compact the edges that have candidates; exclusive prefix of counts
    const uint32_t nz = __ballot_sync(0xffffffffu, cnt > 0);
    uint32_t inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    const uint32_t pre = inc - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    if (cnt) {
      const uint32_t k = __popc(nz & ((1u << lane) - 1));
      w_u[wid][k] = eu;
      w_v[wid][k] = ev;
      w_he[wid][k] = ehe;
      if (DECOR) w_he64[DECOR ? wid : 0][k] = ehe64;
      if (WIC) w_T[wid][k] = eT;
      w_lo[wid][k] = elo - pre;  // slot of candidate position idx: w_lo + idx
    }
    __syncwarp();
    // ---- 32 (edge, slot) candidate pairs per round; lane -> edge by the
    //      start positions of this round (no search): rank = edges started
    //      before the round + starts at or below the lane, minus one
    for (uint32_t c0 = 0; c0 < total; c0 += 32) {
      const uint32_t idx = c0 + lane;
      const uint32_t smask =
          __reduce_or_sync(0xffffffffu, (cnt && pre >= c0 && pre < c0 + 32) ? 1u << (pre - c0) : 0u);
      const uint32_t before = __popc(__ballot_sync(0xffffffffu, cnt && pre < c0));
      uint32_t j = 0, u = 0, v = 0;
      bool lv = false;
      if (idx < total) {
        const uint32_t a = before + __popc(smask & (0xffffffffu >> (31 - lane))) - 1;
        j = w_lo[wid][a] + idx;
        const uint64_t T = WIC ? w_T[wid][a] : t32;
        if (DECOR)  // R20
          lv = T >= (1ull << 32) ||
               (pc_mix64(__ldg(hr64 + j) ^ w_he64[DECOR ? wid : 0][a]) >> 32) < T;
        else
          lv = (uint64_t)(shr[j] ^ w_he[wid][a]) < T;
        u = w_u[wid][a];
        v = w_v[wid][a];
      }
      if (REC)  // live edges of hubs, staged per warp (before the union: u, v, j
                // need not survive it)
        hla.stage(u & ~PACIM_HUBF, v & ~PACIM_HUBF, j, (lv && (u & PACIM_HUBF)) ? 1u : 0u,
                  (lv && (v & PACIM_HUBF)) ? 1u : 0u, w_hla[REC ? wid : 0], hla_n);
      if (CS >= 2) {
        const uint32_t uu = u & ~PACIM_HUBF, vv = v & ~PACIM_HUBF;
        if (CS == 2) {
          // mask pass: the lanes of one (row, word) combine (u-side runs are
          // adjacent), one atomicOr each; the v side is one atomicOr per pair
          const unsigned long long ku = lv ? ((unsigned long long)uu << 8 | (j >> 5)) : ~0ull;
          const uint32_t peers = __match_any_sync(0xffffffffu, ku);
          const uint32_t bits = __reduce_or_sync(peers, lv ? 1u << (j & 31) : 0u);
          if (lv && (threadIdx.x & 31) == __ffs(peers) - 1)
            atomicOr(L + ((size_t)uu * MW + (j >> 5)) * 2 + 1, bits);
          if (lv) atomicOr(L + ((size_t)vv * MW + (j >> 5)) * 2 + 1, 1u << (j & 31));
        }
        live += lv;
        // CS = 3 (edge-partitioned sharded build): the pair list only, slot =
        // the global sorted slot of the sketch (its owner rank routes it)
        if (pl.p)  // the pair for the union pass, into the warp's reserved chunk
          pl_append(pl, pl_base, pl_used, lv,
                    (unsigned long long)uu << 36 | (unsigned long long)vv << 8 | j, lane);
      } else {
        // the hook list of an epoch build (CS = 0, EP, pl.p): {parent << 36 |
        // row << 8 | slot} of every successful hook — exactly the build's
        // non-root slots, so the compression pass reads them instead of
        // streaming the store (k_compress_count<…, LIST>)
        uint32_t hu = NONE, hp = 0;
        if (lv) {
          if (CS == 1)
            uf_unite(L, 2, 0, pc_cs_pos(rec, MW, u & ~PACIM_HUBF, j),
                     pc_cs_pos(rec, MW, v & ~PACIM_HUBF, j));
          else
            uf_unite(L, Bb, j - j0, u & ~PACIM_HUBF, v & ~PACIM_HUBF, EP ? ep : Ep{},
                     (CS == 0 && EP) ? &hu : nullptr, (CS == 0 && EP) ? &hp : nullptr);
          live++;
        }
        if (CS == 0 && EP && pl.p)
          pl_append(pl, pl_base, pl_used, hu != NONE,
                    (unsigned long long)hp << 36 | (unsigned long long)hu << 8 | (j - j0), lane);
      }
    }
    __syncwarp();
  }
  if (REC) hla.flush(w_hla[REC ? wid : 0], hla_n);
  if ((CS >= 2 || (CS == 0 && EP)) && pl.p)  // the last chunk's holes
    for (uint32_t q = pl_used + lane; q < PL_CHUNK; q += 32)
      if (pl_base + q < pl.cap) pl.p[pl_base + q] = ~0ull;
  // block-aggregated counter
  for (int d = 16; d; d >>= 1) live += __shfl_xor_sync(0xffffffffu, live, d);
  __shared__ unsigned long long bsum;
  if (threadIdx.x == 0) bsum = 0;
  __syncthreads();
  if (lane == 0 && live) atomicAdd(&bsum, live);
  __syncthreads();
  if (threadIdx.x == 0 && bsum) atomicAdd(live_ctr, bsum);
}

// ---------------------------------------------------------- hot roots
// read-only find that also stops at a converted root slot (HIGH set)
__device__ __forceinline__ uint32_t find_ro(const uint32_t *L, uint32_t B, uint32_t j,
                                            uint32_t x, Ep ep = Ep{}) {
  for (;;) {
    const uint32_t p = ep_rd(ld_cg(L + (size_t)x * B + j), ep);
    if (p == x || (p & PACIM_HIGH)) return x;
    x = p;
  }
}

// find with path halving for compress_count: every write is an atomicMin, so
// a slot only ever moves towards its root (ids decrease along parent
// pointers) and racing halvings can never undo an owner's full compression.
// ep: slot epochs; *root_raw = the root slot's word as read (stale: the root
// was never written in this build — add_to_root makes it current first)
__device__ __forceinline__ uint32_t find_halve(uint32_t *L, uint32_t B, uint32_t j, uint32_t x,
                                               Ep ep = Ep{}, uint32_t *root_raw = nullptr) {
  for (;;) {
    const uint32_t rp = ld_cg(L + (size_t)x * B + j), p = ep_rd(rp, ep);
    if (p == x || (p & PACIM_HIGH)) {
      if (root_raw) *root_raw = rp;
      return x;
    }
    const uint32_t rg = ld_cg(L + (size_t)p * B + j), gp = ep_rd(rg, ep);
    if (gp == p || (gp & PACIM_HIGH)) {
      if (root_raw) *root_raw = rg;
      return p;
    }
    atomicMin(L + (size_t)x * B + j, gp | ep.tag);  // same epoch bits: the min of the ids
    x = gp;
  }
}

__global__ void k_hot_roots(const uint32_t *L, uint32_t nr, uint32_t B, uint32_t hub,
                            uint32_t *hot, Ep ep) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x)
    hot[j] = hub < nr ? find_ro(L, B, j, hub, ep) : NONE;
}

// ------------------------------------------------------ k_compress_count
// For every non-root (v, j): slot <- root (full compression, H4; halving and
// the owner's write are atomicMin, so the final slot is the root); the
// root slot becomes HIGH | size by CAS(root -> HIGH|1) then atomicAdd per
// member (H5).  Members of the slot's hot root are counted in shared memory
// and added once per block.  ctr[1] += non-roots (the CCs of size >= 2 are
// counted into ctr[0] by the gain pass that reads every root slot anyway).
__device__ __forceinline__ void add_to_root(uint32_t *L, uint32_t B, uint32_t j, uint32_t root,
                                            uint32_t cnt, Ep ep = Ep{}, uint32_t root_raw = 0) {
  uint32_t *a = L + (size_t)root * B + j;
  if ((root_raw & ep.mask) != ep.tag) {
    // a stale root slot (a singleton until this build): the claim writes
    // HIGH | (1 + cnt) of this epoch in one CAS (the claimer's count rides
    // on it: one random atomic per CC fewer); racing members: the first CAS
    // wins, the others see a current word and add
    uint32_t x = root_raw;
    for (;;) {
      const uint32_t y = atomicCAS(a, x, ((PACIM_HIGH | 1u) | ep.tag) + cnt);
      if (y == x) return;
      if ((y & ep.mask) == ep.tag) break;
      x = y;
    }
  }
  // the root slot is HIGH | size (ROOT1 from k_init or the line above): one
  // atomic whose result is not waited for (the CCs are counted by the gain pass)
  atomicAdd(a, cnt);
}

// warp-reduced counter update (lane 0 adds)
__device__ __forceinline__ void add_count(unsigned long long *ctr, unsigned long long c) {
  for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(ctr, c);
}

constexpr uint32_t CLCAP = 256 + 31;  // pending finds per warp: < 32 carried + one 256-slot block
template <bool COMPACT, bool EP, bool LIST = false>
__global__ void __launch_bounds__(256) k_compress_count(uint32_t *L, uint32_t n, uint32_t B,
                                                        const uint32_t *hot,
                                                        unsigned long long *ctr, Ep ep_in,
                                                        const unsigned long long *hl = nullptr,
                                                        const unsigned long long *hl_cnt = nullptr,
                                                        unsigned long long hl_cap = 0) {
  const Ep ep = EP ? ep_in : Ep{};  // without epochs every epoch operation folds away
  extern __shared__ uint32_t hsm[];
  __shared__ uint32_t cl_v[COMPACT ? 8 : 1][COMPACT ? CLCAP : 1],
      cl_j[COMPACT ? 8 : 1][COMPACT ? CLCAP : 1], cl_s[COMPACT ? 8 : 1][COMPACT ? CLCAP : 1];
  const uint32_t H = min(B, HOT_MAX);
  uint32_t *hroot = hsm, *hcnt = hsm + H;
  for (uint32_t j = threadIdx.x; j < H; j += blockDim.x) {
    hroot[j] = hot[j];
    hcnt[j] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long nnr = 0;
  // the non-root slots that need a find, compacted per warp (over rows until
  // >= 32 are pending) so that each lane walks one chain per round: a row's
  // cost is its longest chain, not the sum over the 8 slots a lane holds
  // (c2 compress 1.05 -> 0.79 ms, c4 21.6 -> 19.7 ms; dense stores keep the
  // per-lane walk: on c3 compaction cost 18 -> 24 ms)
  const int wib = COMPACT ? threadIdx.x >> 5 : 0;
  uint32_t *cv = cl_v[wib], *cj = cl_j[wib], *cs = cl_s[wib];
  uint32_t cnt = 0;  // warp-uniform
  auto flush = [&]() {
    __syncwarp();
    for (uint32_t base = 0; base < cnt; base += 32) {
      const uint32_t k = base + lane;
      if (k < cnt) {
        const uint32_t v = cv[k], j = cj[k], s = cs[k];
        uint32_t rr = 0;
        const uint32_t root = find_halve(L, B, j, s, ep, &rr);
        if (root != s) atomicMin(L + (size_t)v * B + j, root | ep.tag);
        if (j < H && root == hroot[j])
          atomicAdd(hcnt + j, 1u);
        else
          add_to_root(L, B, j, root, 1u, ep, rr);
      }
    }
    __syncwarp();
    cnt = 0;
  };
  // LIST: the fallback of k_compress_list — the row stream only when the hook
  // list overflowed its capacity
  if (LIST && *hl_cnt <= hl_cap) return;
  for (size_t v = warp; v < n; v += nw) {
    for (uint32_t j0 = 0; j0 < B; j0 += 256) {
      uint32_t sv[8];  // prefetch up to 8 slots per lane (independent loads)
#pragma unroll
      for (int i = 0; i < 8; i++) {
        uint32_t j = j0 + lane + 32 * i;
        sv[i] = j < B ? ld_cg(L + v * B + j) : PACIM_HIGH;  // past B: skipped as a root
      }
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const uint32_t j = j0 + lane + 32 * i;
        // a member of this epoch (stale slots and roots need nothing)
        const bool nonroot = (sv[i] & (PACIM_HIGH | ep.mask)) == ep.tag;
        const uint32_t s = sv[i] & ~ep.mask;
        // parent already the hot root: no walk (the common case for members
        // of the giant CC)
        const bool hotp = nonroot && j < H && s == hroot[j];
        if (hotp) atomicAdd(hcnt + j, 1u);
        nnr += nonroot;
        const bool need = nonroot && !hotp;
        if (!COMPACT) {  // dense stores (c3): each lane walks its slots' chains in turn
          if (need) {
            uint32_t rr = 0;
            const uint32_t root = find_halve(L, B, j, s, ep, &rr);
            if (root != s) atomicMin(L + v * B + j, root | ep.tag);
            if (j < H && root == hroot[j])
              atomicAdd(hcnt + j, 1u);
            else
              add_to_root(L, B, j, root, 1u, ep, rr);
          }
          continue;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, need);
        if (need) {
          const uint32_t pos = cnt + __popc(m & ((1u << lane) - 1));
          cv[pos] = (uint32_t)v;
          cj[pos] = j;
          cs[pos] = s;
        }
        cnt += __popc(m);
      }
      if (COMPACT && cnt >= 32) flush();
    }
  }
  if (COMPACT) flush();
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < H; j += blockDim.x)
    if (hcnt[j])
      add_to_root(L, B, j, hroot[j], hcnt[j], ep, ld_cg(L + (size_t)hroot[j] * B + j));
  for (int d = 16; d; d >>= 1) nnr += __shfl_xor_sync(0xffffffffu, nnr, d);
  __shared__ unsigned long long s1;
  if (threadIdx.x == 0) s1 = 0;
  __syncthreads();
  if (lane == 0 && nnr) atomicAdd(&s1, nnr);
  __syncthreads();
  if (threadIdx.x == 0 && s1) atomicAdd(ctr + 1, s1);
}

// k_compress_count from the hook list (epoch builds): when k_edges' list is
// complete (*hl_cnt <= hl_cap) the non-root slots are read from it — lane per
// entry, the find starting at the parent recorded at the hook (an ancestor:
// later splices only moved the slot closer to the root) — instead of
// streaming all rows x B slots of the store (c4: 37 GB for 0.54 G
// non-roots).  An overflowed list: nothing here, k_compress_count<…, LIST>
// streams the rows instead (both launched, each decides on the device)
template <bool EP>
__global__ void __launch_bounds__(256, 8) k_compress_list(uint32_t *L, uint32_t B,
                                                          const uint32_t *hot,
                                                          unsigned long long *ctr, Ep ep_in,
                                                          const unsigned long long *__restrict__ hl,
                                                          const unsigned long long *hl_cnt,
                                                          unsigned long long hl_cap,
                                                          unsigned long long *work) {
  const Ep ep = EP ? ep_in : Ep{};
  const unsigned long long hl_n = *hl_cnt;
  if (hl_n > hl_cap) return;
  extern __shared__ uint32_t hsm[];
  const uint32_t H = min(B, HOT_MAX);
  uint32_t *hroot = hsm, *hcnt = hsm + H;
  for (uint32_t j = threadIdx.x; j < H; j += blockDim.x) {
    hroot[j] = hot[j];
    hcnt[j] = 0;
  }
  __syncthreads();
  unsigned long long nnr = 0;
  // dynamic work distribution: a warp takes LCH entries at a time from
  // *work (zeroed before the launch) — chains and root contention differ
  // between entries, so a static split leaves SMs idle at the end
  constexpr uint32_t LCH = 2048;
  const int lane = threadIdx.x & 31;
  unsigned long long b = 0, b_end = 0;  // warp-uniform
  for (;;) {
    if (b >= b_end) {
      unsigned long long c0 = 0;
      if (lane == 0) c0 = atomicAdd(work, (unsigned long long)LCH);
      c0 = __shfl_sync(0xffffffffu, c0, 0);
      if (c0 >= hl_n) break;
      b = c0;
      b_end = min(c0 + LCH, hl_n);
    }
    const unsigned long long i = b + lane;
    b += 32;
    const unsigned long long e = i < b_end ? hl[i] : ~0ull;
    if (e == ~0ull) continue;  // a chunk's hole (or past the end)
    const uint32_t j = (uint32_t)e & 255u, v = (uint32_t)(e >> 8) & 0x0FFFFFFFu,
                   s = (uint32_t)(e >> 36);
    nnr++;
    if (j < H && s == hroot[j]) {  // hooked under the hot root itself
      atomicAdd(hcnt + j, 1u);
      continue;
    }
    uint32_t rr = 0;
    const uint32_t root = find_halve(L, B, j, s, ep, &rr);
    if (root != s) atomicMin(L + (size_t)v * B + j, root | ep.tag);
    if (j < H && root == hroot[j])
      atomicAdd(hcnt + j, 1u);
    else
      add_to_root(L, B, j, root, 1u, ep, rr);
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < H; j += blockDim.x)
    if (hcnt[j]) add_to_root(L, B, j, hroot[j], hcnt[j], ep, ld_cg(L + (size_t)hroot[j] * B + j));
  add_count(ctr + 1, nnr);
}

// ------------------------------------------------------- k_gain0_narrow
// k_gain0 for narrow stores (B <= 32 S slots, S = 1, 2, 4: a rank's shard of
// a sharded build, P >= 2 at R = 256): S slots per lane and 32 / S rows per warp
// iteration (32 loads in flight per lane, as k_gain0's 8 slots x 4 rows); the
// per-row sums through shared memory (lane r adds row r's 32 partials) —
// k_gain0 kept 8 slot loads per lane of which B = 32 used one (c4 shard at
// P = 8: 7.7 ms for an eighth of the one-GPU store)
template <bool EP, int S>
__global__ void __launch_bounds__(256) k_gain0_narrow(const uint32_t *__restrict__ L, uint32_t n,
                                                      uint32_t B, const uint32_t *rmap,
                                                      int64_t *gain0, int acc,
                                                      unsigned long long *ncc_ctr, Ep ep_in) {
  const Ep ep = EP ? ep_in : Ep{};
  constexpr int GR = 32 / S;
  using part_t = typename std::conditional<(S <= 2), uint32_t, unsigned long long>::type;
  __shared__ part_t red[8][GR][33];
  unsigned long long ncc = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t szm = PACIM_LOW & ~ep.mask;
  for (size_t v0 = warp * GR; v0 < n; v0 += nw * GR) {
    uint32_t sv[GR][S];
#pragma unroll
    for (int r = 0; r < GR; r++)
#pragma unroll
      for (int i = 0; i < S; i++) {
        const uint32_t j = lane + 32 * i;
        sv[r][i] = (j < B && v0 + r < n) ? L[(v0 + r) * B + j] : NONE;
      }
#pragma unroll
    for (int r = 0; r < GR; r++)
#pragma unroll
      for (int i = 0; i < S; i++) {
        const uint32_t j = lane + 32 * i, raw = sv[r][i];
        if (raw == NONE) continue;
        const bool cur = (raw & ep.mask) == ep.tag;
        const uint32_t s = raw & ~ep.mask;
        if (!cur || (raw & PACIM_HIGH)) {
          ncc += cur && (s & PACIM_LOW) >= 2;
          if (!cur) sv[r][i] = (PACIM_HIGH | 1u) | ep.tag;
        } else {
          sv[r][i] = __ldg(L + (size_t)s * B + j);  // the root's word (of this epoch)
        }
      }
#pragma unroll
    for (int r = 0; r < GR; r++) {
      part_t p = 0;  // S <= 2: at most two sizes below 2^31 fit 32 bits
#pragma unroll
      for (int i = 0; i < S; i++)
        if (sv[r][i] != NONE) p += sv[r][i] & szm;
      red[wid][r][lane] = p;
    }
    __syncwarp();
    if (lane < GR && v0 + lane < n) {
      long long t = 0;
#pragma unroll 8
      for (int l = 0; l < 32; l++) t += red[wid][lane][l];
      const uint32_t v = rmap[v0 + lane];
      if (acc) {
        if (t != (long long)B) gain0[v] += t - (long long)B;
      } else {
        gain0[v] = t;
      }
    }
    __syncwarp();
  }
  add_count(ncc_ctr, ncc);
}

// ---------------------------------------------------------------- k_gain0
// Warp per store row, 8 slots prefetched per lane: gain0[v] = sum_j |C_j(v)|
// (H7), the CC size read from the root slot (HIGH | size).
// acc: window of a multi-window store, gain0[v] += sum (|C| - 1) over its
// slots (gain0 starts at B); else gain0[v] = the sum over all B slots
constexpr int GR_PLAIN = 4;  // rows per warp iteration in k_gain0 (4 KB of slots in flight)
// HOT: also hotsum[v] = the sizes of the hot (hub's) CCs above big_t that
// contain v — the select covers them by one vector pass when they are
// exactly the step's dense set (k_select phase D)
template <bool HOT, bool EP>
__global__ void __launch_bounds__(256) k_gain0(const uint32_t *__restrict__ L, uint32_t n,
                                               uint32_t B, const uint32_t *rmap, int64_t *gain0,
                                               int acc, unsigned long long *ncc_ctr,
                                               const uint32_t *hot, const uint32_t *hot_size,
                                               uint32_t big_t, int64_t *hotsum, Ep ep_in) {
  const Ep ep = EP ? ep_in : Ep{};
  constexpr int GR = HOT ? 2 : GR_PLAIN;  // fewer rows in flight: the hot sums' registers
  unsigned long long ncc = 0;  // roots of size >= 2: the non-singleton CCs
  extern __shared__ uint32_t hsm[];
  const uint32_t H = HOT ? min(B, HOT_MAX) : 0;
  uint32_t *hroot = hsm, *hsz = hsm + H;
  if (HOT) {
    for (uint32_t j = threadIdx.x; j < H; j += blockDim.x) {
      hroot[j] = hot[j];
      hsz[j] = hot_size[j] > big_t ? hot_size[j] : 0u;  // 0: not a giant
    }
    __syncthreads();
  }

  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t v0 = warp * GR; v0 < n; v0 += nw * GR) {
    long long g[GR], hs[GR];
#pragma unroll
    for (int r = 0; r < GR; r++) g[r] = hs[r] = 0;
    for (uint32_t j0 = 0; j0 < B; j0 += 256) {
      uint32_t sv[GR][8];
#pragma unroll
      for (int r = 0; r < GR; r++)
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const uint32_t j = j0 + lane + 32 * i;
          sv[r][i] = (j < B && v0 + r < n) ? L[(v0 + r) * B + j] : NONE;
        }
      // a non-root slot becomes its root's HIGH | size: the root loads of
      // both rows in flight together (raw words: the epoch bits are masked
      // off in the sum, a stale slot becomes HIGH | 1 of this epoch)
#pragma unroll
      for (int r = 0; r < GR; r++)
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const uint32_t j = j0 + lane + 32 * i;
          const uint32_t raw = sv[r][i];
          if (raw == NONE) continue;
          const bool cur = (raw & ep.mask) == ep.tag;
          const bool nonroot = cur && !(raw & PACIM_HIGH);
          const uint32_t s = raw & ~ep.mask;
          if (HOT && j < H && hsz[j]) {  // a member of slot j's giant hot CC
            const uint32_t root = nonroot ? s : (uint32_t)(v0 + r);
            if (root == hroot[j]) hs[r] += hsz[j];
          }
          if (!nonroot) {
            ncc += cur && (s & PACIM_LOW) >= 2;
            if (!cur) sv[r][i] = (PACIM_HIGH | 1u) | ep.tag;
          } else {
            sv[r][i] = __ldg(L + (size_t)s * B + j);  // the root's word (of this epoch)
          }
        }
      const uint32_t szm = PACIM_LOW & ~ep.mask;
#pragma unroll
      for (int r = 0; r < GR; r++)
#pragma unroll
        for (int i = 0; i < 8; i++)
          if (sv[r][i] != NONE) g[r] += sv[r][i] & szm;
    }
#pragma unroll
    for (int r = 0; r < GR; r++) {
      long long t = g[r];
      for (int d = 16; d; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
      if (lane == 0 && v0 + r < n) {
        if (acc) {
          if (t != (long long)B) gain0[rmap[v0 + r]] += t - (long long)B;
        } else {
          gain0[rmap[v0 + r]] = t;
        }
      }
      if (HOT) {
        long long h = hs[r];
        for (int d = 16; d; d >>= 1) h += __shfl_xor_sync(0xffffffffu, h, d);
        if (lane == 0 && v0 + r < n) hotsum[rmap[v0 + r]] = h;
      }
    }
  }
  add_count(ncc_ctr, ncc);
}

// k_gain0 for B <= 256 (HOT: with the hot sums): a lane's slots (j = lane + 32 i) are the same
// in every row, so the giant hot roots and sizes sit in registers; empty
// entries (j >= B, rows past n) read as HIGH | 0 — a root of size 0, never a
// stored value — so no entry needs a validity test (the HOT pass was issue
// bound: 73 % SM throughput at c2 / c3 in ncu)
template <int GR, bool HOT, bool EP>
__global__ void __launch_bounds__(256, GR == 2 ? (EP ? 3 : 4) : 2) k_gain0_fast(const uint32_t *__restrict__ L, uint32_t n,
                                                   uint32_t B, const uint32_t *rmap,
                                                   int64_t *gain0, unsigned long long *ncc_ctr,
                                                   const uint32_t *hot, const uint32_t *hot_size,
                                                   uint32_t big_t, int64_t *hotsum, Ep ep_in) {
  const Ep ep = EP ? ep_in : Ep{};
  const uint32_t VOID = PACIM_HIGH | ep.tag;  // HIGH | 0 of this epoch
  const int lane = threadIdx.x & 31;
  uint32_t hr[8], hz[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const uint32_t j = lane + 32 * i;
    const bool giant = HOT && j < B && hot_size[j] > big_t;
    hr[i] = giant ? hot[j] : NONE;  // NONE: never a row
    hz[i] = giant ? hot_size[j] : 0u;
  }
  uint32_t ncc = 0;  // roots of size >= 2
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t v0 = warp * GR; v0 < n; v0 += nw * GR) {
    uint32_t sv[GR][8];
#pragma unroll
    for (int r = 0; r < GR; r++) {
      const uint32_t *Lr = L + (v0 + r) * B;
      const bool rv = v0 + r < n;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const uint32_t j = lane + 32 * i;
        sv[r][i] = (rv && j < B) ? Lr[j] : VOID;
      }
    }
    unsigned long long hs[GR];
#pragma unroll
    for (int r = 0; r < GR; r++) {
      hs[r] = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const uint32_t raw = sv[r][i];
        const bool cur = (raw & ep.mask) == ep.tag;
        const uint32_t s = raw & ~ep.mask;
        const bool isroot = !cur || (raw & PACIM_HIGH) != 0;  // stale: a singleton root
        const uint32_t root = isroot ? (uint32_t)(v0 + r) : s;
        if (HOT) hs[r] += root == hr[i] ? hz[i] : 0u;
        if (isroot) {
          ncc += cur && (s & PACIM_LOW) >= 2;
          if (!cur) sv[r][i] = (PACIM_HIGH | 1u) | ep.tag;
        } else {
          sv[r][i] = __ldg(L + (size_t)s * B + lane + 32 * i);  // the root's word (this epoch)
        }
      }
    }
#pragma unroll
    for (int r = 0; r < GR; r++) {
      // sizes < 2^31: a pair sums in 32 bits
      unsigned long long t = 0;
#pragma unroll
      const uint32_t szm = PACIM_LOW & ~ep.mask;
#pragma unroll
      for (int i = 0; i < 8; i += 2) t += (sv[r][i] & szm) + (sv[r][i + 1] & szm);
      unsigned long long h = hs[r];
      for (int d = 16; d; d >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, d);
        if (HOT) h += __shfl_xor_sync(0xffffffffu, h, d);
      }
      if (lane == 0 && v0 + r < n) {
        const uint32_t v = rmap[v0 + r];
        gain0[v] = (long long)t;
        if (HOT) hotsum[v] = (long long)h;
      }
    }
  }
  add_count(ncc_ctr, ncc);
}

// per slot the hot (hub's) CC size, read from its root slot after compression
__global__ void k_hot_sizes(const uint32_t *L, uint32_t n, uint32_t B, const uint32_t *hot,
                            uint32_t *hot_size, Ep ep) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x)
    hot_size[j] = hot[j] < n ? (ep_rd(L[(size_t)hot[j] * B + j], ep) & PACIM_LOW) : 0u;
}

// HLA: entries sorted by key -> rows, and the segment offsets: off[q] = the
// first entry of key >= q (off[nkeys] = n), each boundary filling the gap of
// keys without entries
__global__ void k_hla_offsets(const unsigned long long *sorted, unsigned long long n,
                              unsigned long long nkeys, unsigned long long *off, uint32_t *rows) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long kc = i < n ? sorted[i] >> 32 : nkeys;
    const long long kp = i > 0 ? (long long)(sorted[i - 1] >> 32) : -1;
    for (long long q = kp + 1; q <= (long long)kc; q++) off[q] = i;
    if (i < n) rows[i] = (uint32_t)sorted[i];
  }
}

// ------------------------------------------------ narrow-window kernels
// A window of c slots is a contiguous nr x c block.  A warp covers 32 / c
// rows per iteration (lane -> (row offset, column), computed once), so all
// lanes stream consecutive words; c >= 32: one row per iteration, lanes
// striding the columns.
struct WLanes {
  uint32_t rpw, r, jj;
  bool act;
  __device__ __forceinline__ explicit WLanes(uint32_t c) {
    const uint32_t lane = threadIdx.x & 31;
    if (c >= 32) {
      rpw = 1;
      r = 0;
      jj = lane;
      act = true;
    } else {
      rpw = 32 / c;
      r = lane / c;
      jj = lane % c;
      act = r < rpw;
    }
  }
};

__global__ void __launch_bounds__(256) k_init_w(uint32_t *L, uint32_t nr, uint32_t c) {
  const WLanes wl(c);
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t row0 = warp * wl.rpw; row0 < nr; row0 += nw * wl.rpw) {
    const size_t row = row0 + wl.r;
    if (!wl.act || row >= nr) continue;
    for (uint32_t j = wl.jj; j < c; j += 32) L[row * c + j] = ROOT1;
  }
}

// compress_count for a narrow window (same contract as k_compress_count);
// WU row groups per lane loaded before any find (loads in flight together)
constexpr int WU = 4;
__global__ void __launch_bounds__(256) k_compress_w(uint32_t *L, uint32_t nr, uint32_t c,
                                                    const uint32_t *hot, unsigned long long *ctr) {
  extern __shared__ uint32_t hsm[];
  const uint32_t H = min(c, HOT_MAX);
  uint32_t *hroot = hsm, *hcnt = hsm + H;
  for (uint32_t j = threadIdx.x; j < H; j += blockDim.x) {
    hroot[j] = hot[j];
    hcnt[j] = 0;
  }
  __syncthreads();
  const WLanes wl(c);
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long nnr = 0;
  const size_t step = (size_t)wl.rpw * WU;
  for (size_t row0 = warp * step; row0 < nr; row0 += nw * step) {
    for (uint32_t j = wl.jj; j < c; j += 32) {
      uint32_t sv[WU];
#pragma unroll
      for (int u = 0; u < WU; u++) {
        const size_t v = row0 + (size_t)u * wl.rpw + wl.r;
        sv[u] = (wl.act && v < nr) ? ld_cg(L + v * c + j) : NONE;
      }
#pragma unroll
      for (int u = 0; u < WU; u++) {
        const size_t v = row0 + (size_t)u * wl.rpw + wl.r;
        const uint32_t s = sv[u];
        if (s == NONE || (s & PACIM_HIGH)) continue;  // a root (of a singleton or not)
        const uint32_t root = (j < H && s == hroot[j]) ? s : find_halve(L, c, j, s);
        if (root != s) atomicMin(L + v * c + j, root);
        nnr++;
        if (j < H && root == hroot[j]) atomicAdd(hcnt + j, 1u);
        else add_to_root(L, c, j, root, 1u);
      }
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < H; j += blockDim.x)
    if (hcnt[j]) add_to_root(L, c, j, hroot[j], hcnt[j]);
  add_count(ctr + 1, nnr);
}

// gain0 over a narrow window: acc ? gain0[v] += sum (|C| - 1) (gain0 starts
// at B) : gain0[v] = sum |C| over the window (= all slots); the lanes of one
// row are consecutive: segmented sum by shuffles; WU row groups in flight
__global__ void __launch_bounds__(256) k_gain_w(const uint32_t *__restrict__ L, uint32_t nr,
                                                uint32_t c, const uint32_t *rmap, int64_t *gain0,
                                                int acc, unsigned long long *ncc_ctr) {
  unsigned long long ncc = 0;  // roots of size >= 2: the non-singleton CCs
  const WLanes wl(c);
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t seg = c >= 32 ? 32 : c;  // lanes per row
  const size_t step = (size_t)wl.rpw * WU;
  for (size_t row0 = warp * step; row0 < nr; row0 += nw * step) {
    long long g[WU];
#pragma unroll
    for (int u = 0; u < WU; u++) g[u] = 0;
    for (uint32_t j = wl.jj; j < c; j += 32) {
      uint32_t sv[WU], sz[WU];
#pragma unroll
      for (int u = 0; u < WU; u++) {
        const size_t v = row0 + (size_t)u * wl.rpw + wl.r;
        sv[u] = (wl.act && v < nr) ? __ldcs(L + v * c + j) : NONE;
      }
#pragma unroll
      for (int u = 0; u < WU; u++) {  // root sizes of the non-roots, in flight together
        const size_t v = row0 + (size_t)u * wl.rpw + wl.r;
        const uint32_t s = sv[u];
        sz[u] = (s != NONE && !(s & PACIM_HIGH))
                    ? (__ldg(L + (size_t)s * c + j) & PACIM_LOW) : 0u;
      }
#pragma unroll
      for (int u = 0; u < WU; u++) {
        const size_t v = row0 + (size_t)u * wl.rpw + wl.r;
        const uint32_t s = sv[u];
        if (s == NONE) continue;
        const uint32_t size = (s & PACIM_HIGH) ? (s & PACIM_LOW) : sz[u];
        ncc += (s & PACIM_HIGH) && size >= 2;
        g[u] += acc ? (long long)size - 1 : (long long)size;
      }
    }
#pragma unroll
    for (int u = 0; u < WU; u++) {
      long long t = g[u];
      for (uint32_t d = 1; d < seg; d <<= 1) {
        const long long y = __shfl_down_sync(0xffffffffu, t, d);
        if (wl.jj + d < seg) t += y;
      }
      const size_t v = row0 + (size_t)u * wl.rpw + wl.r;
      if (wl.act && wl.jj == 0 && v < nr) {
        if (acc) {
          if (t) gain0[rmap[v]] += t;
        } else {
          gain0[rmap[v]] = t;
        }
      }
    }
  }
  add_count(ncc_ctr, ncc);
}

// ------------------------------------------------------ edge partition
// Per build: the upper edges grouped by the top W bits of hash(e) (their
// candidate sketches all lie in the slot bucket with the same top bits of
// hash(r); R2 candidate enumeration).  Counting pass + scatter pass; the
// order inside a bucket is arbitrary (union-find is order-independent).
__global__ void k_bucket_count(const uint64_t *keys, uint64_t m, uint64_t K, uint32_t W,
                               unsigned long long *cnt) {
  extern __shared__ unsigned long long hcnt_s[];
  const uint32_t NB = 1u << W;
  for (uint32_t i = threadIdx.x; i < NB; i += blockDim.x) hcnt_s[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(size_t)31; base < m;
       base += (size_t)gridDim.x * blockDim.x) {
    const size_t e = base + lane;
    const uint32_t b = e < m ? (uint32_t)(pc_mix64(keys[e] ^ K) >> 32) >> (32 - W) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, b);  // one shared add per bucket
    if (b != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(hcnt_s + b, (unsigned long long)__popc(peers));
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < NB; i += blockDim.x)
    if (hcnt_s[i]) atomicAdd(cnt + i, hcnt_s[i]);
}

__global__ void k_bucket_scatter(const uint64_t *keys, const uint64_t *ckeys, uint64_t m,
                                 uint64_t K, uint32_t W, unsigned long long *cur, uint64_t *okeys,
                                 uint64_t *ockeys) {
  const int lane = threadIdx.x & 31;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(size_t)31; base < m;
       base += (size_t)gridDim.x * blockDim.x) {
    const size_t e = base + lane;
    const bool ok = e < m;
    uint64_t k = 0, ck = 0;
    uint32_t b = 0xFFFFFFFFu;
    if (ok) {
      k = keys[e];
      ck = ckeys[e];
      b = (uint32_t)(pc_mix64(k ^ K) >> 32) >> (32 - W);
    }
    // one cursor update per bucket present in the warp
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    const int leader = __ffs(peers) - 1;
    unsigned long long pos = 0;
    if (ok && lane == leader) pos = atomicAdd(cur + b, (unsigned long long)__popc(peers));
    pos = __shfl_sync(peers, pos, leader) + __popc(peers & ((1u << lane) - 1));
    if (ok) {
      okeys[pos] = k;
      ockeys[pos] = ck;
    }
  }
}

// isolated vertices are singletons in every sketch: gain0 = B
__global__ void k_fill_i64(int64_t *a, uint32_t n, int64_t x) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x)
    a[v] = x;
}

}  // namespace

// ------------------------------------------------------------------ host
static float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Host slot table: this ctx's sketches sorted by hi32(hash(r)) (R2) and the
// candidate bucket table of k_edges; uploaded once per build.
void pc_slot_table(pacim_ctx *ctx) {
  const uint32_t B = ctx->R_local;
  ctx->slot_r.clear();
  ctx->r_slot.assign(ctx->R, -1);
  std::vector<std::pair<uint64_t, uint32_t>> hs;
  for (uint32_t r = ctx->rank; r < ctx->R; r += ctx->world) {
    uint64_t h = pc_mix64(((1ull << 63) | (uint64_t)r) ^ ctx->K);
    hs.push_back({h, r});
  }
  std::sort(hs.begin(), hs.end(),
            [](const std::pair<uint64_t, uint32_t> &a, const std::pair<uint64_t, uint32_t> &b) {
              return (a.first >> 32) != (b.first >> 32) ? (a.first >> 32) < (b.first >> 32)
                                                        : a.second < b.second;
            });
  ctx->shr.resize(B);
  ctx->hr64.resize(B);
  ctx->slot_r.resize(B);
  for (uint32_t j = 0; j < B; j++) {
    ctx->shr[j] = (uint32_t)(hs[j].first >> 32);
    ctx->hr64[j] = hs[j].first;
    ctx->slot_r[j] = hs[j].second;
    ctx->r_slot[hs[j].second] = (int32_t)j;
  }
  const uint32_t NT = 1u << PACIM_TB;
  ctx->tab.assign(NT + 1, 0);
  uint32_t j = 0;
  for (uint32_t p = 0; p <= NT; p++) {
    while (j < B && (ctx->shr[j] >> (32 - PACIM_TB)) < p) j++;
    ctx->tab[p] = (uint16_t)j;
  }
  pc_ensure(ctx, ctx->d_shr, B * sizeof(uint32_t));
  pc_ensure(ctx, ctx->d_tab, (NT + 1) * sizeof(uint16_t));
  PC_CUDA(cudaMemcpyAsync(ctx->d_shr.p, ctx->shr.data(), B * 4, cudaMemcpyHostToDevice,
                          ctx->stream));
  PC_CUDA(cudaMemcpyAsync(ctx->d_tab.p, ctx->tab.data(), (NT + 1) * 2, cudaMemcpyHostToDevice,
                          ctx->stream));
  pc_ensure(ctx, ctx->d_hr64, B * sizeof(uint64_t));
  PC_CUDA(cudaMemcpyAsync(ctx->d_hr64.p, ctx->hr64.data(), B * 8, cudaMemcpyHostToDevice,
                          ctx->stream));
}

// One sketch pass over the edge list for slots [j0, j0+Bb): parent arrays in
// ---------------------------------------------------------------- HLA
bool pc_hla_begin(pacim_ctx *ctx, Hla *hla, double max_per_edge) {
  ctx->hla_ok = false;
  // (HLA recording reads the edge lists' hub flags: not when the build
  // streams the upper edges and the lists were not derived — c5)
  if (ctx->nhub == 0 || ctx->lean || (ctx->ucsr && !ctx->elist_ok)) return false;
  const uint32_t B = ctx->R_local;
  // expected live (hub, slot, neighbour) entries: every CSR entry of a hub is
  // live in a slot with its edge probability — p (constant), the mean of
  // U(lo, hi) (R19); WIC (R4): sum over a hub's entries of 2/(d_u + d_w),
  // at most 2 and measured 0.9-1.2 per (hub, slot) on c4: 1.25 (the cap adds
  // another 25 %)
  double E;
  if (ctx->pmodel == PACIM_P_WIC) {
    E = 1.25 * ctx->nhub * B;
  } else {
    double p = (double)ctx->t32 / 4294967296.0;
    if (ctx->pmodel == PACIM_P_UNIFORM)
      p = 0.5 * ((double)(ctx->t32 >> 32) + (double)(ctx->t32 & 0xFFFFFFFFull)) / 4294967296.0;
    E = std::min(p, 1.0) * (double)ctx->hub_entries * B;
  }
  if (E > max_per_edge * (double)ctx->m) return false;  // recording would cost more than it saves
  const unsigned long long cap = (unsigned long long)(1.25 * E) + (1ull << 20);
  const size_t keys = (size_t)ctx->nhub * B + 1;
  if (keys >= (1ull << 32)) return false;  // key field of an entry is 32 bits
  size_t fr = 0, tot = 0;
  pc_mem_info(ctx, &fr, &tot);
  // raw + the sort's second buffer (8 B each), grouped rows (4 B), offsets
  const size_t need = (cap + 1) * 20 + keys * 8 + (64ull << 20);
  if (need > fr / 4 && ctx->Ltmp.bytes) {
    // a compressed build's batch buffer kept from the previous build: release
    // it (the batch is sized after the HLA) rather than build without the HLA
    pc_free(ctx, ctx->Ltmp);
    pc_mem_info(ctx, &fr, &tot);
  }
  if (need > fr / 4) return false;
  pc_ensure(ctx, ctx->hla_raw, (cap + 1) * 8);
  PC_CUDA(cudaMemsetAsync(ctx->hla_raw.p, 0, 8, ctx->stream));
  hla->tab = ctx->hub_tab.as<unsigned long long>();
  hla->mask = ctx->hub_mask;
  hla->n = ctx->hla_raw.as<unsigned long long>();
  hla->raw = hla->n + 1;
  hla->cap = cap;
  hla->B = B;
  return true;
}

void pc_hla_finish(pacim_ctx *ctx, Hla *hla) {
  // sort the entries by key (the bits above the row), then rows + offsets
  const unsigned long long nkeys = (unsigned long long)ctx->nhub * ctx->R_local;
  unsigned long long nraw = 0;
  PC_CUDA(cudaMemcpyAsync(&nraw, hla->n, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (nraw <= hla->cap) {
    int kb = 1;
    while (kb < 32 && (nkeys >> kb)) kb++;
    TmpBuf alt(ctx), tmp(ctx);
    pc_ensure(ctx, alt, std::max<size_t>(nraw, 1) * 8);
    cub::DoubleBuffer<unsigned long long> db(hla->raw, alt.as<unsigned long long>());
    size_t tb = 0;
    PC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)nraw, 32, 32 + kb, ctx->stream));
    pc_ensure(ctx, tmp, std::max<size_t>(tb, 1));
    PC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, (int64_t)nraw, 32, 32 + kb, ctx->stream));
    pc_ensure(ctx, ctx->hla_off, (nkeys + 1) * 8);
    pc_ensure(ctx, ctx->hla_row, std::max<size_t>(nraw, 1) * 4);
    k_hla_offsets<<<pc_grid(ctx, nraw + 1, 256), 256, 0, ctx->stream>>>(
        db.Current(), nraw, nkeys, ctx->hla_off.as<unsigned long long>(), ctx->hla_row.as<uint32_t>());
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->hla_ok = true;
    ctx->hla_n = nraw;
    ctx->launches += 2;
  }
  pc_free(ctx, ctx->hla_raw);  // scratch
}

// The zeroed chunk counter and chunk size of one k_edges launch over
// `items` edges (CSR entries for lean graphs) with `grid` blocks: ~16 chunks
// per warp, at least 4 iterations each (one counter add per chunk)
static EdgeWork edge_work(pacim_ctx *ctx, uint64_t items, unsigned grid) {
  pc_ensure(ctx, ctx->edge_work, 64);
  EdgeWork w;
  w.ctr = ctx->edge_work.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(w.ctr, 0, 8, ctx->stream));
  const uint64_t niter = (items + 31) / 32, warps = (uint64_t)grid * (EDGE_THREADS / 32);
  w.citer = (uint32_t)std::max<uint64_t>(4, std::min<uint64_t>(niter / (warps * 16) + 1, 1u << 20));
  return w;
}

// Lb (rows x Bb), unions, full compression and CC sizes (root slot HIGH|size).
// ctr[1] += non-roots, ctr[4] += live pairs (ctr[0], the non-singleton CCs:
// the gain pass that follows).
// ev (optional, 3 events) is recorded after init, edges and compress.
void pc_sketch_pass(pacim_ctx *ctx, uint32_t *Lb, uint32_t j0, uint32_t Bb,
                    unsigned long long *ctr, cudaEvent_t *ev, const Hla *hla_in,
                    const EdgeSet *es_in) {
  Hla hla{};
  if (hla_in) hla = *hla_in;
  EdgeSet es;
  if (es_in) {
    es = *es_in;
  } else {
    es.m = ctx->m;  // the edge lists, if used, below
  }
  const uint32_t n = ctx->nr, B = ctx->R_local;
  const bool ep_on = ctx->ep.mask != 0;  // slot epochs (pc_build)
  const uint32_t NT = 1u << PACIM_TB;
  pc_ensure(ctx, ctx->d_hot, 2 * (size_t)B * sizeof(uint32_t));
  uint32_t *hot_root = ctx->d_hot.as<uint32_t>();
  const uint32_t H = std::min<uint32_t>(Bb, HOT_MAX);
  const unsigned rows_grid = pc_grid(ctx, (size_t)n * 32, 256, 16);
  const bool narrow = Bb < NARROW_W;  // lanes over (row, slot) pairs
  const unsigned wgrid = pc_grid(ctx, (size_t)n * Bb, 256, 16);
  if (ctx->skip_init) {
    // slot epochs (pc_build): the stale slots of earlier builds read as roots
  } else if (narrow) {
    k_init_w<<<wgrid, 256, 0, ctx->stream>>>(Lb, n, Bb);
  } else {
    k_init<<<rows_grid, 256, 0, ctx->stream>>>(Lb, n, Bb);
  }
  PC_CHECK_LAUNCH();
  if (ev) PC_CUDA(cudaEventRecord(ev[0], ctx->stream));
  // the hook list of an epoch build (k_edges records every successful hook,
  // k_compress_count<…, LIST> reads it): capacity from the non-root count of
  // the last dense build of this graph (+ chunk holes); an overflow makes the
  // compression stream the store (decided on the device).  PACIM_HOOKLIST =
  // 0: off; > 1: that capacity (tests)
  // compacted finds unless the store is dense in non-roots: expected live
  // (row, slot) pairs per row 2 m p / rows >= 1.5 (c3: 2.3; c2: 0.84; WIC:
  // small p on most edges)
  double p = (double)ctx->t32 / 4294967296.0;
  if (ctx->pmodel == PACIM_P_UNIFORM)
    p = 0.5 * ((double)(ctx->t32 >> 32) + (double)(ctx->t32 & 0xFFFFFFFFull)) / 4294967296.0;
  const bool dense = ctx->pmodel != PACIM_P_WIC && 2.0 * ctx->m * p >= 1.5 * std::max(n, 1u);
  PairList hk{};
  ctx->hk_cap = 0;
  {
    const long long env = getenv("PACIM_HOOKLIST") ? atoll(getenv("PACIM_HOOKLIST")) : 1;
    const bool known = ctx->hk_gen == ctx->hint_gen && ctx->hk_B == Bb;
    if (ep_on && !dense && !narrow && env != 0 && Bb <= 256 && j0 == 0 && n < (1u << 28) && (known || env > 1)) {
      unsigned long long cap = env > 1 ? (unsigned long long)env
                                       : ctx->hk_hint + ctx->hk_hint / 8 + (1ull << 24);
      if (ctx->hk_list.bytes < cap * 8 || ctx->hk_list.bytes > 2 * cap * 8 + (64ull << 20)) {
        pc_free(ctx, ctx->hk_list);
        if (pc_mem_free(ctx) > cap * 8 + (2ull << 30)) pc_ensure(ctx, ctx->hk_list, cap * 8);
      }
      if (ctx->hk_list.bytes >= cap * 8) {
        hk.p = ctx->hk_list.as<unsigned long long>();
        hk.cnt = ctr + 20;
        hk.cap = cap;
        ctx->hk_cap = cap;
      }
    }
  }
  {
    size_t smem = B * sizeof(uint32_t) + (NT + 1) * sizeof(uint16_t);
    unsigned g = pc_grid(ctx, (es.m + 31) / 32 * 32, EDGE_THREADS, PACIM_EDGE_BLOCKS);
    // graphs loaded with the upper-edge stream (derive_edges): the dense
    // store's one-window builds without HLA recording read it
    const bool ucsr = ctx->ucsr && !ctx->lean && !es_in && !hla.raw;
    if (!ctx->lean && !ucsr) {
      pc_ensure_edge_lists(ctx);
      if (!es_in) {
        es.keys = ctx->keys.as<uint64_t>();
        es.ckeys = ctx->ckeys.as<uint64_t>();
      }
    }
    UpperCsr uc;
    if (ucsr && ctx->ucsr_direct) {
      uc.nv = ctx->n;
      uc.off = ctx->off.as<uint64_t>();
      uc.nbr = ctx->upper_src ? nullptr : ctx->nbr.as<uint32_t>();
      uc.unbr = ctx->upper_src ? ctx->unbr.as<uint32_t>() : nullptr;
      uc.uoff = ctx->uoff.as<uint64_t>();
      uc.ucrow = ctx->ucrow.as<uint32_t>();
      uc.rk = ctx->rk.as<uint2>();
    } else if (ucsr) {
      uc.nv = ctx->n;
      uc.uoff = ctx->uoff.as<uint64_t>();
      uc.unbr = ctx->unbr.as<uint32_t>();
      uc.ud16 = ctx->ud16.as<uint16_t>();
      uc.ucrowr = ctx->ucrowr.as<uint32_t>();
      uc.uvrow = ctx->uvrow.p ? ctx->uvrow.as<uint32_t>() : nullptr;
      uc.ucrow = ctx->ucrow.as<uint32_t>();
      uc.rk = ctx->rk.as<uint2>();
    }
    if (ucsr && ctx->ucsr_direct) {
      const bool pe = ctx->pmodel != PACIM_P_CONST;
      auto kern = ctx->hash_rule
                      ? (pe ? (ep_on ? k_edges<true, false, true, 4, 0, true> : k_edges<true, false, true, 4>)
                            : (ep_on ? k_edges<false, false, true, 4, 0, true> : k_edges<false, false, true, 4>))
                      : (pe ? (ep_on ? k_edges<true, false, false, 4, 0, true> : k_edges<true, false, false, 4>)
                            : (ep_on ? k_edges<false, false, false, 4, 0, true> : k_edges<false, false, false, 4>));
      PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
          nullptr, nullptr, pe ? ctx->tm1.as<uint32_t>() : nullptr, ctx->m, ctx->K,
          pe ? ctx->toff() : ctx->t32, ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(), B, j0, Bb, Lb,
          ctr + 4, Hla{}, ctx->d_hr64.as<uint64_t>(), nullptr, 0u, hk, ctx->ep,
          edge_work(ctx, ctx->m, g), uc);
    } else if (ucsr) {
      const bool pe = ctx->pmodel != PACIM_P_CONST;
      auto kern = ctx->hash_rule
                      ? (pe ? (ep_on ? k_edges<true, false, true, 2, 0, true> : k_edges<true, false, true, 2>)
                            : (ep_on ? k_edges<false, false, true, 2, 0, true> : k_edges<false, false, true, 2>))
                      : (pe ? (ep_on ? k_edges<true, false, false, 2, 0, true> : k_edges<true, false, false, 2>)
                            : (ep_on ? k_edges<false, false, false, 2, 0, true> : k_edges<false, false, false, 2>));
      PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
          nullptr, nullptr, pe ? ctx->tm1.as<uint32_t>() : nullptr, ctx->m, ctx->K,
          pe ? ctx->toff() : ctx->t32, ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(), B, j0, Bb, Lb,
          ctr + 4, Hla{}, ctx->d_hr64.as<uint64_t>(), nullptr, 0u, hk, ctx->ep,
          edge_work(ctx, ctx->m, g), uc);
    } else if (ctx->lean && ctx->uoff.p && (!getenv("PACIM_LEAN_UPPER") || atoi(getenv("PACIM_LEAN_UPPER")) != 0)) {
      // no edge list (c5): the upper entries of the CSR by the upper offsets
      // (half the lanes of the full-CSR pass below, which drops the lower ones)
      auto kern = ctx->hash_rule ? (ep_on ? k_edges<false, false, true, 3, 0, true> : k_edges<false, false, true, 3>) : (ep_on ? k_edges<false, false, false, 3, 0, true> : k_edges<false, false, false, 3>);
      PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      UpperCsr ul;
      ul.nv = ctx->n;
      ul.uoff = ctx->uoff.as<uint64_t>();
      const unsigned gl = pc_grid(ctx, (ctx->m + 31) / 32 * 32, EDGE_THREADS, PACIM_EDGE_BLOCKS);
      kern<<<gl, EDGE_THREADS, smem, ctx->stream>>>(
          ctx->off.as<uint64_t>(), reinterpret_cast<const uint64_t *>(ctx->nbr.p),
          ctx->ucrow.as<uint32_t>(), ctx->m, ctx->K, ctx->t32, ctx->d_shr.as<uint32_t>(),
          ctx->d_tab.as<uint16_t>(), B, j0, Bb, Lb, ctr + 4, Hla{}, ctx->d_hr64.as<uint64_t>(), nullptr, 0u, hk, ctx->ep,
          edge_work(ctx, ctx->m, gl), ul);
    } else if (ctx->lean) {  // no edge list: the upper edges from the CSR (c5)
      auto kern = ctx->hash_rule ? (ep_on ? k_edges<false, false, true, true, 0, true> : k_edges<false, false, true, true>) : (ep_on ? k_edges<false, false, false, true, 0, true> : k_edges<false, false, false, true>);
      PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const uint64_t nnz = 2 * ctx->m;
      const unsigned gl = pc_grid(ctx, (nnz + 31) / 32 * 32, EDGE_THREADS, PACIM_EDGE_BLOCKS);
      kern<<<gl, EDGE_THREADS, smem, ctx->stream>>>(
          ctx->off.as<uint64_t>(), reinterpret_cast<const uint64_t *>(ctx->nbr.p),
          ctx->crow.as<uint32_t>(), nnz, ctx->K, ctx->t32, ctx->d_shr.as<uint32_t>(),
          ctx->d_tab.as<uint16_t>(), B, j0, Bb, Lb, ctr + 4, Hla{}, ctx->d_hr64.as<uint64_t>(), nullptr, 0u, hk, ctx->ep,
          edge_work(ctx, nnz, gl), UpperCsr{ctx->n});
    } else if (ctx->pmodel != PACIM_P_CONST) {  // per-edge thresholds (WIC, Uniform)
      auto kern = ctx->hash_rule ? (hla.raw ? (ep_on ? k_edges<true, true, true, false, 0, true> : k_edges<true, true, true, false>) : (ep_on ? k_edges<true, false, true, false, 0, true> : k_edges<true, false, true, false>))
                                 : (hla.raw ? (ep_on ? k_edges<true, true, false, false, 0, true> : k_edges<true, true, false, false>) : (ep_on ? k_edges<true, false, false, false, 0, true> : k_edges<true, false, false, false>));
      PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
          es.keys, es.ckeys, ctx->tm1.as<uint32_t>(), es.m,
          ctx->K, ctx->toff(), ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(), B, j0, Bb, Lb, ctr + 4, hla,
          ctx->d_hr64.as<uint64_t>(), nullptr, 0u, hk, ctx->ep, edge_work(ctx, es.m, g), UpperCsr{});
    } else {
      auto kern = ctx->hash_rule ? (hla.raw ? (ep_on ? k_edges<false, true, true, false, 0, true> : k_edges<false, true, true, false>) : (ep_on ? k_edges<false, false, true, false, 0, true> : k_edges<false, false, true, false>))
                                 : (hla.raw ? (ep_on ? k_edges<false, true, false, false, 0, true> : k_edges<false, true, false, false>) : (ep_on ? k_edges<false, false, false, false, 0, true> : k_edges<false, false, false, false>));
      PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
          es.keys, es.ckeys, nullptr, es.m, ctx->K, ctx->t32,
          ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(), B, j0, Bb, Lb, ctr + 4, hla,
          ctx->d_hr64.as<uint64_t>(), nullptr, 0u, hk, ctx->ep, edge_work(ctx, es.m, g), UpperCsr{});
    }
    PC_CHECK_LAUNCH();
  }
  if (ev) PC_CUDA(cudaEventRecord(ev[1], ctx->stream));
  k_hot_roots<<<(Bb + 255) / 256, 256, 0, ctx->stream>>>(Lb, n, Bb, ctx->hub_row, hot_root, ctx->ep);
  PC_CHECK_LAUNCH();
  if (narrow)
    k_compress_w<<<wgrid, 256, 2 * H * sizeof(uint32_t), ctx->stream>>>(Lb, n, Bb, hot_root, ctr);
  else
  {
    // grid-stride kernels: one full wave of resident blocks (pc_grid_occ)
    const size_t csm = 2 * H * sizeof(uint32_t);
    if (dense) {
      auto kc = ctx->ep.mask ? k_compress_count<false, true> : k_compress_count<false, false>;
      kc<<<pc_grid_occ(ctx, kc, (size_t)n * 32, 256, csm), 256, csm, ctx->stream>>>(
          Lb, n, Bb, hot_root, ctr, ctx->ep, nullptr, nullptr, 0);
    } else if (hk.p) {
      auto kl = k_compress_list<true>;
      PC_CUDA(cudaMemsetAsync(ctr + 21, 0, 8, ctx->stream));
      kl<<<pc_grid_occ(ctx, kl, (size_t)n * 32, 256, csm), 256, csm, ctx->stream>>>(
          Lb, Bb, hot_root, ctr, ctx->ep, hk.p, hk.cnt, hk.cap, ctr + 21);
      auto kc = k_compress_count<true, true, true>;  // only if the list overflowed
      kc<<<pc_grid_occ(ctx, kc, (size_t)n * 32, 256, csm), 256, csm, ctx->stream>>>(
          Lb, n, Bb, hot_root, ctr, ctx->ep, hk.p, hk.cnt, hk.cap);
    } else {
      auto kc = ctx->ep.mask ? k_compress_count<true, true> : k_compress_count<true, false>;
      kc<<<pc_grid_occ(ctx, kc, (size_t)n * 32, 256, csm), 256, csm, ctx->stream>>>(
          Lb, n, Bb, hot_root, ctr, ctx->ep, nullptr, nullptr, 0);
    }
  }
  PC_CHECK_LAUNCH();
  if (ev) PC_CUDA(cudaEventRecord(ev[2], ctx->stream));
  ctx->launches += 4;
}

// The union pass over the compact store (store_cs.cu): every upper edge,
// its live sketches, unions of the flat entries in P.  ctr[4] += live pairs.
template <int MODE>
static void cs_edges(pacim_ctx *ctx, uint32_t *L, const uint2 *rec, uint32_t MW,
                     unsigned long long *ctr, PairList pl = PairList{}) {
  const uint32_t B = ctx->R_local;
  const uint32_t NT = 1u << PACIM_TB;
  const size_t smem = B * sizeof(uint32_t) + (NT + 1) * sizeof(uint16_t);
  if (ctx->lean) {
    auto kern = ctx->hash_rule ? k_edges<false, false, true, true, MODE>
                               : k_edges<false, false, false, true, MODE>;
    PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint64_t nnz = 2 * ctx->m;
    const unsigned gl = pc_grid(ctx, (nnz + 31) / 32 * 32, EDGE_THREADS, PACIM_EDGE_BLOCKS);
    kern<<<gl, EDGE_THREADS, smem, ctx->stream>>>(
        ctx->off.as<uint64_t>(), reinterpret_cast<const uint64_t *>(ctx->nbr.p),
        ctx->crow.as<uint32_t>(), nnz, ctx->K, ctx->t32, ctx->d_shr.as<uint32_t>(),
        ctx->d_tab.as<uint16_t>(), B, 0, B, L, ctr + 4, Hla{}, ctx->d_hr64.as<uint64_t>(), rec, MW, pl, Ep{},
        edge_work(ctx, nnz, gl), UpperCsr{ctx->n});
  } else if (ctx->ucsr && !ctx->elist_ok) {
    // the upper-edge stream's CSR-direct form (no edge lists derived)
    const bool pe = ctx->pmodel != PACIM_P_CONST;
    auto kern = pe ? (ctx->hash_rule ? k_edges<true, false, true, 4, MODE>
                                     : k_edges<true, false, false, 4, MODE>)
                   : (ctx->hash_rule ? k_edges<false, false, true, 4, MODE>
                                     : k_edges<false, false, false, 4, MODE>);
    PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PC_REQUIRE(ctx->rk.p && ctx->ucrow.p, PACIM_ESTATE, "upper-edge stream tables missing");
    UpperCsr uc;
    uc.nv = ctx->n;
    uc.off = ctx->off.as<uint64_t>();
    uc.nbr = ctx->upper_src ? nullptr : ctx->nbr.as<uint32_t>();
    uc.unbr = ctx->upper_src ? ctx->unbr.as<uint32_t>() : nullptr;
    uc.uoff = ctx->uoff.as<uint64_t>();
    uc.ucrow = ctx->ucrow.as<uint32_t>();
    uc.rk = ctx->rk.as<uint2>();
    const unsigned g = pc_grid(ctx, (ctx->m + 31) / 32 * 32, EDGE_THREADS, PACIM_EDGE_BLOCKS);
    kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
        nullptr, nullptr, pe ? ctx->tm1.as<uint32_t>() : nullptr, ctx->m, ctx->K,
        pe ? ctx->toff() : ctx->t32, ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(), B, 0, B, L,
        ctr + 4, Hla{}, ctx->d_hr64.as<uint64_t>(), rec, MW, pl, Ep{}, edge_work(ctx, ctx->m, g), uc);
  } else {
    pc_ensure_edge_lists(ctx);
    const bool pe = ctx->pmodel != PACIM_P_CONST;
    auto kern = pe ? (ctx->hash_rule ? k_edges<true, false, true, false, MODE>
                                     : k_edges<true, false, false, false, MODE>)
                   : (ctx->hash_rule ? k_edges<false, false, true, false, MODE>
                                     : k_edges<false, false, false, false, MODE>);
    PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned g = pc_grid(ctx, (ctx->m + 31) / 32 * 32, EDGE_THREADS, PACIM_EDGE_BLOCKS);
    kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
        ctx->keys.as<uint64_t>(), ctx->ckeys.as<uint64_t>(),
        pe ? ctx->tm1.as<uint32_t>() : nullptr, ctx->m, ctx->K, pe ? ctx->toff() : ctx->t32,
        ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(), B, 0, B, L, ctr + 4, Hla{},
        ctx->d_hr64.as<uint64_t>(), rec, MW, pl, Ep{}, edge_work(ctx, ctx->m, g), UpperCsr{});
  }
  PC_CHECK_LAUNCH();
  ctx->launches++;
}

// The union pass over the compact store (store_cs.cu): every upper edge,
// its live sketches, unions of the entries' P words.  ctr[4] += live pairs.
void pc_cs_edges(pacim_ctx *ctx, uint32_t *E, const uint2 *rec, uint32_t MW,
                 unsigned long long *ctr) {
  cs_edges<1>(ctx, E, rec, MW, ctr);
}

// The mask pass over the upper edges: the live slots of every edge set in
// both endpoints' row masks (rec.y words).  ctr[5] += live pairs.  With a
// pair list (plist != null) the live pairs are also written there, in chunks
// of PL_CHUNK entries reserved per warp (*pcnt = the slots reserved, holes
// ~0; entries at or past cap are dropped: *pcnt > cap means overflow).
void pc_cs_mask_edges(pacim_ctx *ctx, uint32_t *rec_words, uint32_t MW, unsigned long long *ctr,
                      unsigned long long *plist, unsigned long long *pcnt, unsigned long long cap) {
  PairList pl;
  pl.p = plist;
  pl.cnt = pcnt;
  pl.cap = cap;
  cs_edges<2>(ctx, rec_words, nullptr, MW, ctr + 1, pl);
}

// The edge-partitioned pass of a sharded compact build (dist.cu): the upper
// edges [e0, e1) against all R sketches (the global sorted slot table
// d_shr_all / d_tab_all), every live (edge, global slot) into the pair list
// (PL_CHUNK chunks per warp; *pcnt = slots reserved).  ctr[4] += live pairs.
void pc_ep_edges(pacim_ctx *ctx, uint64_t e0, uint64_t e1, const uint32_t *d_shr_all,
                 const uint16_t *d_tab_all, uint32_t R, unsigned long long *plist,
                 unsigned long long *pcnt, unsigned long long cap, unsigned long long *ctr) {
  PC_REQUIRE(!ctx->lean && !ctx->hash_rule && R <= 256, PACIM_ENOTIMPL,
             "edge-partitioned build: edge lists, rule R2, R <= 256");
  if (e1 <= e0) return;
  pc_ensure_edge_lists(ctx);
  PairList pl;
  pl.p = plist;
  pl.cnt = pcnt;
  pl.cap = cap;
  const uint32_t NT = 1u << PACIM_TB;
  const size_t smem = R * sizeof(uint32_t) + (NT + 1) * sizeof(uint16_t);
  const bool pe = ctx->pmodel != PACIM_P_CONST;
  auto kern = pe ? k_edges<true, false, false, false, 3> : k_edges<false, false, false, false, 3>;
  PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const uint64_t m = e1 - e0;
  const unsigned g = pc_grid(ctx, (m + 31) / 32 * 32, EDGE_THREADS, PACIM_EDGE_BLOCKS);
  kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
      ctx->keys.as<uint64_t>() + e0, ctx->ckeys.as<uint64_t>() + e0,
      pe ? ctx->tm1.as<uint32_t>() + e0 : nullptr, m, ctx->K, pe ? ctx->toff() : ctx->t32, d_shr_all,
      d_tab_all, R, 0, R, nullptr, ctr + 4, Hla{}, nullptr, nullptr, 0u, pl, Ep{}, edge_work(ctx, m, g), UpperCsr{});
  PC_CHECK_LAUNCH();
  ctx->launches++;
}

namespace {
// the union pass from the mask pass's pair list: no edge is read or hashed
// again (H2, H3 on the recorded live pairs)
__global__ void __launch_bounds__(256) k_cs_list_unite(uint32_t *E, const uint2 *__restrict__ rec,
                                                       uint32_t MW,
                                                       const unsigned long long *__restrict__ pl,
                                                       unsigned long long cnt,
                                                       unsigned long long *live_ctr,
                                                       const unsigned long long *mask_live) {
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(live_ctr, *mask_live);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long x = pl[i];
    if (x == ~0ull) continue;  // a hole of a warp's chunk
    const uint32_t u = (uint32_t)(x >> 36), v = (uint32_t)(x >> 8) & 0x0FFFFFFFu, j = (uint32_t)x & 255u;
    uf_unite(E, 2, 0, pc_cs_pos(rec, MW, u, j), pc_cs_pos(rec, MW, v, j));
  }
}
}  // namespace

void pc_cs_list_unite(pacim_ctx *ctx, uint32_t *E, const uint2 *rec, uint32_t MW,
                      const unsigned long long *plist, unsigned long long cnt,
                      unsigned long long *ctr, const unsigned long long *mask_live) {
  k_cs_list_unite<<<pc_grid(ctx, cnt, 256, 8), 256, 0, ctx->stream>>>(E, rec, MW, plist, cnt, ctr + 4,
                                                                     mask_live);
  PC_CHECK_LAUNCH();
  ctx->launches++;
}

// Slot windows of the store for this build.  With a constant
// threshold the live sketches of an edge all lie in the bucket of slots whose
// top w = clz(T - 1) bits of hash(r) equal those of hash(e); the slots are
// sorted by hash(r), so every bucket is a contiguous slot range.  When a
// bucket's parent arrays (rows x slots x 4 B) fit the L2 budget, the build
// runs one window (a bucket, or a slice of an oversized one) at a time over
// that bucket's edges only: the unions, compression and CC counting of a
// window hit L2 instead of HBM.  Otherwise (WIC thresholds, or rows too
// many) one window [0, B) over all edges.  Returns the bucket bits W (0: one
// window).
static uint32_t plan_windows(pacim_ctx *ctx) {
  const uint32_t B = ctx->R_local, nr = ctx->nr;
  ctx->win_first.assign({0u, B});
  // opt-in (PACIM_L2_BUDGET = bytes of parent arrays per window): measured on
  // c2 (profiles/r01_v7_windows.md) the windows do not stay L2-resident and
  // 35 windows x 4 short kernels cost more than they save, so the default is
  // the single window [0, B)
  uint64_t budget = 0;
  if (const char *e = getenv("PACIM_L2_BUDGET")) budget = (uint64_t)atoll(e);
  if (ctx->pmodel != PACIM_P_CONST || ctx->hash_rule != 0 || ctx->lean || ctx->t32 < 2 ||
      ctx->t32 >= (1ull << 32) || nr == 0 ||
      budget == 0 || ctx->compressed)
    return 0;
  const uint32_t w = __builtin_clz((uint32_t)(ctx->t32 - 1));
  const uint64_t g = budget / ((uint64_t)nr * 4);  // slots per window that fit the budget
  if (g >= B || g < 1) return 0;                   // everything fits, or nothing does
  uint32_t W = std::min<uint32_t>(w, 10);
  if (W == 0) return 0;
  // windows: each bucket split into slices of <= g slots
  std::vector<uint32_t> wf;
  uint32_t j = 0;
  for (uint32_t b = 0; b < (1u << W); b++) {
    uint32_t e = j;
    while (e < B && (ctx->shr[e] >> (32 - W)) == b) e++;
    for (uint32_t f = j; f < e; f += (uint32_t)g) wf.push_back(f);
    j = e;
  }
  wf.push_back(B);
  if (wf.size() <= 2) return 0;
  ctx->win_first = wf;
  return W;
}

__global__ void k_fill_smap(const uint32_t *wf, uint32_t nw, uint32_t *smap) {
  for (uint32_t w = blockIdx.x; w < nw; w += gridDim.x)
    for (uint32_t j = wf[w] + threadIdx.x; j < wf[w + 1]; j += blockDim.x)
      smap[j] = (wf[w] << 16) | (wf[w + 1] - wf[w]);
}

static double host_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void pc_build(pacim_ctx *ctx) {
  const bool htime = getenv("PACIM_HOST_TIMING") != nullptr;  // diagnostics: host phases to stderr
  double h0 = htime ? host_ms() : 0, h1 = 0, h2 = 0, h3 = 0;
  const uint32_t n = ctx->nr, B = ctx->R_local;  // store rows = non-isolated vertices
  PC_REQUIRE(B >= 1 && B <= 65535, PACIM_EINVAL, "local sketch count must be in [1, 65535]");
  PC_REQUIRE(!ctx->compressed, PACIM_ENOTIMPL, "compressed store not built by pc_build");
  // the compact store (store_cs.cu) unless the sketches are dense (c3) or the
  // dense layout is asked for (PACIM_STORE=dense)
  ctx->stats.build_hook_list = 0;
  ctx->hk_cap = 0;
  if (pc_cs_build(ctx)) return;
  pc_cs_free(ctx);
  pc_slot_table(ctx);
  // a compressed store of an earlier build is released first (capacity for
  // this one: at c4 the two do not fit together)
  for (DevBuf *d : {&ctx->clabel, &ctx->csz, &ctx->csz_work, &ctx->Ltmp, &ctx->cwork,
                    &ctx->hla_off, &ctx->hla_row, &ctx->hla_raw})
    pc_free(ctx, *d);
  ctx->hla_ok = false;
  const bool want_hla = (getenv("PACIM_HLA") != nullptr || getenv("PACIM_FORCE_HLA") != nullptr);
  const uint32_t W = plan_windows(ctx);
  const uint32_t nwin = (uint32_t)ctx->win_first.size() - 1;
  const bool fresh = !ctx->L.p || ctx->L.bytes < (size_t)n * B * sizeof(uint32_t);
  pc_ensure(ctx, ctx->L, (size_t)n * B * sizeof(uint32_t));
  // slot epochs (Ep, pacim_internal.cuh): no reset pass over the store in
  // this build unless the epoch count wraps (every 2^bits builds), the store
  // is new, or an earlier build reset it without epochs (slot windows,
  // narrow slot counts, HLA recording: their kernels read slots as stored).
  // The epoch field takes the bits between the largest id / size (<= rows)
  // and COV (bit 30), at most 6 (PACIM_EPOCH_BITS caps it; 0: off)
  {
    const int idbits = 32 - __builtin_clz(std::max(n, 1u));
    int eb = std::min(6, 30 - idbits);
    const char *eb_env = getenv("PACIM_EPOCH_BITS");
    if (eb_env) eb = std::min(eb, atoi(eb_env));
    // worth it when the reset is large against the unions: the epoch tests
    // cost ~4 ps per live pair in the union, compression and gain passes,
    // the reset ~0.6 ps per slot (c4: 9.3 G slots, 0.54 G pairs: -5.3 ms
    // reset, +2.1 ms; c2: 0.6 G slots, 0.33 G pairs and c3: 4.3 G slots,
    // 4.9 G pairs lose); judged on the last dense build of this graph
    const bool worth = eb_env ? true
                              : ctx->ep_live_gen == ctx->hint_gen &&
                                    (double)n * B > 7.0 * ctx->ep_live_per_slot * B;
    const bool on = eb >= 1 && nwin == 1 && B >= NARROW_W && !want_hla && worth;
    if (!on) {
      ctx->ep = Ep{};
      ctx->ep_clean = false;
      ctx->skip_init = false;
    } else {
      const bool cont = !fresh && ctx->ep_clean && ctx->ep_bits == (uint32_t)eb &&
                        ctx->ep_store == ctx->L.p && ctx->ep_nr == n && ctx->ep_B == B &&
                        ctx->ep_cur + 1 < (1u << eb);
      ctx->ep_cur = cont ? ctx->ep_cur + 1 : 0;  // 0: a full reset writes HIGH | 1 (epoch 0)
      ctx->skip_init = cont;
      ctx->ep_bits = (uint32_t)eb;
      ctx->ep_clean = true;
      ctx->ep_store = ctx->L.p;
      ctx->ep_nr = n;
      ctx->ep_B = B;
      const uint32_t sh = 30 - (uint32_t)eb;
      ctx->ep.tag = ctx->ep_cur << sh;
      ctx->ep.mask = ((1u << eb) - 1) << sh;
    }
  }
  const bool ep_on = ctx->ep.mask != 0;
  pc_ensure(ctx, ctx->gain0, (size_t)ctx->n * sizeof(int64_t));
  pc_ensure(ctx, ctx->counters, 64 * sizeof(uint64_t));
  unsigned long long *ctr = ctx->counters.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(ctr, 0, 64 * sizeof(uint64_t), ctx->stream));
  uint32_t *L = ctx->L.as<uint32_t>();
  ctx->launches = 0;
  const unsigned rows_grid = pc_grid(ctx, (size_t)n * 32, 256, 16);
  // live hub adjacency (HLA) of the hub rows: opt-in (PACIM_HLA=1): on c4
  // recording costs more build time than the selection saves (its traversal
  // is bound by hop latency, not edge work)
  ctx->hla_ok = false;
  Hla hla{};
  const bool rec_hla = want_hla && pc_hla_begin(ctx, &hla, 1e30);
  ctx->hot_any = false;  // set by the single-window gain pass when hot sums are kept
  if (ctx->smap_of != ctx->win_first || ctx->d_smap.bytes < (size_t)B * 4) {
    // per-slot window table (select / labels address the store through it);
    // rebuilt only when the windows change (one window [0, B) by default)
    pc_ensure(ctx, ctx->d_smap, (size_t)B * 4);
    TmpBuf wf(ctx);
    pc_ensure(ctx, wf, ctx->win_first.size() * 4);
    PC_CUDA(cudaMemcpyAsync(wf.p, ctx->win_first.data(), ctx->win_first.size() * 4,
                            cudaMemcpyHostToDevice, ctx->stream));
    k_fill_smap<<<std::min<uint32_t>(nwin, 1024), 256, 0, ctx->stream>>>(wf.as<uint32_t>(), nwin,
                                                                         ctx->d_smap.as<uint32_t>());
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->smap_of = ctx->win_first;
  }
  // events: start, then per window init / edges / compress / gain done
  std::vector<cudaEvent_t> ev(2 + 4 * (size_t)nwin);
  for (auto &e : ev) PC_CUDA(cudaEventCreate(&e));
  PC_CUDA(cudaEventRecord(ev[0], ctx->stream));
  if (htime) h1 = host_ms();
  // gain0 (H7): isolated vertices are singletons everywhere (gain B)
  k_fill_i64<<<pc_grid(ctx, ctx->n, 256), 256, 0, ctx->stream>>>(ctx->gain0.as<int64_t>(), ctx->n,
                                                                (int64_t)B);
  PC_CHECK_LAUNCH();
  // partition of the edges by bucket (W > 0)
  std::vector<unsigned long long> boff;
  if (W) {
    const uint32_t NB = 1u << W;
    const uint64_t m = ctx->m;
    pc_ensure_edge_lists(ctx);
    pc_ensure(ctx, ctx->pkeys, std::max<uint64_t>(m, 1) * 16 + (NB + 1) * 16);
    uint64_t *pk = ctx->pkeys.as<uint64_t>(), *pck = pk + m;
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(pck + m);
    unsigned long long *cur = cnt + NB;
    PC_CUDA(cudaMemsetAsync(cnt, 0, NB * 8, ctx->stream));
    k_bucket_count<<<pc_grid(ctx, m, 256, 4), 256, NB * 8, ctx->stream>>>(ctx->keys.as<uint64_t>(),
                                                                         m, ctx->K, W, cnt);
    PC_CHECK_LAUNCH();
    std::vector<unsigned long long> hc(NB);
    PC_CUDA(cudaMemcpyAsync(hc.data(), cnt, NB * 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    boff.assign(NB + 1, 0);
    for (uint32_t b = 0; b < NB; b++) boff[b + 1] = boff[b] + hc[b];
    PC_CUDA(cudaMemcpyAsync(cur, boff.data(), NB * 8, cudaMemcpyHostToDevice, ctx->stream));
    k_bucket_scatter<<<pc_grid(ctx, m, 256, 8), 256, 0, ctx->stream>>>(
        ctx->keys.as<uint64_t>(), ctx->ckeys.as<uint64_t>(), m, ctx->K, W, cur, pk, pck);
    PC_CHECK_LAUNCH();
    ctx->launches += 2;
  }
  for (uint32_t w = 0; w < nwin; w++) {
    const uint32_t f = ctx->win_first[w], c = ctx->win_first[w + 1] - f;
    uint32_t *Lw = L + (size_t)n * f;
    EdgeSet es;
    if (W) {
      const uint32_t b = ctx->shr[f] >> (32 - W);
      const uint64_t *pk = ctx->pkeys.as<uint64_t>();
      es.keys = pk + boff[b];
      es.ckeys = pk + ctx->m + boff[b];
      es.m = boff[b + 1] - boff[b];
    }
    PC_CUDA(cudaEventRecord(ev[1 + 4 * w], ctx->stream));
    pc_sketch_pass(ctx, Lw, f, c, ctr, ev.data() + 2 + 4 * w, rec_hla ? &hla : nullptr,
                   W ? &es : nullptr);
    // CC sizes of the window into gain0 while it is still cached
    if (c < NARROW_W)
      k_gain_w<<<pc_grid(ctx, (size_t)n * c, 256, 16), 256, 0, ctx->stream>>>(
          Lw, n, c, ctx->rmap.as<uint32_t>(), ctx->gain0.as<int64_t>(), nwin > 1, ctr);
    else if (nwin == 1) {
      // one window: the hot CCs' sizes decide whether the per-vertex hot sums
      // are worth accumulating (some slot's hot CC above the select's dense
      // threshold — the same formula as make_sel)
      const uint32_t big_t = (uint32_t)(getenv("PACIM_BIG_T")
                                            ? std::max(1LL, atoll(getenv("PACIM_BIG_T")))
                                            : std::max<uint64_t>(65536, n / 8));
      pc_ensure(ctx, ctx->d_hot_size, (size_t)B * 4);
      k_hot_sizes<<<(c + 255) / 256, 256, 0, ctx->stream>>>(Lw, n, c, ctx->d_hot.as<uint32_t>(),
                                                            ctx->d_hot_size.as<uint32_t>(), ctx->ep);
      PC_CHECK_LAUNCH();
      ctx->hot_size.resize(B);
      PC_CUDA(cudaMemcpyAsync(ctx->hot_size.data(), ctx->d_hot_size.p, (size_t)B * 4,
                              cudaMemcpyDeviceToHost, ctx->stream));
      PC_CUDA(cudaStreamSynchronize(ctx->stream));
      bool any = false;
      for (uint32_t j = 0; j < B; j++) any |= ctx->hot_size[j] > big_t;
      ctx->hot_any = any;
      ctx->hot_big_t = big_t;
      if (any) {
        pc_ensure(ctx, ctx->hotsum, (size_t)ctx->n * 8);
        PC_CUDA(cudaMemsetAsync(ctx->hotsum.p, 0, (size_t)ctx->n * 8, ctx->stream));  // isolated: 0
        const char *gr = getenv("PACIM_GAIN_HOT");  // A/B: 0 = the generic kernel
        const int ghot = c <= 256 ? (gr ? atoi(gr) : 2) : 0;
        if (ghot == 4) {
          auto kg = ep_on ? k_gain0_fast<4, true, true> : k_gain0_fast<4, true, false>;
          kg<<<rows_grid, 256, 0, ctx->stream>>>(
              Lw, n, c, ctx->rmap.as<uint32_t>(), ctx->gain0.as<int64_t>(), ctr,
              ctx->d_hot.as<uint32_t>(), ctx->d_hot_size.as<uint32_t>(), big_t,
              ctx->hotsum.as<int64_t>(), ctx->ep);
        } else if (ghot) {
          auto kg = ep_on ? k_gain0_fast<2, true, true> : k_gain0_fast<2, true, false>;
          kg<<<rows_grid, 256, 0, ctx->stream>>>(
              Lw, n, c, ctx->rmap.as<uint32_t>(), ctx->gain0.as<int64_t>(), ctr,
              ctx->d_hot.as<uint32_t>(), ctx->d_hot_size.as<uint32_t>(), big_t,
              ctx->hotsum.as<int64_t>(), ctx->ep);
        } else {
          auto kg = ep_on ? k_gain0<true, true> : k_gain0<true, false>;
          const size_t gsm = 2 * std::min<uint32_t>(c, HOT_MAX) * sizeof(uint32_t);
          kg<<<rows_grid, 256, gsm,
                          ctx->stream>>>(Lw, n, c, ctx->rmap.as<uint32_t>(),
                                         ctx->gain0.as<int64_t>(), 0, ctr,
                                         ctx->d_hot.as<uint32_t>(), ctx->d_hot_size.as<uint32_t>(),
                                         big_t, ctx->hotsum.as<int64_t>(), ctx->ep);
        }
      } else if (c <= 128 && !(getenv("PACIM_GAIN_NARROW") && !atoi(getenv("PACIM_GAIN_NARROW")))) {
        const int S = c <= 32 ? 1 : c <= 64 ? 2 : 4;
        auto kg = S == 1 ? (ep_on ? k_gain0_narrow<true, 1> : k_gain0_narrow<false, 1>)
                : S == 2 ? (ep_on ? k_gain0_narrow<true, 2> : k_gain0_narrow<false, 2>)
                         : (ep_on ? k_gain0_narrow<true, 4> : k_gain0_narrow<false, 4>);
        kg<<<pc_grid(ctx, (size_t)n * S, 256, 8), 256, 0, ctx->stream>>>(
            Lw, n, c, ctx->rmap.as<uint32_t>(), ctx->gain0.as<int64_t>(), 0, ctr, ctx->ep);
      } else {
        auto kg = ep_on ? k_gain0<false, true> : k_gain0<false, false>;
        kg<<<rows_grid, 256, 0, ctx->stream>>>(Lw, n, c, ctx->rmap.as<uint32_t>(),
                                                          ctx->gain0.as<int64_t>(), 0, ctr,
                                                          nullptr, nullptr, 0, nullptr, ctx->ep);
      }
    } else {
      k_gain0<false, false><<<rows_grid, 256, 0, ctx->stream>>>(Lw, n, c, ctx->rmap.as<uint32_t>(),
                                                        ctx->gain0.as<int64_t>(), 1, ctr, nullptr,
                                                        nullptr, 0, nullptr, ctx->ep);
    }
    PC_CHECK_LAUNCH();
    ctx->launches++;
  }
  PC_CUDA(cudaEventRecord(ev.back(), ctx->stream));
  ctx->skip_init = false;  // other callers of pc_sketch_pass reset their stores
  if (rec_hla) pc_hla_finish(ctx, &hla);
  ctx->launches += 1;  // fill
  unsigned long long h[21];
  PC_CUDA(cudaMemcpyAsync(h, ctr, 21 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          ctx->stream));
  if (htime) h2 = host_ms();
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (htime) h3 = host_ms();
  ctx->ncomp = h[0];
  ctx->nnonsingle = h[0] + h[1];
  ctx->nmember = 0;
  ctx->stats.live_pairs = h[4];
  ctx->hk_gen = ctx->hint_gen;  // the hook list's capacity in the next build
  ctx->hk_B = B;
  ctx->hk_hint = h[1];
  ctx->stats.build_hook_list = ctx->hk_cap && h[20] <= ctx->hk_cap ? 1 : 0;
  ctx->ep_live_gen = ctx->hint_gen;  // the slot-epoch decision of the next build
  ctx->ep_live_per_slot = (double)h[4] / std::max(B, 1u);
  double ti = 0, te = 0, tc = 0, tg = 0;
  for (uint32_t w = 0; w < nwin; w++) {
    cudaEvent_t *e = ev.data() + 1 + 4 * w;  // window start, init, edges, compress
    ti += ev_ms(e[0], e[1]);
    te += ev_ms(e[1], e[2]);
    tc += ev_ms(e[2], e[3]);
    tg += ev_ms(e[3], w + 1 < nwin ? e[4] : ev.back());  // gain0 of the window
  }
  ctx->stats.t_init_ms = ti;
  ctx->stats.t_edges_ms = te;
  ctx->stats.t_compress_ms = tc;
  ctx->stats.t_gain_ms = tg;
  ctx->stats.t_compact_ms = ev_ms(ev[0], ev[1]);  // gain fill + edge partition
  ctx->stats.t_centers_ms = 0;
  ctx->stats.t_build_ms = ev_ms(ev[0], ev.back());
  ctx->stats.kernel_launches_build = ctx->launches;
  for (auto &e : ev) cudaEventDestroy(e);
  if (htime)
    fprintf(stderr, "[pc_build host ms] prep %.3f enqueue %.3f wait %.3f tail %.3f (gpu %.3f)\n", h1 - h0,
            h2 - h1, h3 - h2, host_ms() - h3, ctx->stats.t_build_ms);
}

// canonical labels of one slot: slot value is v (singleton), HIGH|ci (root:
// label v) or the root id (R8: min id of the CC)
namespace {
__global__ void k_labels(const uint32_t *L, uint32_t n, uint32_t nr, const uint32_t *smap, uint32_t j,
                         const uint32_t *cid, const uint32_t *rmap, uint32_t *out, Ep ep) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    const uint32_t c = cid[v];
    if (c == 0xFFFFFFFFu) {  // isolated vertex: singleton
      out[v] = (uint32_t)v;
      continue;
    }
    const uint32_t s = ep_rd(L[pc_addr(smap, nr, c, j)], ep);
    out[v] = (s == c || (s & PACIM_HIGH)) ? (uint32_t)v : rmap[s];
  }
}
}  // namespace

void pc_get_labels(pacim_ctx *ctx, uint32_t slot, uint32_t *host_out) {
  if (ctx->cs) return pc_cs_get_labels(ctx, slot, host_out);
  TmpBuf t(ctx);
  pc_ensure(ctx, t, (size_t)ctx->n * 4);
  k_labels<<<pc_grid(ctx, ctx->n, 256), 256, 0, ctx->stream>>>(ctx->L.as<uint32_t>(), ctx->n,
                                                              ctx->nr, ctx->d_smap.as<uint32_t>(), slot,
                                                              ctx->cid.as<uint32_t>(),
                                                              ctx->rmap.as<uint32_t>(),
                                                              t.as<uint32_t>(), ctx->ep);
  PC_CHECK_LAUNCH();
  PC_CUDA(cudaMemcpyAsync(host_out, t.p, (size_t)ctx->n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}
