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
#include <algorithm>
#include <cstdlib>

#include "pacim_internal.cuh"

namespace {

constexpr uint32_t HOT_MAX = 1024;  // slots with a shared-memory hot-root cache
constexpr uint32_t NONE = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t ld_cg(const uint32_t *p) { return __ldcg(p); }

// ---------------------------------------------------------------- k_init
__global__ void k_init(uint32_t *L, uint32_t n, uint32_t B) {
  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  if ((B & 3) == 0) {
    const uint32_t B4 = B >> 2;
    for (size_t v = warp; v < n; v += nw) {
      uint4 *row = reinterpret_cast<uint4 *>(L + v * B);
      uint4 x = make_uint4((uint32_t)v, (uint32_t)v, (uint32_t)v, (uint32_t)v);
      for (uint32_t j = lane; j < B4; j += 32) row[j] = x;
    }
  } else {
    for (size_t v = warp; v < n; v += nw)
      for (uint32_t j = lane; j < B; j += 32) L[v * B + j] = (uint32_t)v;
  }
}

// ------------------------------------------------------------- union-find
// Rem's union with splicing, lock-free (the UniteRemCAS variant of ConnectIt
// the paper uses, P:8 / P:1328): walk both paths one step at a time from the
// side with the larger parent; hook a root under the other side's parent, or
// splice the non-root's pointer over to the other side's (smaller) parent.
// Parents stay strictly smaller than children, so the final root of every
// CC is its minimum id (R8).  Two independent loads per step; the walk stops
// as soon as the two paths meet.
__device__ __forceinline__ void uf_unite(uint32_t *L, uint32_t B, uint32_t j, uint32_t u,
                                         uint32_t v) {
  uint32_t *Lj = L + j;
  for (;;) {
    uint32_t pu = ld_cg(Lj + (size_t)u * B);
    uint32_t pv = ld_cg(Lj + (size_t)v * B);
    if (pu == pv) return;
    if (pu < pv) {
      uint32_t t = u;
      u = v;
      v = t;
      t = pu;
      pu = pv;
      pv = t;
    }
    // now pu > pv
    if (u == pu) {
      if (atomicCAS(Lj + (size_t)u * B, u, pv) == u) return;  // hook root u under pv
    } else {
      atomicCAS(Lj + (size_t)u * B, pu, pv);  // splice (may lose a race harmlessly)
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

template <bool WIC, bool REC>
__global__ void __launch_bounds__(EDGE_THREADS, 8) k_edges(const uint64_t *__restrict__ keys,
                                                        const uint64_t *__restrict__ ckeys,
                                                        const uint32_t *__restrict__ tm1,
                                                        uint64_t m, uint64_t K, uint64_t t32,
                                                        const uint32_t *__restrict__ g_shr,
                                                        const uint16_t *__restrict__ g_tab,
                                                        uint32_t B, uint32_t j0, uint32_t Bb,
                                                        uint32_t *L,
                                                        unsigned long long *live_ctr, Hla hla) {
  // slots [j0, j0 + Bb) of the B sorted slots go to L (row stride Bb)
  extern __shared__ uint32_t sm[];
  uint32_t *shr = sm;
  uint16_t *tab = reinterpret_cast<uint16_t *>(sm + B);
  __shared__ uint32_t w_u[EDGE_WARPS][32], w_v[EDGE_WARPS][32], w_he[EDGE_WARPS][32];
  __shared__ uint32_t w_lo[EDGE_WARPS][32];
  __shared__ uint64_t w_T[EDGE_WARPS][32];
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) shr[i] = g_shr[i];
  for (uint32_t i = threadIdx.x; i <= (1u << PACIM_TB); i += blockDim.x) tab[i] = g_tab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t gw = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long live = 0;
  for (size_t base = gw * 32; base < m; base += nw * 32) {
    // ---- one edge per lane: hash and candidate slot range
    const size_t e = base + lane;
    uint32_t cnt = 0, eu = 0, ev = 0, ehe = 0, elo = 0;
    uint64_t eT = 0;
    if (e < m) {
      const uint64_t key = keys[e];
      const uint64_t T = WIC ? (uint64_t)tm1[e] + 1 : t32;
      const uint32_t he = (uint32_t)(pc_mix64(key ^ K) >> 32);
      uint32_t lo = 0, hi = 0;
      if (T != 0) {
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
      const uint64_t ck = ckeys[e];  // the endpoints' store rows (+ hub flags)
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
        lv = (uint64_t)(shr[j] ^ w_he[wid][a]) < T;
        u = w_u[wid][a];
        v = w_v[wid][a];
        if (lv) {
          uf_unite(L, Bb, j - j0, u & ~PACIM_HUBF, v & ~PACIM_HUBF);
          live++;
        }
      }
      if (REC)  // live edges of hubs, appended with one counter update per warp
        hla.add_warp(u & ~PACIM_HUBF, v & ~PACIM_HUBF, j, (lv && (u & PACIM_HUBF)) ? 1u : 0u,
                     (lv && (v & PACIM_HUBF)) ? 1u : 0u);
    }
    __syncwarp();
  }
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
                                            uint32_t x) {
  for (;;) {
    uint32_t p = ld_cg(L + (size_t)x * B + j);
    if (p == x || (p & PACIM_HIGH)) return x;
    x = p;
  }
}

// find with path halving for compress_count: every write is an atomicMin, so
// a slot only ever moves towards its root (ids decrease along parent
// pointers) and racing halvings can never undo an owner's full compression.
__device__ __forceinline__ uint32_t find_halve(uint32_t *L, uint32_t B, uint32_t j, uint32_t x) {
  for (;;) {
    uint32_t p = ld_cg(L + (size_t)x * B + j);
    if (p == x || (p & PACIM_HIGH)) return x;
    uint32_t gp = ld_cg(L + (size_t)p * B + j);
    if (gp == p || (gp & PACIM_HIGH)) return p;
    atomicMin(L + (size_t)x * B + j, gp);
    x = gp;
  }
}

__global__ void k_hot_roots(const uint32_t *L, uint32_t nr, uint32_t B, uint32_t hub,
                            uint32_t *hot) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x)
    hot[j] = hub < nr ? find_ro(L, B, j, hub) : NONE;
}

// ------------------------------------------------------ k_compress_count
// For every non-root (v, j): slot <- root (full compression, H4; halving and
// the owner's write are atomicMin, so the final slot is the root); the
// root slot becomes HIGH | size by CAS(root -> HIGH|1) then atomicAdd per
// member (H5).  Members of the slot's hot root are counted in shared memory
// and added once per block.  ctr[0] += CCs of size >= 2, ctr[1] += non-roots.
__device__ __forceinline__ bool add_to_root(uint32_t *L, uint32_t B, uint32_t j, uint32_t root,
                                            uint32_t cnt) {
  uint32_t *rs = L + (size_t)root * B + j;
  if (!(ld_cg(rs) & PACIM_HIGH)) atomicCAS(rs, root, PACIM_HIGH | 1u);
  uint32_t old = atomicAdd(rs, cnt);
  return old == (PACIM_HIGH | 1u);  // the first add after conversion: a new CC
}

__global__ void __launch_bounds__(256) k_compress_count(uint32_t *L, uint32_t n, uint32_t B,
                                                        const uint32_t *hot,
                                                        unsigned long long *ctr) {
  extern __shared__ uint32_t hsm[];
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
  unsigned long long ncc = 0, nnr = 0;
  for (size_t v = warp; v < n; v += nw) {
    for (uint32_t j0 = 0; j0 < B; j0 += 256) {
      uint32_t sv[8];  // prefetch up to 8 slots per lane (independent loads)
#pragma unroll
      for (int i = 0; i < 8; i++) {
        uint32_t j = j0 + lane + 32 * i;
        sv[i] = j < B ? ld_cg(L + v * B + j) : (uint32_t)v;
      }
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const uint32_t j = j0 + lane + 32 * i;
        const uint32_t s = sv[i];
        if (s == (uint32_t)v || (s & PACIM_HIGH)) continue;  // root (or singleton)
        // parent already the hot root: no walk (the common case for members
        // of the giant CC)
        uint32_t root = (j < H && s == hroot[j]) ? s : find_halve(L, B, j, s);
        if (root != s) atomicMin(L + v * B + j, root);
        nnr++;
        if (j < H && root == hroot[j]) {
          atomicAdd(hcnt + j, 1u);
        } else if (add_to_root(L, B, j, root, 1u)) {
          ncc++;
        }
      }
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < H; j += blockDim.x)
    if (hcnt[j] && add_to_root(L, B, j, hroot[j], hcnt[j])) ncc++;
  for (int d = 16; d; d >>= 1) {
    ncc += __shfl_xor_sync(0xffffffffu, ncc, d);
    nnr += __shfl_xor_sync(0xffffffffu, nnr, d);
  }
  __shared__ unsigned long long s0, s1;
  if (threadIdx.x == 0) s0 = s1 = 0;
  __syncthreads();
  if (lane == 0) {
    if (ncc) atomicAdd(&s0, ncc);
    if (nnr) atomicAdd(&s1, nnr);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s0) atomicAdd(ctr + 0, s0);
    if (s1) atomicAdd(ctr + 1, s1);
  }
}

// ---------------------------------------------------------------- k_gain0
// Warp per store row, 8 slots prefetched per lane: gain0[v] = sum_j |C_j(v)|
// (H7), the CC size read from the root slot (HIGH | size).
__global__ void __launch_bounds__(256) k_gain0(const uint32_t *__restrict__ L, uint32_t n,
                                               uint32_t B, const uint32_t *rmap, int64_t *gain0) {
  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t v = warp; v < n; v += nw) {
    long long g = 0;
    for (uint32_t j0 = 0; j0 < B; j0 += 256) {
      uint32_t sv[8];
#pragma unroll
      for (int i = 0; i < 8; i++) {
        uint32_t j = j0 + lane + 32 * i;
        sv[i] = j < B ? L[v * B + j] : NONE;
      }
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const uint32_t j = j0 + lane + 32 * i;
        const uint32_t s = sv[i];
        if (s == NONE) continue;
        if (s == (uint32_t)v) {
          g += 1;  // singleton CC
        } else if (s & PACIM_HIGH) {
          g += s & PACIM_LOW;
        } else {
          g += __ldg(L + (size_t)s * B + j) & PACIM_LOW;
        }
      }
    }
    for (int d = 16; d; d >>= 1) g += __shfl_xor_sync(0xffffffffu, g, d);
    if (lane == 0) gain0[rmap[v]] = g;
  }
}

// HLA: raw entries -> rows grouped by (hub, slot); cur = a copy of the offsets
__global__ void k_hla_scatter(const unsigned long long *raw, unsigned long long n,
                              unsigned long long *cur, uint32_t *rows) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long r = raw[i];
    rows[atomicAdd(cur + (r >> 32), 1ull)] = (uint32_t)r;
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
  std::vector<std::pair<uint32_t, uint32_t>> hs;
  for (uint32_t r = ctx->rank; r < ctx->R; r += ctx->world) {
    uint64_t h = pc_mix64(((1ull << 63) | (uint64_t)r) ^ ctx->K);
    hs.push_back({(uint32_t)(h >> 32), r});
  }
  std::sort(hs.begin(), hs.end());
  ctx->shr.resize(B);
  ctx->slot_r.resize(B);
  for (uint32_t j = 0; j < B; j++) {
    ctx->shr[j] = hs[j].first;
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
}

// One sketch pass over the edge list for slots [j0, j0+Bb): parent arrays in
// Lb (rows x Bb), unions, full compression and CC sizes (root slot HIGH|size).
// ctr[0] += non-singleton CCs, ctr[1] += non-roots, ctr[4] += live pairs.
// ev (optional, 3 events) is recorded after init, edges and compress.
void pc_sketch_pass(pacim_ctx *ctx, uint32_t *Lb, uint32_t j0, uint32_t Bb,
                    unsigned long long *ctr, cudaEvent_t *ev, const Hla *hla_in) {
  Hla hla{};
  if (hla_in) hla = *hla_in;
  const uint32_t n = ctx->nr, B = ctx->R_local;
  const uint32_t NT = 1u << PACIM_TB;
  pc_ensure(ctx, ctx->d_hot, 2 * (size_t)B * sizeof(uint32_t));
  uint32_t *hot_root = ctx->d_hot.as<uint32_t>();
  const uint32_t H = std::min<uint32_t>(Bb, HOT_MAX);
  const unsigned rows_grid = pc_grid(ctx, (size_t)n * 32, 256, 16);
  k_init<<<rows_grid, 256, 0, ctx->stream>>>(Lb, n, Bb);
  PC_CHECK_LAUNCH();
  if (ev) PC_CUDA(cudaEventRecord(ev[0], ctx->stream));
  {
    size_t smem = B * sizeof(uint32_t) + (NT + 1) * sizeof(uint16_t);
    unsigned g = pc_grid(ctx, (ctx->m + 31) / 32 * 32, EDGE_THREADS, 8);
    if (ctx->pmodel == PACIM_P_WIC) {
      auto kern = hla.cnt ? k_edges<true, true> : k_edges<true, false>;
      PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
          ctx->keys.as<uint64_t>(), ctx->ckeys.as<uint64_t>(), ctx->tm1.as<uint32_t>(), ctx->m,
          ctx->K, 0, ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(), B, j0, Bb, Lb, ctr + 4, hla);
    } else {
      auto kern = hla.cnt ? k_edges<false, true> : k_edges<false, false>;
      PC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<g, EDGE_THREADS, smem, ctx->stream>>>(
          ctx->keys.as<uint64_t>(), ctx->ckeys.as<uint64_t>(), nullptr, ctx->m, ctx->K, ctx->t32,
          ctx->d_shr.as<uint32_t>(), ctx->d_tab.as<uint16_t>(), B, j0, Bb, Lb, ctr + 4, hla);
    }
    PC_CHECK_LAUNCH();
  }
  if (ev) PC_CUDA(cudaEventRecord(ev[1], ctx->stream));
  k_hot_roots<<<(Bb + 255) / 256, 256, 0, ctx->stream>>>(Lb, n, Bb, ctx->hub_row, hot_root);
  PC_CHECK_LAUNCH();
  k_compress_count<<<rows_grid, 256, 2 * H * sizeof(uint32_t), ctx->stream>>>(Lb, n, Bb, hot_root,
                                                                              ctr);
  PC_CHECK_LAUNCH();
  if (ev) PC_CUDA(cudaEventRecord(ev[2], ctx->stream));
  ctx->launches += 4;
}

void pc_build(pacim_ctx *ctx) {
  const uint32_t n = ctx->nr, B = ctx->R_local;  // store rows = non-isolated vertices
  PC_REQUIRE(B >= 1 && B <= 65535, PACIM_EINVAL, "local sketch count must be in [1, 65535]");
  PC_REQUIRE(!ctx->compressed, PACIM_ENOTIMPL, "compressed store not built by pc_build");
  pc_slot_table(ctx);
  pc_ensure(ctx, ctx->L, (size_t)n * B * sizeof(uint32_t));
  pc_ensure(ctx, ctx->gain0, (size_t)ctx->n * sizeof(int64_t));
  pc_ensure(ctx, ctx->counters, 64 * sizeof(uint64_t));
  unsigned long long *ctr = ctx->counters.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(ctr, 0, 64 * sizeof(uint64_t), ctx->stream));
  uint32_t *L = ctx->L.as<uint32_t>();
  cudaEvent_t ev[6];
  for (auto &e : ev) PC_CUDA(cudaEventCreate(&e));
  ctx->launches = 0;
  const unsigned rows_grid = pc_grid(ctx, (size_t)n * 32, 256, 16);
  // live hub adjacency (HLA) of the hub rows: opt-in (PACIM_HLA=1): on c4 recording costs more build time than the
  // selection saves (its traversal is bound by hop latency, not edge work)
  const bool want_hla = ctx->nhub > 0 && (getenv("PACIM_HLA") != nullptr ||
                                          getenv("PACIM_FORCE_HLA") != nullptr);
  ctx->hla_ok = false;
  Hla hla{};
  if (want_hla) {
    const size_t keys = (size_t)ctx->nhub * B + 1;
    const unsigned long long cap = std::max<unsigned long long>(1ull << 20, (ctx->m / 16));
    pc_ensure(ctx, ctx->hla_off, keys * 8);
    pc_ensure(ctx, ctx->hla_raw, (cap + 1) * 8);
    PC_CUDA(cudaMemsetAsync(ctx->hla_off.p, 0, keys * 8, ctx->stream));
    PC_CUDA(cudaMemsetAsync(ctx->hla_raw.p, 0, 8, ctx->stream));
    hla.hidx = ctx->hidx.as<uint32_t>();
    hla.cnt = ctx->hla_off.as<unsigned long long>();
    hla.n = ctx->hla_raw.as<unsigned long long>();
    hla.raw = hla.n + 1;
    hla.cap = cap;
    hla.B = B;
  }
  PC_CUDA(cudaEventRecord(ev[0], ctx->stream));
  pc_sketch_pass(ctx, L, 0, B, ctr, ev + 1, want_hla ? &hla : nullptr);
  PC_CUDA(cudaEventRecord(ev[4], ctx->stream));
  // gain0 (H7): isolated vertices are singletons everywhere (gain B); every
  // store row sums its CC sizes read from the root slots (HIGH | size)
  k_fill_i64<<<pc_grid(ctx, ctx->n, 256), 256, 0, ctx->stream>>>(ctx->gain0.as<int64_t>(), ctx->n,
                                                                (int64_t)B);
  PC_CHECK_LAUNCH();
  k_gain0<<<rows_grid, 256, 0, ctx->stream>>>(L, n, B, ctx->rmap.as<uint32_t>(),
                                             ctx->gain0.as<int64_t>());
  PC_CHECK_LAUNCH();
  if (want_hla) {
    // counts -> offsets (in place via scratch), then rows grouped by key
    const size_t keys = (size_t)ctx->nhub * B + 1;
    unsigned long long nraw = 0;
    PC_CUDA(cudaMemcpyAsync(&nraw, hla.n, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (nraw <= hla.cap) {
      TmpBuf cur(ctx);
      pc_ensure(ctx, cur, keys * 8);
      pc_exclusive_scan_u64(ctx, reinterpret_cast<const uint64_t *>(hla.cnt), cur.as<uint64_t>(), keys);
      PC_CUDA(cudaMemcpyAsync(hla.cnt, cur.p, keys * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      pc_ensure(ctx, ctx->hla_row, std::max<size_t>(nraw, 1) * 4);
      k_hla_scatter<<<pc_grid(ctx, nraw, 256), 256, 0, ctx->stream>>>(
          hla.raw, nraw, cur.as<unsigned long long>(), ctx->hla_row.as<uint32_t>());
      PC_CHECK_LAUNCH();
      PC_CUDA(cudaStreamSynchronize(ctx->stream));
      ctx->hla_ok = true;
      ctx->hla_n = nraw;
      ctx->launches += 2;
    }
  }
  PC_CUDA(cudaEventRecord(ev[5], ctx->stream));
  ctx->launches += 2;  // fill, gain0
  unsigned long long h[6];
  PC_CUDA(cudaMemcpyAsync(h, ctr, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->ncomp = h[0];
  ctx->nnonsingle = h[0] + h[1];
  ctx->nmember = 0;
  ctx->stats.live_pairs = h[4];
  ctx->stats.t_init_ms = ev_ms(ev[0], ev[1]);
  ctx->stats.t_edges_ms = ev_ms(ev[1], ev[2]);
  ctx->stats.t_compress_ms = ev_ms(ev[2], ev[3]);
  ctx->stats.t_compact_ms = ev_ms(ev[3], ev[4]);
  ctx->stats.t_gain_ms = ev_ms(ev[4], ev[5]);
  ctx->stats.t_centers_ms = 0;
  ctx->stats.t_build_ms = ev_ms(ev[0], ev[5]);
  ctx->stats.kernel_launches_build = ctx->launches;
  for (auto &e : ev) cudaEventDestroy(e);
}

// canonical labels of one slot: slot value is v (singleton), HIGH|ci (root:
// label v) or the root id (R8: min id of the CC)
namespace {
__global__ void k_labels(const uint32_t *L, uint32_t n, uint32_t B, uint32_t j,
                         const uint32_t *cid, const uint32_t *rmap, uint32_t *out) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    const uint32_t c = cid[v];
    if (c == 0xFFFFFFFFu) {  // isolated vertex: singleton
      out[v] = (uint32_t)v;
      continue;
    }
    uint32_t s = L[(size_t)c * B + j];
    out[v] = (s == c || (s & PACIM_HIGH)) ? (uint32_t)v : rmap[s];
  }
}
}  // namespace

void pc_get_labels(pacim_ctx *ctx, uint32_t slot, uint32_t *host_out) {
  TmpBuf t(ctx);
  pc_ensure(ctx, t, (size_t)ctx->n * 4);
  k_labels<<<pc_grid(ctx, ctx->n, 256), 256, 0, ctx->stream>>>(ctx->L.as<uint32_t>(), ctx->n,
                                                              ctx->R_local, slot,
                                                              ctx->cid.as<uint32_t>(),
                                                              ctx->rmap.as<uint32_t>(),
                                                              t.as<uint32_t>());
  PC_CHECK_LAUNCH();
  PC_CUDA(cudaMemcpyAsync(host_out, t.p, (size_t)ctx->n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}
