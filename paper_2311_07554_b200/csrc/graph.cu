// graph.cu — H0/H1: CSR load, validation, upper edge list, WIC thresholds,
// and the on-device synthetic generators (DESIGN.md §Input recipe).
//
// Sorting in the generators uses CUB radix sort (setup stage, outside the
// timed build/select step); every other kernel here is hand-written.
#include <cub/cub.cuh>

#include <cstdlib>
#include <vector>

#include "pacim_internal.cuh"

// ------------------------------------------------------------------- scan
// Exclusive prefix sum of u64 (3-phase: tile reduce, recursive scan of tile
// sums, tile scan + base).  In-place allowed.
namespace {
constexpr int SCAN_BLOCK = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

__device__ __forceinline__ uint64_t block_excl_scan(uint64_t x, uint64_t *warp_tot,
                                                    uint64_t &block_total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t inc = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    uint64_t t = lane < nw ? warp_tot[lane] : 0, ti = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, ti, d);
      if (lane >= d) ti += y;
    }
    if (lane < nw) warp_tot[lane] = ti - t;
    if (lane == nw - 1) warp_tot[32] = ti;
  }
  __syncthreads();
  block_total = warp_tot[32];
  uint64_t r = inc - x + warp_tot[wid];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_reduce(const uint64_t *in, size_t N,
                                                            uint64_t *sums) {
  __shared__ uint64_t wt[33];
  size_t base = (size_t)blockIdx.x * SCAN_TILE;
  uint64_t s = 0;
  for (int i = 0; i < SCAN_ITEMS; i++) {
    size_t idx = base + (size_t)i * SCAN_BLOCK + threadIdx.x;
    if (idx < N) s += in[idx];
  }
  uint64_t tot;
  block_excl_scan(s, wt, tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_apply(const uint64_t *in, uint64_t *out,
                                                           size_t N, const uint64_t *tile_base) {
  __shared__ uint64_t tile[SCAN_TILE];
  __shared__ uint64_t wt[33];
  size_t base = (size_t)blockIdx.x * SCAN_TILE;
  for (int i = 0; i < SCAN_ITEMS; i++) {
    size_t idx = base + (size_t)i * SCAN_BLOCK + threadIdx.x;
    tile[i * SCAN_BLOCK + threadIdx.x] = idx < N ? in[idx] : 0;
  }
  __syncthreads();
  uint64_t v[SCAN_ITEMS], s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    v[i] = tile[threadIdx.x * SCAN_ITEMS + i];
    s += v[i];
  }
  uint64_t tot;
  uint64_t run = block_excl_scan(s, wt, tot) + (tile_base ? tile_base[blockIdx.x] : 0);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    tile[threadIdx.x * SCAN_ITEMS + i] = run;
    run += v[i];
  }
  __syncthreads();
  for (int i = 0; i < SCAN_ITEMS; i++) {
    size_t idx = base + (size_t)i * SCAN_BLOCK + threadIdx.x;
    if (idx < N) out[idx] = tile[i * SCAN_BLOCK + threadIdx.x];
  }
}
}  // namespace

static void scan_rec(pacim_ctx *ctx, const uint64_t *in, uint64_t *out, size_t N,
                     uint64_t *tmp) {
  size_t nb = (N + SCAN_TILE - 1) / SCAN_TILE;
  if (nb <= 1) {
    k_scan_apply<<<1, SCAN_BLOCK, 0, ctx->stream>>>(in, out, N, nullptr);
    PC_CHECK_LAUNCH();
    ctx->launches++;
    return;
  }
  uint64_t *sums = tmp;
  k_scan_reduce<<<(unsigned)nb, SCAN_BLOCK, 0, ctx->stream>>>(in, N, sums);
  PC_CHECK_LAUNCH();
  scan_rec(ctx, sums, sums, nb, tmp + nb);
  k_scan_apply<<<(unsigned)nb, SCAN_BLOCK, 0, ctx->stream>>>(in, out, N, sums);
  PC_CHECK_LAUNCH();
  ctx->launches += 2;
}

void pc_exclusive_scan_u64(pacim_ctx *ctx, const uint64_t *in, uint64_t *out, size_t N) {
  if (N == 0) return;
  size_t need = 0, t = N;
  while (t > 1) {
    t = (t + SCAN_TILE - 1) / SCAN_TILE;
    need += t + 1;
  }
  pc_ensure(ctx, ctx->scratch2, (need + 1) * sizeof(uint64_t));
  scan_rec(ctx, in, out, N, ctx->scratch2.as<uint64_t>());
}

// ------------------------------------------------------------- validation
namespace {
// One warp per vertex: offsets monotone, ids < n, no self loop, strictly
// increasing lists.  bad[0] = smallest offending vertex (atomicMin).
__global__ void k_validate(const uint64_t *off, const uint32_t *nbr, uint32_t n,
                           uint32_t *bad) {
  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t v = warp; v < n; v += nwarps) {
    uint64_t a = off[v], b = off[v + 1];
    bool ok = b >= a;
    if (ok) {
      for (uint64_t e = a + lane; e < b; e += 32) {
        uint32_t w = nbr[e];
        if (w >= n || w == (uint32_t)v || (e > a && nbr[e - 1] >= w)) ok = false;
      }
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok && lane == 0) atomicMin(bad, (uint32_t)v);
  }
}

// Symmetry: for each entry (v, w), v must appear in w's (sorted) list.
__global__ void k_validate_sym(const uint64_t *off, const uint32_t *nbr, uint32_t n,
                               uint32_t *bad) {
  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t v = warp; v < n; v += nwarps) {
    bool ok = true;
    for (uint64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
      uint32_t w = nbr[e];
      uint64_t lo = off[w], hi = off[w + 1];
      while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (nbr[mid] < (uint32_t)v) lo = mid + 1; else hi = mid;
      }
      if (lo == off[w + 1] || nbr[lo] != (uint32_t)v) ok = false;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok && lane == 0) atomicMin(bad, (uint32_t)v);
  }
}

// Upper degree: number of neighbours w > v (lists are sorted).
__global__ void k_upper_count(const uint64_t *off, const uint32_t *nbr, uint32_t n,
                              uint64_t *ucnt) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    uint64_t lo = off[v], hi = off[v + 1], end = hi;
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (nbr[mid] <= (uint32_t)v) lo = mid + 1; else hi = mid;
    }
    ucnt[v] = end - lo;
  }
}

// row of CSR entry e: the chunk table gives the row of entry 32 * (e >> 5),
// advanced past row ends (lane per entry: balanced whatever the degrees; a
// warp per vertex left a hub's 10^6 entries to one warp: 87 ms at c4)
__device__ __forceinline__ uint32_t entry_row(const uint64_t *off, const uint32_t *crow,
                                              uint64_t e) {
  uint32_t u = crow[e >> 5];
  while (e >= off[u + 1]) u++;
  return u;
}

// per vertex: degree << 32 | store row (+ hub flag) — the one gather per CSR
// entry of k_edge_derive (separate cid / hidx / off gathers cost 5 random
// reads per upper edge: 105 ms at c4)
__global__ void k_vinfo(const uint64_t *off, const uint32_t *cid, const uint32_t *hidx,
                        uint32_t n, uint64_t *vinfo) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    uint32_t c = cid[v];
    if (c != 0xFFFFFFFFu && hidx[c] != 0xFFFFFFFFu) c |= PACIM_HUBF;
    vinfo[v] = ((off[v + 1] - off[v]) << 32) | c;
  }
}

// Lane per CSR entry e = (u, w): the upper edge list (keys[ustart[u] + i] =
// u<<32 | w for the i-th neighbour w > u; lists are sorted, so keys are), the
// same edge as store rows + hub flags (ckeys), and for the per-edge models the
// threshold T32 - toff per upper edge (tm1) and per CSR entry (tcsr):
// WIC R4 T32 = min(2^32, floor(2^33 / (d_u + d_w))), Uniform R19
// pc_t32_uniform(packed, key).
// keys / ckeys null: the thresholds only (the per-build stream reads the CSR,
// UpperCsr); tm1 null: the edge lists only (pc_ensure_edge_lists).
// unbr / ud8 (UpperCsr): the upper neighbours and row deltas (ucrow given).
__global__ void k_edge_derive(const uint64_t *off, const uint32_t *nbr, const uint32_t *crow,
                              uint64_t nnz, const uint64_t *uoff,
                              const uint64_t *vinfo, int pmodel, uint64_t t32, uint32_t toff,
                              uint64_t *keys, uint64_t *ckeys, uint32_t *tm1, uint32_t *tcsr,
                              uint32_t *unbr = nullptr, uint16_t *ud16 = nullptr,
                              const uint32_t *ucrow = nullptr, uint32_t *uvrow = nullptr,
                              const uint32_t *ucrowr = nullptr, bool cap_all = false) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (size_t)gridDim.x * blockDim.x) {
    const uint32_t u = entry_row(off, crow, e), w = nbr[e];
    if (!tcsr && w < u) continue;  // lower entries: nothing to write
    if (unbr) {
      const uint64_t pos = uoff[u + 1] - (off[u + 1] - e);
      unbr[pos] = w;
      const uint32_t du = min(255u, u - ucrow[pos >> 5]),
                     dr = min(255u, ((uint32_t)vinfo[u] & ~PACIM_HUBF) - ucrowr[pos >> 5]);
      ud16[pos] = cap_all ? (uint16_t)0xFFFF : (uint16_t)(du | dr << 8);
      if (uvrow) uvrow[pos] = (uint32_t)vinfo[w] & ~PACIM_HUBF;
    }
    if (!tcsr && !tm1 && !keys) continue;
    const uint64_t iu = vinfo[u], iw = vinfo[w];
    uint64_t T = 0;
    if (!tm1 && !tcsr) {
    } else if (pmodel == PACIM_P_WIC) {
      T = (1ull << 33) / ((iu >> 32) + (iw >> 32));
      if (T > (1ull << 32)) T = 1ull << 32;
    } else if (pmodel == PACIM_P_UNIFORM) {
      const uint64_t a = u < w ? u : w, b = u < w ? w : u;
      T = pc_t32_uniform(t32, (a << 32) | b);
    }
    if (tcsr) tcsr[e] = (uint32_t)(T - toff);
    if (w > u) {
      const uint64_t pos = uoff[u + 1] - (off[u + 1] - e);  // upper edge index
      if (keys) {
        keys[pos] = ((uint64_t)u << 32) | w;
        ckeys[pos] = ((iu & 0xFFFFFFFFull) << 32) | (iw & 0xFFFFFFFFull);
      }
      if (tm1 && pmodel != PACIM_P_CONST) tm1[pos] = (uint32_t)(T - toff);
    }
  }
}

// k_edge_derive for a graph held as an upper CSR (uoff, unbr; lane per upper
// edge e, its row by the chunk table ucrow and pc_row_of): the edge lists
// (keys, ckeys) or the stream's deltas and neighbour rows (ud16, uvrow), and
// tm1 for the per-edge models
__global__ void k_edge_derive_up(const uint64_t *uoff, const uint32_t *unbr, const uint32_t *ucrow,
                                 uint64_t m, uint32_t n, const uint64_t *vinfo, int pmodel,
                                 uint64_t t32, uint32_t toff, uint64_t *keys, uint64_t *ckeys,
                                 uint32_t *tm1, uint16_t *ud16, uint32_t *uvrow,
                                 const uint32_t *ucrowr, bool cap_all) {
  const uint64_t nch = (m + 31) / 32;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (size_t)gridDim.x * blockDim.x) {
    const uint64_t c = e >> 5;
    const uint32_t u0 = ucrow[c];
    const uint32_t u = pc_row_of(uoff, u0, c + 1 < nch ? ucrow[c + 1] : n - 1, e);
    const uint32_t w = unbr[e];
    const uint64_t iu = vinfo[u], iw = vinfo[w];
    if (keys) {
      keys[e] = ((uint64_t)u << 32) | w;
      ckeys[e] = ((iu & 0xFFFFFFFFull) << 32) | (iw & 0xFFFFFFFFull);
    }
    if (ud16) {
      const uint32_t du = min(255u, u - u0),
                     dr = min(255u, ((uint32_t)iu & ~PACIM_HUBF) - ucrowr[c]);
      ud16[e] = cap_all ? (uint16_t)0xFFFF : (uint16_t)(du | dr << 8);
      if (uvrow) uvrow[e] = (uint32_t)iw & ~PACIM_HUBF;
    }
    if (tm1 && pmodel != PACIM_P_CONST) {
      uint64_t T;
      if (pmodel == PACIM_P_WIC) {
        T = (1ull << 33) / ((iu >> 32) + (iw >> 32));
        if (T > (1ull << 32)) T = 1ull << 32;
      } else {
        T = pc_t32_uniform(t32, ((uint64_t)u << 32) | w);
      }
      tm1[e] = (uint32_t)(T - toff);
    }
  }
}

// lower degrees of an upper CSR: lcnt[v] = #{upper edges (u, v)}
__global__ void k_lower_hist(const uint32_t *unbr, uint64_t m, uint32_t *lcnt) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (size_t)gridDim.x * blockDim.x)
    atomicAdd(lcnt + unbr[e], 1u);
}
// deg[v] = upper + lower degree (deg[n] = 0, for the exclusive scan)
__global__ void k_up_deg(const uint64_t *uoff, const uint32_t *lcnt, uint32_t n, uint64_t *deg) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
       v += (size_t)gridDim.x * blockDim.x)
    deg[v] = v < n ? uoff[v + 1] - uoff[v] + lcnt[v] : 0;
}

// store row of every chunk's first upper-edge vertex (UpperCsr)
__global__ void k_chunk_rows(const uint32_t *ucrow, const uint32_t *cid, uint64_t nch,
                             uint32_t *ucrowr) {
  for (size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x; c < nch;
       c += (size_t)gridDim.x * blockDim.x)
    ucrowr[c] = cid[ucrow[c]];
}

// rank map of the store rows (UpperCsr): warp per 32 vertices, rk[w] = {row
// of the word's first non-isolated vertex (cid), bitmap of its non-isolated
// vertices}; rows keep the vertex order, so row(v) = rk.x + popc(below v)
__global__ void k_rank_map(const uint64_t *off, const uint32_t *cid, uint32_t n, uint2 *rk) {
  const uint32_t lane = threadIdx.x & 31;
  const size_t nw = ((size_t)n + 31) / 32;
  for (size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((size_t)gridDim.x * blockDim.x) >> 5) {
    const size_t v = w * 32 + lane;
    const bool ni = v < n && off[v + 1] > off[v];
    const uint32_t bm = __ballot_sync(0xffffffffu, ni);
    if (lane == 0) rk[w] = make_uint2(bm ? cid[w * 32 + __ffs(bm) - 1] : 0u, bm);
  }
}
}  // namespace

// ------------------------------------------------------------------ hub
namespace {
// packed (degree << 32 | ~v) max: the largest degree, smallest id on ties
__global__ void k_max_deg(const uint64_t *off, uint32_t n, unsigned long long *best) {
  unsigned long long b = 0;
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    unsigned long long d = off[v + 1] - off[v];
    unsigned long long key = (d << 32) | (0xFFFFFFFFull - v);
    if (key > b) b = key;
  }
  for (int s = 16; s; s >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, b, s);
    if (o > b) b = o;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(best, b);
}
}  // namespace

namespace {
__global__ void k_nonisolated(const uint64_t *off, uint32_t n, uint64_t *flag) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x)
    flag[v] = off[v + 1] > off[v] ? 1 : 0;
}

__global__ void k_rowmap(const uint64_t *flag, const uint64_t *pos, uint32_t n, uint32_t *cid,
                         uint32_t *rmap) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    if (flag[v]) {
      cid[v] = (uint32_t)pos[v];
      rmap[pos[v]] = (uint32_t)v;
    } else {
      cid[v] = 0xFFFFFFFFu;
    }
  }
}

// hub index of the store rows: degree > hub_deg
__global__ void k_hub_index(const uint64_t *off, const uint32_t *rmap, uint32_t nr,
                            uint64_t hub_deg, uint32_t *hidx, unsigned long long *cnt) {
  for (size_t u = (size_t)blockIdx.x * blockDim.x + threadIdx.x; u < nr;
       u += (size_t)gridDim.x * blockDim.x) {
    const uint32_t x = rmap[u];
    const uint64_t d = off[x + 1] - off[x];
    hidx[u] = d > hub_deg ? (uint32_t)atomicAdd(cnt, 1ull) : 0xFFFFFFFFu;
    if (d > hub_deg) atomicAdd(cnt + 1, (unsigned long long)d);  // hub CSR entries
  }
}

// the hub rows into the hash table of Hla::hub_of (all slots start empty, ~0)
__global__ void k_hub_table(const uint32_t *hidx, uint32_t nr, unsigned long long *tab,
                            uint32_t mask) {
  for (size_t u = (size_t)blockIdx.x * blockDim.x + threadIdx.x; u < nr;
       u += (size_t)gridDim.x * blockDim.x) {
    const uint32_t hi = hidx[u];
    if (hi == 0xFFFFFFFFu) continue;
    const unsigned long long e = ((unsigned long long)u << 32) | hi;
    for (uint32_t h = ((uint32_t)u * 2654435761u) & mask;; h = (h + 1) & mask)
      if (atomicCAS(tab + h, ~0ull, e) == ~0ull) break;
  }
}
}  // namespace

// Everything derived from (off, nbr, keys): hub vertex, the store's row map
// (isolated vertices are singletons in every sketch and get no row; rows keep
// the vertex order, so min row = min id), compact edge endpoints, WIC T32.
static void derive_lean(pacim_ctx *ctx);
namespace {
__global__ void k_crow(const uint64_t *off, uint32_t n, uint32_t *crow);
__global__ void k_crow_of(const uint64_t *off, uint32_t n, uint32_t *crow);
__global__ void k_iota_u32(uint32_t *a, uint32_t n);
}  // namespace

// crow[c] = row of CSR entry 32 c: the chunk table of the lane-per-entry kernels
static void make_crow(pacim_ctx *ctx, DevBuf &crow) {
  const uint64_t nch = (2 * ctx->m + 31) / 32;
  pc_ensure(ctx, crow, (nch + 1) * 4);
  k_crow<<<pc_grid(ctx, ctx->n, 256), 256, 0, ctx->stream>>>(ctx->off.as<uint64_t>(), ctx->n,
                                                            crow.as<uint32_t>());
  PC_CHECK_LAUNCH();
  ctx->launches++;
}

// from the degrees alone: hub vertex, store rows (cid / rmap), hub rows
static void derive_rows(pacim_ctx *ctx) {
  const uint32_t n = ctx->n;
  uint64_t *off = ctx->off.as<uint64_t>();
  {
    pc_ensure(ctx, ctx->counters, 64 * 8);
    unsigned long long *t = ctx->counters.as<unsigned long long>();
    PC_CUDA(cudaMemsetAsync(t, 0, 8, ctx->stream));
    k_max_deg<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(off, n, t);
    PC_CHECK_LAUNCH();
    unsigned long long h = 0;
    PC_CUDA(cudaMemcpyAsync(&h, t, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->hub = (uint32_t)(0xFFFFFFFFull - (h & 0xFFFFFFFFull));
    ctx->hub_degree = h >> 32;
    if (ctx->hub >= n) ctx->hub = 0;
  }
  {
    // persistent scratch (capacity reused across loads: no cudaMalloc/cudaFree)
    pc_ensure(ctx, ctx->scratch, 2 * ((size_t)n + 1) * 8);
    DevBuf flag, pos;
    flag.p = ctx->scratch.p;
    pos.p = ctx->scratch.as<uint64_t>() + n + 1;

    k_nonisolated<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(off, n, flag.as<uint64_t>());
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaMemsetAsync(flag.as<uint64_t>() + n, 0, 8, ctx->stream));
    pc_exclusive_scan_u64(ctx, flag.as<uint64_t>(), pos.as<uint64_t>(), (size_t)n + 1);
    uint64_t nr = 0;
    PC_CUDA(cudaMemcpyAsync(&nr, pos.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->nr = (uint32_t)nr;
    pc_ensure(ctx, ctx->cid, (size_t)n * 4);
    pc_ensure(ctx, ctx->rmap, std::max<size_t>(nr, 1) * 4);
    k_rowmap<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(flag.as<uint64_t>(), pos.as<uint64_t>(),
                                                           n, ctx->cid.as<uint32_t>(),
                                                           ctx->rmap.as<uint32_t>());
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaMemcpyAsync(&ctx->hub_row, ctx->cid.as<uint32_t>() + ctx->hub, 4,
                            cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  {
    // hub rows (degree > hub_deg): their live edges are recorded by the build
    if (const char *e = getenv("PACIM_HUB_DEG")) ctx->hub_deg = (uint64_t)std::max(1LL, atoll(e));
    pc_ensure(ctx, ctx->hidx, std::max<size_t>(ctx->nr, 1) * 4);
    unsigned long long *t = ctx->counters.as<unsigned long long>();
    PC_CUDA(cudaMemsetAsync(t, 0, 16, ctx->stream));
    k_hub_index<<<pc_grid(ctx, ctx->nr, 256), 256, 0, ctx->stream>>>(
        off, ctx->rmap.as<uint32_t>(), ctx->nr, ctx->hub_deg, ctx->hidx.as<uint32_t>(), t);
    PC_CHECK_LAUNCH();
    unsigned long long h[2] = {0, 0};
    PC_CUDA(cudaMemcpyAsync(h, t, 16, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->nhub = (uint32_t)h[0];
    ctx->hub_entries = h[1];
    uint32_t tsz = 1024;
    while (tsz < 2ull * ctx->nhub) tsz *= 2;
    ctx->hub_mask = tsz - 1;
    pc_ensure(ctx, ctx->hub_tab, (size_t)tsz * 8);
    PC_CUDA(cudaMemsetAsync(ctx->hub_tab.p, 0xFF, (size_t)tsz * 8, ctx->stream));
    k_hub_table<<<pc_grid(ctx, ctx->nr, 256), 256, 0, ctx->stream>>>(
        ctx->hidx.as<uint32_t>(), ctx->nr, ctx->hub_tab.as<unsigned long long>(), ctx->hub_mask);
    PC_CHECK_LAUNCH();
  }
}

// from the CSR: upper edge list, its store-row form, per-edge thresholds
// (counts -> scan -> one lane-per-entry pass, k_edge_derive)
static void derive_edges(pacim_ctx *ctx) {
  const uint32_t n = ctx->n;
  const uint64_t m = ctx->m, nnz = 2 * m;
  uint64_t *off = ctx->off.as<uint64_t>();
  const uint32_t *nbr = ctx->nbr.as<uint32_t>();
  const bool up = ctx->upper_src;  // uoff / unbr / ucrow hold the upper CSR
  if (!up) {
    pc_ensure(ctx, ctx->scratch, ((size_t)n + 1) * sizeof(uint64_t));
    uint64_t *ucnt = ctx->scratch.as<uint64_t>();
    pc_ensure(ctx, ctx->uoff, ((size_t)n + 1) * sizeof(uint64_t));
    k_upper_count<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(off, nbr, n, ucnt);
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaMemsetAsync(ucnt + n, 0, 8, ctx->stream));
    pc_exclusive_scan_u64(ctx, ucnt, ctx->uoff.as<uint64_t>(), (size_t)n + 1);
  }
  uint64_t *uoff = ctx->uoff.as<uint64_t>();
  // Two forms of the upper edges for the build's edge pass (k_edges):
  // * the edge lists keys / ckeys (16 B per upper edge, 25 GB at c4; + tm1):
  //   fastest (k_edges is issue bound: the stream's decode adds ~11 % warp
  //   instructions, c4 22.8 -> 24.3 ms), the default when they take at most a
  //   fifth of the device;
  // * the stream UpperCsr (unbr, ud16, uvrow: 10 B per edge + tm1) otherwise
  //   (or PACIM_UCSR=1/2/3; 0: the lists): the edge lists are then derived
  //   only on first use (pc_ensure_edge_lists: compact store, edge-
  //   partitioned and bucketed builds, HLA recording).
  // On first use either way: the per-CSR-entry thresholds (pc_ensure_tcsr:
  // traversal selections, compressed probes, Monte Carlo)
  // * the CSR-direct form (no per-edge array: rows by the rank map, the
  //   neighbour from the CSR) when not even the stream fits in a fifth (c5),
  //   or PACIM_UCSR=4.
  const char *ue = getenv("PACIM_UCSR");
  const int ucsr = ue ? atoi(ue) : -1;
  {
    size_t fr = 0, tot = 0;
    pc_mem_info(ctx, &fr, &tot);
    ctx->ucsr = ucsr > 0 || (ucsr < 0 && 16 * m > tot / 5);
    ctx->ucsr_direct = ucsr == 4 || (ucsr < 0 && 10 * m > tot / 5);
  }
  const bool per_edge = ctx->pmodel != PACIM_P_CONST;
  if (per_edge) pc_ensure(ctx, ctx->tm1, std::max<size_t>(m, 1) * sizeof(uint32_t));
  ctx->tcsr_ok = false;
  ctx->elist_ok = false;
  if (ctx->ucsr) {
    pc_free(ctx, ctx->keys);
    pc_free(ctx, ctx->ckeys);
    pc_ensure(ctx, ctx->rk, ((size_t)n / 32 + 1) * sizeof(uint2));
    k_rank_map<<<pc_grid(ctx, (size_t)n + 31, 256), 256, 0, ctx->stream>>>(
        off, ctx->cid.as<uint32_t>(), n, ctx->rk.as<uint2>());
    PC_CHECK_LAUNCH();
    if (!up) {
      pc_ensure(ctx, ctx->ucrow, ((m + 31) / 32 + 1) * 4);
      if (m) {
        k_crow_of<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(uoff, n, ctx->ucrow.as<uint32_t>());
        PC_CHECK_LAUNCH();
      }
    }
    ctx->launches += 2;
  } else {
    for (DevBuf *d : {&ctx->rk, &ctx->ud16, &ctx->uvrow, &ctx->ucrowr}) pc_free(ctx, *d);
    if (!up)
      for (DevBuf *d : {&ctx->ucrow, &ctx->unbr}) pc_free(ctx, *d);
    pc_ensure(ctx, ctx->keys, std::max<size_t>(m, 1) * 8);
    pc_ensure(ctx, ctx->ckeys, std::max<size_t>(m, 1) * 8);
  }
  if (nnz) {
    make_crow(ctx, ctx->crow);  // capacity kept across loads (no cudaMalloc per load)
    pc_ensure(ctx, ctx->vinfo, (size_t)n * 8);
    k_vinfo<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(off, ctx->cid.as<uint32_t>(),
                                                          ctx->hidx.as<uint32_t>(), n,
                                                          ctx->vinfo.as<uint64_t>());
    PC_CHECK_LAUNCH();
    if (ctx->ucsr && ctx->ucsr_direct) {  // per-edge arrays: tm1 only
      for (DevBuf *d : {&ctx->ud16, &ctx->uvrow, &ctx->ucrowr}) pc_free(ctx, *d);
      if (!up) pc_free(ctx, ctx->unbr);
      if (per_edge && up) {
        k_edge_derive_up<<<pc_grid(ctx, m, 256, 16), 256, 0, ctx->stream>>>(
            uoff, ctx->unbr.as<uint32_t>(), ctx->ucrow.as<uint32_t>(), m, n, ctx->vinfo.as<uint64_t>(),
            ctx->pmodel, ctx->t32, ctx->toff(), nullptr, nullptr, ctx->tm1.as<uint32_t>(), nullptr,
            nullptr, nullptr, false);
      } else if (per_edge) {
        k_edge_derive<<<pc_grid(ctx, nnz, 256), 256, 0, ctx->stream>>>(
            off, nbr, ctx->crow.as<uint32_t>(), nnz, uoff, ctx->vinfo.as<uint64_t>(), ctx->pmodel,
            ctx->t32, ctx->toff(), nullptr, nullptr, ctx->tm1.as<uint32_t>(), nullptr);
      }
    } else if (up) {  // lane per upper edge of the upper CSR
      const bool vrow = ucsr != 2 && ucsr != 3;
      if (ctx->ucsr) {
        pc_ensure(ctx, ctx->ud16, m * 2);
        pc_ensure(ctx, ctx->ucrowr, ((m + 31) / 32 + 1) * 4);
        k_chunk_rows<<<pc_grid(ctx, (m + 31) / 32, 256), 256, 0, ctx->stream>>>(
            ctx->ucrow.as<uint32_t>(), ctx->cid.as<uint32_t>(), (m + 31) / 32,
            ctx->ucrowr.as<uint32_t>());
        PC_CHECK_LAUNCH();
        if (vrow) pc_ensure(ctx, ctx->uvrow, m * 4);
        else pc_free(ctx, ctx->uvrow);
      }
      k_edge_derive_up<<<pc_grid(ctx, m, 256, 16), 256, 0, ctx->stream>>>(
          uoff, ctx->unbr.as<uint32_t>(), ctx->ucrow.as<uint32_t>(), m, n, ctx->vinfo.as<uint64_t>(),
          ctx->pmodel, ctx->t32, ctx->toff(), ctx->ucsr ? nullptr : ctx->keys.as<uint64_t>(),
          ctx->ucsr ? nullptr : ctx->ckeys.as<uint64_t>(), per_edge ? ctx->tm1.as<uint32_t>() : nullptr,
          ctx->ucsr ? ctx->ud16.as<uint16_t>() : nullptr,
          (ctx->ucsr && vrow) ? ctx->uvrow.as<uint32_t>() : nullptr, ctx->ucrowr.as<uint32_t>(),
          ucsr == 3);
      ctx->elist_ok = !ctx->ucsr;
    } else if (ctx->ucsr) {
      pc_ensure(ctx, ctx->unbr, m * 4);
      pc_ensure(ctx, ctx->ud16, m * 2);
      pc_ensure(ctx, ctx->ucrowr, ((m + 31) / 32 + 1) * 4);
      k_chunk_rows<<<pc_grid(ctx, (m + 31) / 32, 256), 256, 0, ctx->stream>>>(
          ctx->ucrow.as<uint32_t>(), ctx->cid.as<uint32_t>(), (m + 31) / 32,
          ctx->ucrowr.as<uint32_t>());
      PC_CHECK_LAUNCH();
      // the neighbours' store rows as a stream (a rank-map lookup per edge is
      // a dependent L2 gather in k_edges' front end; PACIM_UCSR=2: the rank
      // map; 3, tests: every delta capped — the offsets search and the rank
      // map for every edge)
      const bool vrow = ucsr != 2 && ucsr != 3;
      if (vrow) pc_ensure(ctx, ctx->uvrow, m * 4);
      else pc_free(ctx, ctx->uvrow);
      k_edge_derive<<<pc_grid(ctx, nnz, 256), 256, 0, ctx->stream>>>(
          off, nbr, ctx->crow.as<uint32_t>(), nnz, uoff, ctx->vinfo.as<uint64_t>(), ctx->pmodel,
          ctx->t32, ctx->toff(), nullptr, nullptr, per_edge ? ctx->tm1.as<uint32_t>() : nullptr,
          nullptr, ctx->unbr.as<uint32_t>(), ctx->ud16.as<uint16_t>(), ctx->ucrow.as<uint32_t>(),
          vrow ? ctx->uvrow.as<uint32_t>() : nullptr, ctx->ucrowr.as<uint32_t>(), ucsr == 3);
    } else {
      k_edge_derive<<<pc_grid(ctx, nnz, 256), 256, 0, ctx->stream>>>(
          off, nbr, ctx->crow.as<uint32_t>(), nnz, uoff, ctx->vinfo.as<uint64_t>(), ctx->pmodel,
          ctx->t32, ctx->toff(), ctx->keys.as<uint64_t>(), ctx->ckeys.as<uint64_t>(),
          per_edge ? ctx->tm1.as<uint32_t>() : nullptr, nullptr);
      ctx->elist_ok = true;
    }
    PC_CHECK_LAUNCH();
  } else {
    ctx->elist_ok = !ctx->ucsr;
  }
  ctx->launches += 6;
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

void pc_ensure_edge_lists(pacim_ctx *ctx) {
  if (ctx->lean || ctx->elist_ok) return;
  const uint64_t m = ctx->m, nnz = 2 * m;
  pc_ensure(ctx, ctx->keys, std::max<size_t>(m, 1) * 8);
  pc_ensure(ctx, ctx->ckeys, std::max<size_t>(m, 1) * 8);
  if (ctx->upper_src && m) {
    k_edge_derive_up<<<pc_grid(ctx, m, 256, 16), 256, 0, ctx->stream>>>(
        ctx->uoff.as<uint64_t>(), ctx->unbr.as<uint32_t>(), ctx->ucrow.as<uint32_t>(), m, ctx->n,
        ctx->vinfo.as<uint64_t>(), ctx->pmodel, ctx->t32, ctx->toff(), ctx->keys.as<uint64_t>(),
        ctx->ckeys.as<uint64_t>(), nullptr, nullptr, nullptr, nullptr, false);
    PC_CHECK_LAUNCH();
    ctx->launches++;
  } else if (nnz) {
    k_edge_derive<<<pc_grid(ctx, nnz, 256), 256, 0, ctx->stream>>>(
        ctx->off.as<uint64_t>(), ctx->nbr.as<uint32_t>(), ctx->crow.as<uint32_t>(), nnz,
        ctx->uoff.as<uint64_t>(), ctx->vinfo.as<uint64_t>(), ctx->pmodel, ctx->t32, ctx->toff(),
        ctx->keys.as<uint64_t>(), ctx->ckeys.as<uint64_t>(), nullptr, nullptr);
    PC_CHECK_LAUNCH();
    ctx->launches++;
  }
  ctx->elist_ok = true;
}

namespace {
// tcsr[e] = T32 - toff of CSR entry e = (u, w): WIC R4 from the two degrees
// (vinfo), Uniform R19 from the edge key
__global__ void k_tcsr(const uint64_t *off, const uint32_t *nbr, const uint32_t *crow, uint64_t nnz,
                       const uint64_t *vinfo, int pmodel, uint64_t t32, uint32_t toff,
                       uint32_t *tcsr) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (size_t)gridDim.x * blockDim.x) {
    const uint32_t u = entry_row(off, crow, e), w = nbr[e];
    uint64_t T;
    if (pmodel == PACIM_P_WIC) {
      T = (1ull << 33) / ((vinfo[u] >> 32) + (vinfo[w] >> 32));
      if (T > (1ull << 32)) T = 1ull << 32;
    } else {
      const uint64_t a = u < w ? u : w, b = u < w ? w : u;
      T = pc_t32_uniform(t32, (a << 32) | b);
    }
    tcsr[e] = (uint32_t)(T - toff);
  }
}
}  // namespace

void pc_ensure_tcsr(pacim_ctx *ctx) {
  pc_ensure_sym(ctx);  // every reader of tcsr reads the neighbour lists too
  if (ctx->pmodel == PACIM_P_CONST || ctx->tcsr_ok) return;
  const uint64_t nnz = 2 * ctx->m;
  pc_ensure(ctx, ctx->tcsr, std::max<size_t>(nnz, 1) * sizeof(uint32_t));
  if (nnz)
    k_tcsr<<<pc_grid(ctx, nnz, 256), 256, 0, ctx->stream>>>(
        ctx->off.as<uint64_t>(), ctx->nbr.as<uint32_t>(), ctx->crow.as<uint32_t>(), nnz,
        ctx->vinfo.as<uint64_t>(), ctx->pmodel, ctx->t32, ctx->toff(), ctx->tcsr.as<uint32_t>());
  PC_CHECK_LAUNCH();
  ctx->tcsr_ok = true;
}

static void derive_common(pacim_ctx *ctx) {
  if (ctx->lean) {
    derive_lean(ctx);
    return;
  }
  derive_rows(ctx);   // the store rows first: the edge pass writes edges as rows
  derive_edges(ctx);
}

// Lean graphs (c5 at full scale): no upper edge list and no
// row compaction — the store rows are the vertex ids (isolated vertices are
// singleton rows), k_edges reads the upper edges straight from the CSR
// through the chunk -> row table `crow`.  Constant probabilities only.
static void derive_lean(pacim_ctx *ctx) {
  pc_ensure_sym(ctx);  // k_edges reads the symmetric CSR
  const uint32_t n = ctx->n;
  uint64_t *off = ctx->off.as<uint64_t>();
  PC_REQUIRE(ctx->pmodel == PACIM_P_CONST, PACIM_ENOTIMPL,
             "lean graphs (no edge list) support the constant probability model only");
  pc_ensure(ctx, ctx->counters, 64 * 8);
  {  // hub: a maximum-degree vertex
    unsigned long long *t = ctx->counters.as<unsigned long long>();
    PC_CUDA(cudaMemsetAsync(t, 0, 8, ctx->stream));
    k_max_deg<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(off, n, t);
    PC_CHECK_LAUNCH();
    unsigned long long h = 0;
    PC_CUDA(cudaMemcpyAsync(&h, t, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->hub = (uint32_t)(0xFFFFFFFFull - (h & 0xFFFFFFFFull));
    ctx->hub_degree = h >> 32;
    if (ctx->hub >= n) ctx->hub = 0;
  }
  ctx->nr = n;
  ctx->ucsr = false;
  ctx->hub_row = ctx->hub;
  pc_ensure(ctx, ctx->cid, (size_t)n * 4);
  pc_ensure(ctx, ctx->rmap, (size_t)n * 4);
  k_iota_u32<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(ctx->cid.as<uint32_t>(), n);
  k_iota_u32<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(ctx->rmap.as<uint32_t>(), n);
  PC_CHECK_LAUNCH();
  make_crow(ctx, ctx->crow);
  {
    // the upper offsets and their chunk table: k_edges<…, 3> visits only the
    // upper entries (half the lanes of a pass over the full CSR)
    pc_ensure(ctx, ctx->scratch, ((size_t)n + 1) * 8);
    uint64_t *ucnt = ctx->scratch.as<uint64_t>();
    pc_ensure(ctx, ctx->uoff, ((size_t)n + 1) * 8);
    k_upper_count<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(off, ctx->nbr.as<uint32_t>(), n,
                                                               ucnt);
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaMemsetAsync(ucnt + n, 0, 8, ctx->stream));
    pc_exclusive_scan_u64(ctx, ucnt, ctx->uoff.as<uint64_t>(), (size_t)n + 1);
    pc_ensure(ctx, ctx->ucrow, ((ctx->m + 31) / 32 + 1) * 4);
    if (ctx->m) {
      k_crow_of<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(ctx->uoff.as<uint64_t>(), n,
                                                              ctx->ucrow.as<uint32_t>());
      PC_CHECK_LAUNCH();
    }
  }
  pc_free(ctx, ctx->keys);
  pc_free(ctx, ctx->ckeys);
  pc_free(ctx, ctx->hidx);
  pc_free(ctx, ctx->hub_tab);
  ctx->nhub = 0;
  ctx->hub_entries = 0;
  ctx->launches += 4;
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

// lean when asked (PACIM_LEAN=1) or when the edge lists (keys + ckeys, 16 B
// per upper edge) would take more than a third of the device
// (round 2, late: no longer by default — graphs whose edge lists do not fit
// take the CSR-direct form of the edge stream, which keeps the store-row
// compaction: c5's batch passes then skip the isolated vertices' rows)
static bool want_lean(pacim_ctx *ctx) {
  if (const char *e = getenv("PACIM_LEAN")) return atoi(e) != 0;
  return false;
}

void pc_graph_finish_load(pacim_ctx *ctx, int validate) {
  const uint32_t n = ctx->n;
  uint64_t *off = ctx->off.as<uint64_t>();
  uint32_t *nbr = ctx->nbr.as<uint32_t>();
  pc_ensure(ctx, ctx->counters, 64 * sizeof(uint64_t));
  if (validate) {
    uint32_t *bad = ctx->counters.as<uint32_t>();
    PC_CUDA(cudaMemsetAsync(bad, 0xFF, sizeof(uint32_t), ctx->stream));
    k_validate<<<pc_grid(ctx, (size_t)n * 32, 256), 256, 0, ctx->stream>>>(off, nbr, n, bad);
    PC_CHECK_LAUNCH();
    if (validate >= 2) {
      k_validate_sym<<<pc_grid(ctx, (size_t)n * 32, 256), 256, 0, ctx->stream>>>(off, nbr, n, bad);
      PC_CHECK_LAUNCH();
    }
    uint32_t hbad = 0;
    PC_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hbad != 0xFFFFFFFFu) {
      throw PacimError{PACIM_EINVAL,
                       "CSR invalid at vertex " + std::to_string(hbad) +
                           (validate >= 2 ? " (range/order/loop/duplicate/asymmetry)"
                                          : " (range/order/loop/duplicate)")};
    }
  }
  ctx->lean = want_lean(ctx);
  derive_common(ctx);
}

// --------------------------------------------------- upper CSR -> full CSR
// pacim_load_graph_upper (H0): the caller sends each undirected edge once, as
// the upper CSR (row u lists its neighbours v > u, sorted) — half the bytes of
// the symmetric CSR over PCIe — and the device builds the symmetric CSR.  The
// lower lists are the transpose: the upper entries (u, v) are in u order, so
// a STABLE radix sort of the pairs by v (CUB, LSD: ceil(log2 n) key bits)
// leaves every v's sources sorted; run boundaries of the sorted targets give
// the lower degrees; one lane-per-entry pass writes every row as [lower ++
// upper].  (Atomic cursors + a per-vertex segmented sort cost 255 ms at c4
// against the sort's tens of ms.)
namespace {
// validate = 1 for upper CSRs: offsets non-decreasing, rows strictly
// increasing, every neighbour in (u, n); *bad = the smallest bad vertex
__global__ void k_validate_upper(const uint64_t *uoff, const uint32_t *unbr, uint32_t n,
                                 uint32_t *bad) {
  for (size_t u = (size_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (size_t)gridDim.x * blockDim.x) {
    const uint64_t a = uoff[u], b = uoff[u + 1];
    bool ok = a <= b;
    for (uint64_t e = a; ok && e < b; e++) {
      const uint32_t v = unbr[e];
      ok = v > u && v < n && (e == a || v > unbr[e - 1]);
    }
    if (!ok) atomicMin(bad, (uint32_t)u);
  }
}

// the sort's input: keys = targets v (a copy: unbr is read again for the
// upper halves), values = sources u (row of entry e from the chunk table)
__global__ void k_upper_pairs(const uint64_t *uoff, const uint32_t *ucrow, const uint32_t *unbr,
                              uint64_t m, uint32_t *key, uint32_t *val) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (size_t)gridDim.x * blockDim.x) {
    uint32_t u = ucrow[e >> 5];
    while (e >= uoff[u + 1]) u++;
    key[e] = unbr[e];
    val[e] = u;
  }
}

// run boundaries of the sorted targets: lo[v] = first index, hi[v] = one
// past the last (both 0 for a vertex without lower neighbours)
__global__ void k_target_runs(const uint32_t *skey, uint64_t m, uint64_t *lo, uint64_t *hi) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t k = skey[i];
    if (i == 0 || skey[i - 1] != k) lo[k] = i;
    if (i + 1 == m || skey[i + 1] != k) hi[k] = i + 1;
  }
}

// deg[v] = upper + lower degree, lc[v] = lower degree (deg[n] = lc[n] = 0,
// for the exclusive scans)
__global__ void k_full_deg(const uint64_t *uoff, const uint64_t *lo, const uint64_t *hi,
                           uint32_t n, uint64_t *deg, uint64_t *lc) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
       v += (size_t)gridDim.x * blockDim.x) {
    const uint64_t l = v < n ? hi[v] - lo[v] : 0;
    deg[v] = v < n ? uoff[v + 1] - uoff[v] + l : 0;
    lc[v] = l;
  }
}

// row v of the symmetric CSR = its sorted lower list ++ its upper list
__global__ void k_full_rows(const uint64_t *off, const uint32_t *crow, uint64_t nnz,
                            const uint64_t *loff, const uint32_t *lsorted, const uint64_t *uoff,
                            const uint32_t *unbr, uint32_t *nbr) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (size_t)gridDim.x * blockDim.x) {
    uint32_t v = crow[e >> 5];
    while (e >= off[v + 1]) v++;
    const uint64_t i = e - off[v], nl = loff[v + 1] - loff[v];
    nbr[e] = i < nl ? lsorted[loff[v] + i] : unbr[uoff[v] + (i - nl)];
  }
}

// crow-style chunk table over any offsets array: row of entry 32 c
__global__ void k_crow_of(const uint64_t *off, uint32_t n, uint32_t *crow) {
  for (size_t u = (size_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (size_t)gridDim.x * blockDim.x) {
    const uint64_t c0 = (off[u] + 31) / 32, c1 = (off[u + 1] + 31) / 32;
    for (uint64_t c = c0; c < c1; c++) crow[c] = (uint32_t)u;
  }
}
}  // namespace

void pc_validate_upper(pacim_ctx *ctx, const uint64_t *d_uoff, const uint32_t *d_unbr, uint32_t n) {
  pc_ensure(ctx, ctx->counters, 64 * sizeof(uint64_t));
  uint32_t *bad = ctx->counters.as<uint32_t>();
  PC_CUDA(cudaMemsetAsync(bad, 0xFF, 4, ctx->stream));
  k_validate_upper<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(d_uoff, d_unbr, n, bad);
  PC_CHECK_LAUNCH();
  uint32_t h = 0;
  PC_CUDA(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h != 0xFFFFFFFFu)
    throw PacimError{PACIM_EINVAL, "upper CSR invalid at vertex " + std::to_string(h) +
                                       " (offsets/order/range: neighbours must be > u, < n, sorted)"};
}

void pc_sym_free(pacim_ctx *ctx) {
  for (DevBuf &d : ctx->sym) pc_free(ctx, d);
}

// d_uoff[n+1], d_unbr[m] (device, the upper CSR) -> ctx->off, ctx->nbr (the
// symmetric CSR, 2m entries), on the ctx stream; ctx->m = m already
void pc_symmetrize_upper(pacim_ctx *ctx, const uint64_t *d_uoff, const uint32_t *d_unbr,
                         uint32_t n, uint64_t m) {
  const uint64_t nnz = 2 * m;
  // PACIM_SYM_TIMES=1: phase times on stderr (diagnostics)
  const bool tm = getenv("PACIM_SYM_TIMES") != nullptr;
  std::vector<cudaEvent_t> evs;
  auto mark = [&]() {
    if (!tm) return;
    cudaEvent_t e;
    PC_CUDA(cudaEventCreate(&e));
    PC_CUDA(cudaEventRecord(e, ctx->stream));
    evs.push_back(e);
  };
  mark();
  pc_ensure(ctx, ctx->off, ((size_t)n + 1) * 8);
  pc_ensure(ctx, ctx->nbr, std::max<uint64_t>(nnz, 1) * 4);
  // scratch kept by the ctx (capacity reused by the next upper load: a
  // cudaMalloc / cudaFree of ~25 GB per load at c4 would cost more than the
  // sort); released by a load of the symmetric CSR
  DevBuf *sb = ctx->sym;
  DevBuf &lo = sb[0], &hi = sb[1], &deg = sb[2], &lc = sb[3], &loff = sb[4], &k0 = sb[5],
         &k1 = sb[6], &v0 = sb[7], &v1 = sb[8], &ucrow = sb[9], &stmp = sb[10];
  for (DevBuf *d : {&lo, &hi, &deg, &lc, &loff}) pc_ensure(ctx, *d, ((size_t)n + 1) * 8);
  PC_CUDA(cudaMemsetAsync(lo.p, 0, ((size_t)n + 1) * 8, ctx->stream));
  PC_CUDA(cudaMemsetAsync(hi.p, 0, ((size_t)n + 1) * 8, ctx->stream));
  uint64_t *off = ctx->off.as<uint64_t>();
  const uint32_t *lsorted = nullptr;
  if (m) {
    for (DevBuf *d : {&k0, &k1, &v0, &v1}) pc_ensure(ctx, *d, m * 4);
    pc_ensure(ctx, ucrow, ((m + 31) / 32 + 1) * 4);
    k_crow_of<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(d_uoff, n, ucrow.as<uint32_t>());
    PC_CHECK_LAUNCH();
    k_upper_pairs<<<pc_grid(ctx, m, 256, 16), 256, 0, ctx->stream>>>(
        d_uoff, ucrow.as<uint32_t>(), d_unbr, m, k0.as<uint32_t>(), v0.as<uint32_t>());
    PC_CHECK_LAUNCH();
    mark();
    const int bits = std::max(1, 32 - __builtin_clz(std::max(n - 1, 1u)));
    cub::DoubleBuffer<uint32_t> dk(k0.as<uint32_t>(), k1.as<uint32_t>()),
        dv(v0.as<uint32_t>(), v1.as<uint32_t>());
    size_t tb = 0;
    PC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int64_t)m, 0, bits, ctx->stream));
    pc_ensure(ctx, stmp, tb + 16);
    PC_CUDA(cub::DeviceRadixSort::SortPairs(stmp.p, tb, dk, dv, (int64_t)m, 0, bits, ctx->stream));
    mark();
    k_target_runs<<<pc_grid(ctx, m, 256, 16), 256, 0, ctx->stream>>>(
        dk.Current(), m, lo.as<uint64_t>(), hi.as<uint64_t>());
    PC_CHECK_LAUNCH();
    lsorted = dv.Current();
    ctx->launches += 4;
  }
  k_full_deg<<<pc_grid(ctx, (size_t)n + 1, 256), 256, 0, ctx->stream>>>(
      d_uoff, lo.as<uint64_t>(), hi.as<uint64_t>(), n, deg.as<uint64_t>(), lc.as<uint64_t>());
  PC_CHECK_LAUNCH();
  pc_exclusive_scan_u64(ctx, deg.as<uint64_t>(), off, (size_t)n + 1);
  pc_exclusive_scan_u64(ctx, lc.as<uint64_t>(), loff.as<uint64_t>(), (size_t)n + 1);
  ctx->launches += 3;
  mark();
  if (m) {
    make_crow(ctx, ctx->crow);
    k_full_rows<<<pc_grid(ctx, nnz, 256, 16), 256, 0, ctx->stream>>>(
        off, ctx->crow.as<uint32_t>(), nnz, loff.as<uint64_t>(), lsorted, d_uoff, d_unbr,
        ctx->nbr.as<uint32_t>());
    PC_CHECK_LAUNCH();
    ctx->launches += 1;
  }
  mark();
  if (tm) {
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    fprintf(stderr, "[symmetrize ms]");
    for (size_t i = 1; i < evs.size(); i++) {
      float x = 0;
      cudaEventElapsedTime(&x, evs[i - 1], evs[i]);
      fprintf(stderr, " %.3f", x);
    }
    fprintf(stderr, "  (pairs, sort, runs+degrees+scans, rows)\n");
    for (auto e : evs) cudaEventDestroy(e);
  }
}

void pc_upper_degrees(pacim_ctx *ctx) {
  const uint32_t n = ctx->n;
  const uint64_t m = ctx->m;
  DevBuf *sb = ctx->sym;  // the symmetrization's scratch (kept across upper loads)
  DevBuf &deg = sb[2], &lcnt = sb[3];
  pc_ensure(ctx, deg, ((size_t)n + 1) * 8);
  pc_ensure(ctx, lcnt, ((size_t)n + 1) * 8);
  pc_ensure(ctx, ctx->off, ((size_t)n + 1) * 8);
  PC_CUDA(cudaMemsetAsync(lcnt.p, 0, (size_t)n * 4, ctx->stream));
  pc_ensure(ctx, ctx->ucrow, ((m + 31) / 32 + 1) * 4);
  if (m) {
    k_crow_of<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(ctx->uoff.as<uint64_t>(), n,
                                                            ctx->ucrow.as<uint32_t>());
    PC_CHECK_LAUNCH();
    k_lower_hist<<<pc_grid(ctx, m, 256, 16), 256, 0, ctx->stream>>>(ctx->unbr.as<uint32_t>(), m,
                                                                   lcnt.as<uint32_t>());
    PC_CHECK_LAUNCH();
  }
  k_up_deg<<<pc_grid(ctx, (size_t)n + 1, 256), 256, 0, ctx->stream>>>(
      ctx->uoff.as<uint64_t>(), lcnt.as<uint32_t>(), n, deg.as<uint64_t>());
  PC_CHECK_LAUNCH();
  pc_exclusive_scan_u64(ctx, deg.as<uint64_t>(), ctx->off.as<uint64_t>(), (size_t)n + 1);
  ctx->launches += 4;
  ctx->upper_src = true;
  ctx->sym_pending = true;
}

void pc_ensure_sym(pacim_ctx *ctx) {
  if (!ctx->sym_pending) return;
  pc_symmetrize_upper(ctx, ctx->uoff.as<uint64_t>(), ctx->unbr.as<uint32_t>(), ctx->n, ctx->m);
  ctx->sym_pending = false;
}

// ------------------------------------------------------------- generators
namespace {
// ER candidate j: u = (lo32(w) n) >> 32, v = (hi32(w) n) >> 32 (loop -> ~0).
__global__ void k_gen_er(uint64_t Kg, uint32_t n, uint64_t j0, uint64_t J, uint64_t *key,
                         uint64_t *idx) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < J;
       t += (size_t)gridDim.x * blockDim.x) {
    uint64_t j = j0 + t;
    uint64_t w = pc_mix64(Kg ^ j);
    uint32_t u = (uint32_t)(((w & 0xFFFFFFFFull) * n) >> 32);
    uint32_t v = (uint32_t)(((w >> 32) * n) >> 32);
    uint64_t a = u < v ? u : v, b = u < v ? v : u;
    key[t] = (u == v) ? ~0ull : ((a << 32) | b);
    idx[t] = j;
  }
}

__device__ __forceinline__ uint64_t rmat_perm(uint64_t x, int s) {
  uint64_t mask = (s >= 64) ? ~0ull : ((1ull << s) - 1);
  int sh = (s + 1) / 2;
  x = (x * 0x9E3779B97F4A7C15ull) & mask;
  x ^= x >> sh;
  x = (x * 0xBF58476D1CE4E5B9ull) & mask;
  x ^= x >> sh;
  return x;
}

// R-MAT sample i: per level l, y = mix64(Kg ^ (i*64+l)) >> 11 picks the
// quadrant against 53-bit thresholds; level l sets bit scale-1-l.
// Bucketed R-MAT (the same samples as k_gen_rmat): the directed pairs
// (src << 32 | dst) of every non-loop sample in both orientations whose
// source lies in bucket b (top `bbits` of the scale-bit id), appended at a
// warp-aggregated cursor (order irrelevant: the bucket is sorted next).
// count_only: just count them.
__global__ void k_gen_rmat_bucket(uint64_t Kg, int scale, uint64_t ns, uint64_t ta, uint64_t tab,
                                  uint64_t tabc, int permute, int bbits, uint32_t b,
                                  unsigned long long *cursor, uint64_t *out, int count_only) {
  const int lane = threadIdx.x & 31;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(size_t)31; base < ns;
       base += (size_t)gridDim.x * blockDim.x) {
    const uint64_t i = base + lane;
    uint64_t u = 0, v = 0;
    bool ok = i < ns;
    if (ok) {
      for (int l = 0; l < scale; l++) {
        uint64_t y = pc_mix64(Kg ^ (i * 64 + (uint64_t)l)) >> 11;
        uint64_t bit = 1ull << (scale - 1 - l);
        if (y < ta) {
        } else if (y < tab) {
          v |= bit;
        } else if (y < tabc) {
          u |= bit;
        } else {
          u |= bit;
          v |= bit;
        }
      }
      if (permute) {
        u = rmat_perm(u, scale);
        v = rmat_perm(v, scale);
      }
      ok = u != v;
    }
    const bool eu = ok && (uint32_t)(u >> (scale - bbits)) == b;
    const bool ev = ok && (uint32_t)(v >> (scale - bbits)) == b;
    const uint32_t mine = (eu ? 1u : 0u) + (ev ? 1u : 0u);
    uint32_t pre = mine;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, pre, d);
      if (lane >= d) pre += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
    if (!tot) continue;
    unsigned long long at = 0;
    if (lane == 31) at = atomicAdd(cursor, (unsigned long long)tot);
    at = __shfl_sync(0xffffffffu, at, 31) + (pre - mine);
    if (!count_only) {
      if (eu) out[at++] = (u << 32) | v;
      if (ev) out[at] = (v << 32) | u;
    }
  }
}

// degrees of the bucket's sources from its sorted distinct pairs
__global__ void k_bucket_deg(const uint64_t *p, uint64_t N, uint64_t lo, uint64_t *deg) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long *)(deg + ((p[i] >> 32) - lo)), 1ull);
}
__global__ void k_bucket_nbr(const uint64_t *p, uint64_t N, uint32_t *nbr) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    nbr[i] = (uint32_t)p[i];
}
__global__ void k_add_u64(uint64_t *a, uint64_t N, uint64_t x) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    a[i] += x;
}

// lean graphs: the row of the first CSR entry of every 32-entry chunk
// thread per row: the chunks whose first entry lies in the row (stores only,
// so a hub's many chunks do not stall its thread)
__global__ void k_crow(const uint64_t *off, uint32_t n, uint32_t *crow) {
  for (size_t u = (size_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (size_t)gridDim.x * blockDim.x) {
    const uint64_t c0 = (off[u] + 31) / 32, c1 = (off[u + 1] + 31) / 32;
    for (uint64_t c = c0; c < c1; c++) crow[c] = (uint32_t)u;
  }
}
__global__ void k_iota_u32(uint32_t *a, uint32_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

__global__ void k_gen_rmat(uint64_t Kg, int scale, uint64_t i0, uint64_t cnt, uint64_t ta,
                           uint64_t tab, uint64_t tabc, int permute, uint64_t *key) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
       t += (size_t)gridDim.x * blockDim.x) {
    uint64_t i = i0 + t, u = 0, v = 0;
    for (int l = 0; l < scale; l++) {
      uint64_t y = pc_mix64(Kg ^ (i * 64 + (uint64_t)l)) >> 11;
      uint64_t bit = 1ull << (scale - 1 - l);
      if (y < ta) {
      } else if (y < tab) {
        v |= bit;
      } else if (y < tabc) {
        u |= bit;
      } else {
        u |= bit;
        v |= bit;
      }
    }
    if (permute) {
      u = rmat_perm(u, scale);
      v = rmat_perm(v, scale);
    }
    uint64_t a = u < v ? u : v, b = u < v ? v : u;
    key[t] = (u == v) ? ~0ull : ((a << 32) | b);
  }
}

// Grid: per vertex, count of edges to larger ids (right, down, diagonal).
__device__ __forceinline__ int grid_edges(uint64_t Kg, uint32_t W, uint32_t H, uint64_t d32,
                                          uint64_t v, uint64_t *out) {
  uint64_t i = v / W, j = v % W;
  int c = 0;
  if (j + 1 < W) out[c++] = (v << 32) | (v + 1);
  if (i + 1 < H) out[c++] = (v << 32) | (v + W);
  if (i + 1 < H && j + 1 < W && (pc_mix64(Kg ^ v) >> 32) < d32) out[c++] = (v << 32) | (v + W + 1);
  return c;
}

__global__ void k_grid_count(uint64_t Kg, uint32_t W, uint32_t H, uint64_t d32, uint64_t *cnt) {
  uint64_t nv = (uint64_t)W * H;
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
       v += (size_t)gridDim.x * blockDim.x) {
    uint64_t tmp[3];
    cnt[v] = grid_edges(Kg, W, H, d32, v, tmp);
  }
}

__global__ void k_grid_fill(uint64_t Kg, uint32_t W, uint32_t H, uint64_t d32,
                            const uint64_t *start, uint64_t *keys) {
  uint64_t nv = (uint64_t)W * H;
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
       v += (size_t)gridDim.x * blockDim.x) {
    uint64_t tmp[3];
    int c = grid_edges(Kg, W, H, d32, v, tmp);
    for (int q = 0; q < c; q++) keys[start[v] + q] = tmp[q];
  }
}

// first-occurrence flag of sorted keys (excluding the ~0 loop sentinel)
__global__ void k_first_flag(const uint64_t *k, uint64_t N, uint64_t *flag) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (size_t)gridDim.x * blockDim.x)
    flag[t] = (k[t] != ~0ull && (t == 0 || k[t] != k[t - 1])) ? 1 : 0;
}

__global__ void k_compact2(const uint64_t *k, const uint64_t *v, const uint64_t *flag,
                           const uint64_t *pos, uint64_t N, uint64_t *ko, uint64_t *vo) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (size_t)gridDim.x * blockDim.x)
    if (flag[t]) {
      ko[pos[t]] = k[t];
      if (v) vo[pos[t]] = v[t];
    }
}

// CSR from sorted distinct keys: degree histograms.
__global__ void k_deg_hist(const uint64_t *keys, uint64_t m, uint64_t *dlo, uint64_t *dhi) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (size_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[e];
    atomicAdd((unsigned long long *)&dhi[k >> 32], 1ull);
    atomicAdd((unsigned long long *)&dlo[k & 0xFFFFFFFFull], 1ull);
  }
}

__global__ void k_add2(const uint64_t *a, const uint64_t *b, uint64_t *c, uint64_t N) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (size_t)gridDim.x * blockDim.x)
    c[t] = a[t] + b[t];
}

// upper half of row a: position e - hstart[a] after the dlo[a] lower entries
__global__ void k_fill_hi(const uint64_t *keys, uint64_t m, const uint64_t *off,
                          const uint64_t *dlo, const uint64_t *hstart, uint32_t *nbr) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (size_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[e];
    uint32_t a = (uint32_t)(k >> 32), b = (uint32_t)k;
    nbr[off[a] + dlo[a] + (e - hstart[a])] = b;
  }
}

// lower half of row b from the (b, a)-sorted swapped keys
__global__ void k_fill_lo(const uint64_t *sw, uint64_t m, const uint64_t *off,
                          const uint64_t *lstart, uint32_t *nbr) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (size_t)gridDim.x * blockDim.x) {
    uint64_t k = sw[e];
    uint32_t b = (uint32_t)(k >> 32), a = (uint32_t)k;
    nbr[off[b] + (e - lstart[b])] = a;
  }
}

__global__ void k_swap_halves(const uint64_t *in, uint64_t *out, uint64_t m) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (size_t)gridDim.x * blockDim.x) {
    uint64_t k = in[e];
    out[e] = (k << 32) | (k >> 32);
  }
}
}  // namespace

static void sort_keys(pacim_ctx *ctx, uint64_t *keys, uint64_t *alt, uint64_t N, int end_bit,
                      uint64_t **result) {
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  size_t tmp = 0;
  PC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, (int64_t)N, 0, end_bit, ctx->stream));
  TmpBuf t(ctx);
  pc_ensure(ctx, t, tmp + 16);
  PC_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, db, (int64_t)N, 0, end_bit, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  pc_free(ctx, t);
  *result = db.Current();
}

static void sort_pairs(pacim_ctx *ctx, uint64_t *k, uint64_t *k2, uint64_t *v, uint64_t *v2,
                       uint64_t N, int end_bit, uint64_t **rk, uint64_t **rv) {
  cub::DoubleBuffer<uint64_t> dk(k, k2), dv(v, v2);
  size_t tmp = 0;
  PC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, (int64_t)N, 0, end_bit,
                                          ctx->stream));
  TmpBuf t(ctx);
  pc_ensure(ctx, t, tmp + 16);
  PC_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, dk, dv, (int64_t)N, 0, end_bit, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  pc_free(ctx, t);
  *rk = dk.Current();
  *rv = dv.Current();
}

// Unique sorted keys of k[0..N) into out; returns count.  Uses flag/pos scratch.
static uint64_t unique_sorted(pacim_ctx *ctx, const uint64_t *k, const uint64_t *v, uint64_t N,
                              uint64_t *ko, uint64_t *vo) {
  TmpBuf flag(ctx), pos(ctx);
  pc_ensure(ctx, flag, (N + 1) * sizeof(uint64_t));
  pc_ensure(ctx, pos, (N + 1) * sizeof(uint64_t));
  unsigned g = pc_grid(ctx, N, 256);
  k_first_flag<<<g, 256, 0, ctx->stream>>>(k, N, flag.as<uint64_t>());
  PC_CHECK_LAUNCH();
  pc_exclusive_scan_u64(ctx, flag.as<uint64_t>(), pos.as<uint64_t>(), N + 1);
  uint64_t cnt = 0;
  PC_CUDA(cudaMemcpyAsync(&cnt, pos.as<uint64_t>() + N, 8, cudaMemcpyDeviceToHost, ctx->stream));
  k_compact2<<<g, 256, 0, ctx->stream>>>(k, v, flag.as<uint64_t>(), pos.as<uint64_t>(), N, ko, vo);
  PC_CHECK_LAUNCH();
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  pc_free(ctx, flag);
  pc_free(ctx, pos);
  return cnt;
}

// Build the full CSR (off, nbr) from ctx->keys (sorted distinct, m entries).
static void csr_from_keys(pacim_ctx *ctx) {
  const uint32_t n = ctx->n;
  const uint64_t m = ctx->m;
  pc_ensure(ctx, ctx->off, ((size_t)n + 1) * sizeof(uint64_t));
  pc_ensure(ctx, ctx->nbr, std::max<size_t>(2 * m, 1) * sizeof(uint32_t));
  TmpBuf d(ctx);
  pc_ensure(ctx, d, 5 * ((size_t)n + 1) * sizeof(uint64_t));
  uint64_t *dlo = d.as<uint64_t>(), *dhi = dlo + n + 1, *deg = dhi + n + 1, *lstart = deg + n + 1,
           *hstart = lstart + n + 1;
  PC_CUDA(cudaMemsetAsync(dlo, 0, 2 * ((size_t)n + 1) * sizeof(uint64_t), ctx->stream));
  uint64_t *keys = ctx->keys.as<uint64_t>();
  k_deg_hist<<<pc_grid(ctx, m, 256), 256, 0, ctx->stream>>>(keys, m, dlo, dhi);
  PC_CHECK_LAUNCH();
  k_add2<<<pc_grid(ctx, n + 1, 256), 256, 0, ctx->stream>>>(dlo, dhi, deg, (uint64_t)n + 1);
  PC_CHECK_LAUNCH();
  pc_exclusive_scan_u64(ctx, deg, ctx->off.as<uint64_t>(), (size_t)n + 1);
  pc_exclusive_scan_u64(ctx, dlo, lstart, n);
  pc_exclusive_scan_u64(ctx, dhi, hstart, n);
  k_fill_hi<<<pc_grid(ctx, m, 256), 256, 0, ctx->stream>>>(keys, m, ctx->off.as<uint64_t>(), dlo,
                                                          hstart, ctx->nbr.as<uint32_t>());
  PC_CHECK_LAUNCH();
  TmpBuf sw(ctx), sw2(ctx);
  pc_ensure(ctx, sw, std::max<size_t>(m, 1) * sizeof(uint64_t));
  pc_ensure(ctx, sw2, std::max<size_t>(m, 1) * sizeof(uint64_t));
  k_swap_halves<<<pc_grid(ctx, m, 256), 256, 0, ctx->stream>>>(keys, sw.as<uint64_t>(), m);
  PC_CHECK_LAUNCH();
  uint64_t *sorted = nullptr;
  sort_keys(ctx, sw.as<uint64_t>(), sw2.as<uint64_t>(), m, 64, &sorted);
  k_fill_lo<<<pc_grid(ctx, m, 256), 256, 0, ctx->stream>>>(sorted, m, ctx->off.as<uint64_t>(),
                                                          lstart, ctx->nbr.as<uint32_t>());
  PC_CHECK_LAUNCH();
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  pc_free(ctx, sw);
  pc_free(ctx, sw2);
  pc_free(ctx, d);
}

// R-MAT generated one source-id bucket at a time (sizes beyond one sort, c5):
// per bucket every sample is drawn again, the pairs whose source is in the
// bucket kept (both orientations: the symmetric CSR directly), sorted,
// deduplicated and appended.  Same edge set as the all-at-once path.
static void gen_rmat_bucketed(pacim_ctx *ctx, uint64_t Kg, int scale, uint64_t ns,
                              const uint64_t *params, int bbits) {
  const uint32_t n = ctx->n, NB = 1u << bbits;
  const uint64_t per = (uint64_t)n / NB;  // sources per bucket
  TmpBuf cur(ctx);
  pc_ensure(ctx, cur, 64);
  unsigned long long *cursor = cur.as<unsigned long long>();
  const unsigned g = pc_grid(ctx, ns, 256, 16);
  // pass 0: directed pairs per bucket (capacity of nbr and the bucket buffers)
  std::vector<unsigned long long> cnt(NB);
  for (uint32_t b = 0; b < NB; b++) {
    PC_CUDA(cudaMemsetAsync(cursor, 0, 8, ctx->stream));
    k_gen_rmat_bucket<<<g, 256, 0, ctx->stream>>>(Kg, scale, ns, params[2], params[3], params[4],
                                                  (int)params[5], bbits, b, cursor, nullptr, 1);
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaMemcpyAsync(&cnt[b], cursor, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  unsigned long long tot = 0, mx = 0;
  for (auto c : cnt) {
    tot += c;
    mx = std::max(mx, c);
  }
  pc_free(ctx, ctx->keys);
  pc_free(ctx, ctx->ckeys);
  pc_ensure(ctx, ctx->off, ((size_t)n + 1) * 8);
  pc_ensure(ctx, ctx->nbr, std::max<size_t>(tot, 1) * 4);
  TmpBuf pa(ctx), pb(ctx), deg(ctx);
  pc_ensure(ctx, pa, std::max<size_t>(mx, 1) * 8);
  pc_ensure(ctx, pb, std::max<size_t>(mx, 1) * 8);
  pc_ensure(ctx, deg, (per + 1) * 8);
  uint64_t *off = ctx->off.as<uint64_t>();
  uint64_t base = 0;
  for (uint32_t b = 0; b < NB; b++) {
    PC_CUDA(cudaMemsetAsync(cursor, 0, 8, ctx->stream));
    k_gen_rmat_bucket<<<g, 256, 0, ctx->stream>>>(Kg, scale, ns, params[2], params[3], params[4],
                                                  (int)params[5], bbits, b, cursor, pa.as<uint64_t>(),
                                                  0);
    PC_CHECK_LAUNCH();
    uint64_t *sk = nullptr;
    sort_keys(ctx, pa.as<uint64_t>(), pb.as<uint64_t>(), cnt[b], 64, &sk);
    uint64_t *other = sk == pa.as<uint64_t>() ? pb.as<uint64_t>() : pa.as<uint64_t>();
    const uint64_t u = cnt[b] ? unique_sorted(ctx, sk, nullptr, cnt[b], other, nullptr) : 0;
    // rows [b * per, (b + 1) * per): degrees -> offsets (+ base), neighbours
    PC_CUDA(cudaMemsetAsync(deg.p, 0, (per + 1) * 8, ctx->stream));
    if (u) {
      k_bucket_deg<<<pc_grid(ctx, u, 256), 256, 0, ctx->stream>>>(other, u, (uint64_t)b * per,
                                                                  deg.as<uint64_t>());
      PC_CHECK_LAUNCH();
      k_bucket_nbr<<<pc_grid(ctx, u, 256), 256, 0, ctx->stream>>>(other, u,
                                                                  ctx->nbr.as<uint32_t>() + base);
      PC_CHECK_LAUNCH();
    }
    pc_exclusive_scan_u64(ctx, deg.as<uint64_t>(), off + (size_t)b * per, per);
    k_add_u64<<<pc_grid(ctx, per, 256), 256, 0, ctx->stream>>>(off + (size_t)b * per, per, base);
    PC_CHECK_LAUNCH();
    base += u;
  }
  PC_CUDA(cudaMemcpyAsync(off + n, &base, 8, cudaMemcpyHostToDevice, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->m = base / 2;
  ctx->launches += 5 * NB;
}

void pc_generate(pacim_ctx *ctx, int kind, const uint64_t *params, int nparams,
                 uint64_t gen_seed) {
  uint64_t Kg = pc_mix64(gen_seed ^ 0xD1B54A32D192ED03ull);
  if (kind == PACIM_GEN_ER) {
    PC_REQUIRE(nparams >= 2, PACIM_EINVAL, "ER needs params {n, m}");
    uint64_t n = params[0], m = params[1];
    PC_REQUIRE(n >= 2 && n < (1ull << 31), PACIM_EINVAL, "ER: n out of range");
    PC_REQUIRE(m >= 1 && m <= n * (n - 1) / 4, PACIM_EINVAL, "ER: m must be <= n(n-1)/4");
    ctx->n = (uint32_t)n;
    uint64_t J = m + m / 4 + 1024;
    for (;;) {
      TmpBuf a(ctx), b(ctx), c(ctx), d2(ctx), ko(ctx), vo(ctx);
      pc_ensure(ctx, a, J * 8); pc_ensure(ctx, b, J * 8);
      pc_ensure(ctx, c, J * 8); pc_ensure(ctx, d2, J * 8);
      k_gen_er<<<pc_grid(ctx, J, 256), 256, 0, ctx->stream>>>(Kg, (uint32_t)n, 0, J,
                                                             a.as<uint64_t>(), b.as<uint64_t>());
      PC_CHECK_LAUNCH();
      uint64_t *sk, *sv;
      sort_pairs(ctx, a.as<uint64_t>(), c.as<uint64_t>(), b.as<uint64_t>(), d2.as<uint64_t>(), J,
                 64, &sk, &sv);
      // first occurrence (smallest j, stable sort) of each distinct pair
      pc_ensure(ctx, ko, J * 8); pc_ensure(ctx, vo, J * 8);
      uint64_t cnt = unique_sorted(ctx, sk, sv, J, ko.as<uint64_t>(), vo.as<uint64_t>());
      if (cnt < m) {
        J *= 2;
        continue;
      }
      // order the distinct pairs by their first draw index j; keep the first m
      uint64_t *rk, *rv;
      sort_pairs(ctx, vo.as<uint64_t>(), a.as<uint64_t>(), ko.as<uint64_t>(), b.as<uint64_t>(),
                 cnt, 64, &rk, &rv);
      pc_ensure(ctx, ctx->keys, m * 8);
      PC_CUDA(cudaMemcpyAsync(ctx->keys.p, rv, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      uint64_t *fin;
      sort_keys(ctx, ctx->keys.as<uint64_t>(), c.as<uint64_t>(), m, 64, &fin);
      if (fin != ctx->keys.as<uint64_t>())
        PC_CUDA(cudaMemcpyAsync(ctx->keys.p, fin, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      PC_CUDA(cudaStreamSynchronize(ctx->stream));
      ctx->m = m;
      break;
    }
  } else if (kind == PACIM_GEN_RMAT) {
    PC_REQUIRE(nparams >= 6, PACIM_EINVAL, "RMAT needs {scale, ef, ta, tab, tabc, permute}");
    int scale = (int)params[0];
    uint64_t ef = params[1];
    PC_REQUIRE(scale >= 1 && scale <= 30, PACIM_EINVAL, "RMAT: scale must be in [1, 30]");
    PC_REQUIRE(ef >= 1 && ef <= 64, PACIM_EINVAL, "RMAT: ef must be in [1, 64]");
    ctx->n = 1u << scale;
    uint64_t ns = ef << scale;
    // all samples sorted at once needs ~32 B per sample; else source buckets
    int bbits = 0;
    if (const char *e = getenv("PACIM_GEN_BUCKETS")) {
      while ((1 << bbits) < atoi(e) && bbits < scale) bbits++;
    } else {
      size_t fr = 0, tot = 0;
      pc_mem_info(ctx, &fr, &tot);
      if (32 * ns > fr / 3)  // a bucket holds ~2 ns / NB pairs at 32 B each in flight
        while (bbits < scale && ((64 * ns) >> bbits) > fr / 3) bbits++;
    }
    if (bbits > 0) {
      gen_rmat_bucketed(ctx, Kg, scale, ns, params, bbits);
      ctx->lean = want_lean(ctx);
      if (!ctx->lean) {  // the upper edge list from the CSR, as for a loaded graph
        pc_graph_finish_load(ctx, 0);
        return;
      }
      derive_common(ctx);
      return;
    }
    TmpBuf a(ctx), b(ctx);
    pc_ensure(ctx, a, ns * 8);
    pc_ensure(ctx, b, ns * 8);
    k_gen_rmat<<<pc_grid(ctx, ns, 256, 16), 256, 0, ctx->stream>>>(
        Kg, scale, 0, ns, params[2], params[3], params[4], (int)params[5], a.as<uint64_t>());
    PC_CHECK_LAUNCH();
    uint64_t *sk;
    sort_keys(ctx, a.as<uint64_t>(), b.as<uint64_t>(), ns, 64, &sk);
    uint64_t *other = (sk == a.as<uint64_t>()) ? b.as<uint64_t>() : a.as<uint64_t>();
    uint64_t cnt = unique_sorted(ctx, sk, nullptr, ns, other, nullptr);
    pc_free(ctx, ctx->keys);
    pc_ensure(ctx, ctx->keys, std::max<uint64_t>(cnt, 1) * 8);
    PC_CUDA(cudaMemcpyAsync(ctx->keys.p, other, cnt * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    pc_free(ctx, a);
    pc_free(ctx, b);
    ctx->m = cnt;
  } else if (kind == PACIM_GEN_GRID) {
    PC_REQUIRE(nparams >= 3, PACIM_EINVAL, "GRID needs {W, H, d32}");
    uint64_t W = params[0], H = params[1], d32 = params[2];
    PC_REQUIRE(W >= 1 && H >= 1 && W * H < (1ull << 31), PACIM_EINVAL, "GRID: bad size");
    ctx->n = (uint32_t)(W * H);
    TmpBuf cnt(ctx), start(ctx);
    pc_ensure(ctx, cnt, (W * H + 1) * 8);
    pc_ensure(ctx, start, (W * H + 1) * 8);
    k_grid_count<<<pc_grid(ctx, W * H, 256), 256, 0, ctx->stream>>>(Kg, (uint32_t)W, (uint32_t)H,
                                                                   d32, cnt.as<uint64_t>());
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaMemsetAsync(cnt.as<uint64_t>() + W * H, 0, 8, ctx->stream));
    pc_exclusive_scan_u64(ctx, cnt.as<uint64_t>(), start.as<uint64_t>(), W * H + 1);
    uint64_t m = 0;
    PC_CUDA(cudaMemcpyAsync(&m, start.as<uint64_t>() + W * H, 8, cudaMemcpyDeviceToHost,
                            ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    pc_ensure(ctx, ctx->keys, std::max<uint64_t>(m, 1) * 8);
    k_grid_fill<<<pc_grid(ctx, W * H, 256), 256, 0, ctx->stream>>>(
        Kg, (uint32_t)W, (uint32_t)H, d32, start.as<uint64_t>(), ctx->keys.as<uint64_t>());
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    pc_free(ctx, cnt);
    pc_free(ctx, start);
    ctx->m = m;
  } else {
    throw PacimError{PACIM_EINVAL, "unknown generator kind"};
  }
  csr_from_keys(ctx);
  ctx->lean = getenv("PACIM_LEAN") && atoi(getenv("PACIM_LEAN")) != 0 &&
              ctx->pmodel == PACIM_P_CONST;  // tests force the lean path on small graphs
  derive_common(ctx);
}
