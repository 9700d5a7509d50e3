// mc.cu — NEXT f3: Monte-Carlo influence sigma(S) under the IC model
// (the paper's "Influence ... 20000 simulations" column).
//
// R21: simulation i is a fresh world: edge e = (u, v) is live iff
//   hi32(mix64(mix64(K_mc ^ i) ^ (min<<32 | max))) < T32(e),
// K_mc = mix64(mc_seed ^ 0x4D435349434D4353), T32 = 2^32 always live.
// sigma_hat(S) = (sum over simulations of |reach_i(S)|) / nsims.
//
// One level-synchronous BFS carries MC_W x 32 simulations at once: every
// vertex has MC_W visited words and MC_W frontier words (bit b of word wd =
// simulation 32 * wd + b of the batch).  A warp expands one frontier vertex:
// lanes over its CSR entries, and for each entry only the simulations in the
// vertex's frontier mask are tested (one mix64 per (entry, simulation)).
#include <algorithm>
#include <vector>

#include "pacim_internal.cuh"

namespace {

constexpr int MC_W = 8;  // words per vertex: 256 simulations per batch
constexpr uint32_t NONE = 0xFFFFFFFFu;

struct Mc {
  const uint64_t *off;
  const uint32_t *nbr;
  const uint32_t *tcsr;  // per-edge models: T32 - toff
  uint32_t toff;
  int per_edge;
  uint64_t t32;
  uint32_t n;
  uint32_t *vis;        // n x MC_W
  uint32_t *fm;         // [2][n x MC_W] frontier masks
  uint32_t *flag;       // [2][n] vertex is in that level's list
  uint32_t *list;       // [2][n]
  uint32_t *cnt;        // [2] list sizes (cnt[nxt] reset by the host)
  const unsigned long long *Ki;  // MC_W * 32 per-simulation keys of the batch
};

__global__ void __launch_bounds__(256) k_mc_level(Mc M, uint32_t cur) {
  __shared__ unsigned long long ki[MC_W * 32];
  for (int i = threadIdx.x; i < MC_W * 32; i += blockDim.x) ki[i] = M.Ki[i];
  __syncthreads();
  const uint32_t nxt = cur ^ 1;
  const int lane = threadIdx.x & 31;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t nl = __ldcg(M.cnt + cur);
  uint32_t *fm_cur = M.fm + (size_t)cur * M.n * MC_W, *fm_nxt = M.fm + (size_t)nxt * M.n * MC_W;
  for (size_t t = warp; t < nl; t += nw) {
    const uint32_t x = __ldcg(M.list + (size_t)cur * M.n + t);
    uint32_t mk[MC_W];
#pragma unroll
    for (int wd = 0; wd < MC_W; wd++) mk[wd] = __ldcg(fm_cur + (size_t)x * MC_W + wd);
    __syncwarp();
    if (lane < MC_W) fm_cur[(size_t)x * MC_W + lane] = 0;  // consumed
    if (lane == 0) M.flag[(size_t)cur * M.n + x] = 0;
    const uint64_t e1 = M.off[x + 1];
    for (uint64_t e = M.off[x] + lane; e < e1; e += 32) {
      const uint32_t w = M.nbr[e];
      const uint64_t T = M.per_edge ? (uint64_t)M.tcsr[e] + M.toff : M.t32;
      if (T == 0) continue;
      const uint64_t key = x < w ? ((uint64_t)x << 32) | w : ((uint64_t)w << 32) | x;
      bool pushed = false;
#pragma unroll
      for (int wd = 0; wd < MC_W; wd++) {
        const uint32_t m = mk[wd];
        if (!m) continue;
        uint32_t live = m;
        if (T < (1ull << 32)) {
          live = 0;
          for (uint32_t b = m; b; b &= b - 1) {
            const int bit = __ffs(b) - 1;
            if ((pc_mix64(ki[wd * 32 + bit] ^ key) >> 32) < T) live |= 1u << bit;
          }
          if (!live) continue;
        }
        const uint32_t old = atomicOr(M.vis + (size_t)w * MC_W + wd, live);
        const uint32_t nb = live & ~old;
        if (!nb) continue;
        atomicOr(fm_nxt + (size_t)w * MC_W + wd, nb);
        if (!pushed) {
          pushed = true;
          if (atomicExch(M.flag + (size_t)nxt * M.n + w, 1u) == 0u)
            M.list[(size_t)nxt * M.n + atomicAdd(M.cnt + nxt, 1u)] = w;
        }
      }
    }
  }
}

// the batch's seeds: visited and in the first frontier in every simulation
__global__ void k_mc_seeds(Mc M, const uint32_t *seeds, uint32_t ns, uint32_t last_mask_words,
                           uint32_t last_mask) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ns * MC_W;
       t += gridDim.x * blockDim.x) {
    const uint32_t s = seeds[t / MC_W], wd = t % MC_W;
    const uint32_t m = wd < last_mask_words - 1 ? 0xFFFFFFFFu
                       : wd == last_mask_words - 1 ? last_mask : 0u;
    M.vis[(size_t)s * MC_W + wd] = m;
    M.fm[(size_t)s * MC_W + wd] = m;
    if (wd == 0) {
      M.flag[s] = 1;
      M.list[t / MC_W] = s;
    }
  }
}

__global__ void k_mc_count(const uint32_t *vis, size_t words, unsigned long long *total) {
  unsigned long long c = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (size_t)gridDim.x * blockDim.x)
    c += __popc(vis[i]);
  for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}

}  // namespace

void pc_simulate_ic(pacim_ctx *ctx, const uint32_t *seeds_host, uint32_t ns, uint32_t nsims,
                    uint64_t mc_seed, uint64_t *total_out) {
  const uint32_t n = ctx->n;
  // distinct seeds (a repeated seed is one start vertex)
  std::vector<uint32_t> sd(seeds_host, seeds_host + ns);
  std::sort(sd.begin(), sd.end());
  sd.erase(std::unique(sd.begin(), sd.end()), sd.end());
  for (uint32_t s : sd) PC_REQUIRE(s < n, PACIM_EINVAL, "seed id >= n");
  ns = (uint32_t)sd.size();
  const size_t vw = (size_t)n * MC_W;
  TmpBuf buf(ctx);
  // vis, fm[2], flag[2], list[2], cnt[2] (+pad), Ki, seeds, total
  const size_t words = 3 * vw + 4 * (size_t)n + 4 + 2 * MC_W * 32 + ns + 4;
  pc_ensure(ctx, buf, words * 4);
  uint32_t *base = buf.as<uint32_t>();
  Mc M;
  pc_ensure_tcsr(ctx);  // (and the symmetric lists of an upper-loaded graph)
  M.off = ctx->off.as<uint64_t>();
  M.nbr = ctx->nbr.as<uint32_t>();
  M.per_edge = ctx->pmodel != PACIM_P_CONST;
  pc_ensure_tcsr(ctx);
  M.tcsr = ctx->tcsr.as<uint32_t>();
  M.toff = ctx->toff();
  M.t32 = ctx->t32;
  M.n = n;
  M.vis = base;
  M.fm = base + vw;
  M.flag = base + 3 * vw;
  M.list = M.flag + 2 * (size_t)n;
  M.cnt = M.list + 2 * (size_t)n;
  unsigned long long *Ki = reinterpret_cast<unsigned long long *>(M.cnt + 4);
  M.Ki = Ki;
  uint32_t *d_seeds = reinterpret_cast<uint32_t *>(Ki + MC_W * 32);
  unsigned long long *d_total = reinterpret_cast<unsigned long long *>(d_seeds + ns + (ns & 1));
  PC_CUDA(cudaMemsetAsync(base, 0, words * 4, ctx->stream));  // fm, flags, counters start at 0
  PC_CUDA(cudaMemcpyAsync(d_seeds, sd.data(), (size_t)ns * 4, cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t Kmc = pc_mix64(mc_seed ^ 0x4D435349434D4353ull);
  std::vector<unsigned long long> hk(MC_W * 32);
  const unsigned lgrid = ctx->sm_count * 8;
  for (uint32_t b0 = 0; b0 < nsims; b0 += MC_W * 32) {
    const uint32_t nb = std::min<uint32_t>(MC_W * 32, nsims - b0);
    for (uint32_t i = 0; i < MC_W * 32; i++) hk[i] = pc_mix64(Kmc ^ (uint64_t)(b0 + i));
    PC_CUDA(cudaMemcpyAsync(Ki, hk.data(), hk.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    PC_CUDA(cudaMemsetAsync(M.vis, 0, vw * 4, ctx->stream));
    const uint32_t full_words = (nb + 31) / 32;
    const uint32_t last = nb % 32 ? (1u << (nb % 32)) - 1 : 0xFFFFFFFFu;
    PC_CUDA(cudaMemsetAsync(M.cnt, 0, 8, ctx->stream));
    if (ns) {
      k_mc_seeds<<<std::max<unsigned>(1, std::min<unsigned>((ns * MC_W + 255) / 256, 1024)), 256, 0,
                   ctx->stream>>>(M, d_seeds, ns, full_words, last);
      PC_CHECK_LAUNCH();
    }
    uint32_t lcnt = ns;
    PC_CUDA(cudaMemcpyAsync(M.cnt, &lcnt, 4, cudaMemcpyHostToDevice, ctx->stream));
    for (uint32_t lvl = 0; lcnt; lvl++) {
      const uint32_t cur = lvl & 1, nxt = cur ^ 1;
      PC_CUDA(cudaMemsetAsync(M.cnt + nxt, 0, 4, ctx->stream));
      k_mc_level<<<lgrid, 256, 0, ctx->stream>>>(M, cur);
      PC_CHECK_LAUNCH();
      PC_CUDA(cudaMemcpyAsync(&lcnt, M.cnt + nxt, 4, cudaMemcpyDeviceToHost, ctx->stream));
      PC_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    k_mc_count<<<pc_grid(ctx, vw, 256, 8), 256, 0, ctx->stream>>>(M.vis, vw, d_total);
    PC_CHECK_LAUNCH();
  }
  unsigned long long h = 0;
  PC_CUDA(cudaMemcpyAsync(&h, d_total, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  *total_out = h;
}
