// select.cu — Step 2 of Alg. 1: the device-resident greedy loop.
//
// One persistent cooperative kernel runs all k steps (H8-H12):
//   A  argmax over v of (gain desc, id asc); seeds hold gain -1 (R5, R6)
//   B  MarkSeed: per sketch slot j, the seed's component
//      c = comp(s, j); delta_j = size_work[c]; size_work[c] <- 0      (H9)
//   C  incremental gain update: every member u != s of each newly covered
//      component loses delta_j (H10); gain[s] <- -1
// separated by grid-wide barriers.  gain_num[i] = sum_j delta_j is checked
// against the argmax gain (the two must agree exactly).
#include <cooperative_groups.h>

#include "pacim_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int SEL_THREADS = 512;

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

struct SelParams {
  const uint32_t *L;
  uint32_t n, B;
  const uint64_t *coff;
  const uint32_t *perm;
  uint32_t *csw;          // working sizes (zeroed on cover)
  long long *gain;        // working gains
  Best *partial;          // gridDim entries
  uint64_t *list_off;     // B entries
  uint32_t *list_len;     // B entries
  uint32_t k;
  uint32_t *seeds;
  long long *gain_num;    // k, zeroed
  long long *arg_gain;    // k
  int *flag;              // mismatch flag
  unsigned long long *updates;
};

__global__ void __launch_bounds__(SEL_THREADS) k_select(SelParams P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Best sh[33];
  __shared__ uint32_t pre[1025];
  __shared__ Best chosen;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  unsigned long long upd = 0;
  for (uint32_t step = 0; step < P.k; step++) {
    // ---- A: argmax (gain desc, id asc)
    Best b{LLONG_MIN, 0xFFFFFFFFu};
    for (size_t v = tid; v < P.n; v += nth) {
      long long g = P.gain[v];
      if (better(g, (uint32_t)v, b.g, b.v)) {
        b.g = g;
        b.v = (uint32_t)v;
      }
    }
    b = block_best(b, sh);
    if (threadIdx.x == 0) P.partial[blockIdx.x] = b;
    grid.sync();
    Best c{LLONG_MIN, 0xFFFFFFFFu};
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      Best x = P.partial[i];
      if (better(x.g, x.v, c.g, c.v)) c = x;
    }
    c = block_best(c, sh);
    if (threadIdx.x == 0) chosen = c;
    __syncthreads();
    const uint32_t s = chosen.v;
    // ---- B: MarkSeed on every slot
    for (size_t j = tid; j < P.B; j += nth) {
      uint32_t sl = P.L[(size_t)s * P.B + j];
      uint32_t delta, len = 0;
      uint64_t off = 0;
      if (sl == s) {
        delta = 1;  // singleton {s}: covered now, no other member
      } else {
        uint32_t ci = (sl & PACIM_HIGH) ? (sl & PACIM_LOW)
                                        : (P.L[(size_t)sl * P.B + j] & PACIM_LOW);
        delta = P.csw[ci];
        if (delta) {
          P.csw[ci] = 0;
          len = delta;
          off = P.coff[ci];
        }
      }
      P.list_len[j] = len;
      P.list_off[j] = off;
      atomicAdd((unsigned long long *)&P.gain_num[step], (unsigned long long)delta);
    }
    grid.sync();
    // ---- C: gain updates over the concatenated member ranges
    // per block: exclusive prefix of list_len in chunks of 1024 slots
    for (uint32_t j0 = 0; j0 < P.B; j0 += 1024) {
      const uint32_t cnt = min(1024u, P.B - j0);
      if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (uint32_t q = 0; q < cnt; q++) {
          pre[q] = run;
          run += P.list_len[j0 + q];
        }
        pre[cnt] = run;
      }
      __syncthreads();
      const uint32_t W = pre[cnt];
      for (size_t idx = tid; idx < W; idx += nth) {
        // slot q with pre[q] <= idx < pre[q+1]
        uint32_t lo = 0, hi = cnt;
        while (hi - lo > 1) {
          uint32_t mid = (lo + hi) >> 1;
          if (pre[mid] <= idx) lo = mid; else hi = mid;
        }
        const uint32_t q = lo;
        const uint32_t u = P.perm[P.list_off[j0 + q] + (idx - pre[q])];
        if (u != s) {
          atomicAdd((unsigned long long *)&P.gain[u],
                    (unsigned long long)(-(long long)P.list_len[j0 + q]));
          upd++;
        }
      }
      __syncthreads();
    }
    if (tid == 0) {
      P.seeds[step] = s;
      P.arg_gain[step] = chosen.g;
      if (P.gain_num[step] != chosen.g) *P.flag = 1;
      P.gain[s] = -1;
    }
    grid.sync();
  }
  for (int d = 16; d; d >>= 1) upd += __shfl_xor_sync(0xffffffffu, upd, d);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(P.updates, upd);
}

// standalone argmax for the multi-rank loop
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

// MarkSeed on this rank's slots, member deltas accumulated into delta[]
__global__ void k_cover_local(const uint32_t *L, uint32_t B, uint32_t s, uint32_t *csw,
                              const uint64_t *coff, const uint32_t *perm, long long *delta,
                              unsigned long long *sum) {
  // one block per slot j
  for (uint32_t j = blockIdx.x; j < B; j += gridDim.x) {
    uint32_t sl = L[(size_t)s * B + j];
    uint32_t d;
    uint64_t off = 0;
    bool members = false;
    if (sl == s) {
      d = 1;
    } else {
      uint32_t ci = (sl & PACIM_HIGH) ? (sl & PACIM_LOW) : (L[(size_t)sl * B + j] & PACIM_LOW);
      d = csw[ci];
      off = coff[ci];
      members = d > 0;
    }
    __syncthreads();
    if (members && threadIdx.x == 0) {
      uint32_t ci = (sl & PACIM_HIGH) ? (sl & PACIM_LOW) : (L[(size_t)sl * B + j] & PACIM_LOW);
      csw[ci] = 0;
    }
    if (threadIdx.x == 0) atomicAdd(sum, (unsigned long long)d);
    if (members)
      for (uint32_t i = threadIdx.x; i < d; i += blockDim.x)
        atomicAdd((unsigned long long *)&delta[perm[off + i]], (unsigned long long)(-(long long)d));
    __syncthreads();
  }
}

}  // namespace

void pc_select_reset(pacim_ctx *ctx) {
  PC_CUDA(cudaMemcpyAsync(ctx->csize_work.p, ctx->csize.p, std::max<size_t>(ctx->ncomp, 1) * 4,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

void pc_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
               int64_t *sigma_num) {
  const uint32_t n = ctx->n, B = ctx->R_local;
  int occ = 0;
  PC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_select, SEL_THREADS, 0));
  PC_REQUIRE(occ >= 1, PACIM_ECUDA, "k_select cannot be resident");
  unsigned grid = (unsigned)ctx->sm_count * (unsigned)std::min(occ, 2);
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  pc_ensure(ctx, ctx->sel_partial, (size_t)grid * sizeof(Best));
  pc_ensure(ctx, ctx->sel_list, (size_t)B * 12 + 16);
  pc_ensure(ctx, ctx->sel_seeds, (size_t)k * 4);
  pc_ensure(ctx, ctx->sel_gain, (size_t)k * 16 + 64);
  pc_ensure(ctx, ctx->sel_flag, 64);
  cudaEvent_t e0, e1;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(ctx->gain.p, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  PC_CUDA(cudaMemcpyAsync(ctx->csize_work.p, ctx->csize.p, std::max<size_t>(ctx->ncomp, 1) * 4,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  PC_CUDA(cudaMemsetAsync(ctx->sel_gain.p, 0, (size_t)k * 16 + 64, ctx->stream));
  PC_CUDA(cudaMemsetAsync(ctx->sel_flag.p, 0, 64, ctx->stream));
  SelParams P;
  P.L = ctx->L.as<uint32_t>();
  P.n = n;
  P.B = B;
  P.coff = ctx->coff.as<uint64_t>();
  P.perm = ctx->perm.as<uint32_t>();
  P.csw = ctx->csize_work.as<uint32_t>();
  P.gain = ctx->gain.as<long long>();
  P.partial = ctx->sel_partial.as<Best>();
  P.list_off = ctx->sel_list.as<uint64_t>();
  P.list_len = reinterpret_cast<uint32_t *>(P.list_off + B);
  P.k = k;
  P.seeds = ctx->sel_seeds.as<uint32_t>();
  P.gain_num = ctx->sel_gain.as<long long>();
  P.arg_gain = P.gain_num + k;
  P.flag = ctx->sel_flag.as<int>();
  P.updates = reinterpret_cast<unsigned long long *>(P.gain_num + 2 * k);
  void *args[] = {&P};
  PC_CUDA(cudaLaunchCooperativeKernel((void *)k_select, grid, SEL_THREADS, args, 0, ctx->stream));
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  std::vector<long long> hg(2 * k + 1);
  int flag = 0;
  PC_CUDA(cudaMemcpyAsync(seeds, P.seeds, (size_t)k * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(hg.data(), P.gain_num, (2 * (size_t)k + 1) * 8, cudaMemcpyDeviceToHost,
                          ctx->stream));
  PC_CUDA(cudaMemcpyAsync(&flag, P.flag, 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms = ms;
  ctx->stats.kernel_launches_select = 1;
  ctx->stats.select_member_updates = (uint64_t)hg[2 * k];
  long long run = 0;
  for (uint32_t i = 0; i < k; i++) {
    gain_num[i] = hg[i];
    run += hg[i];
    sigma_num[i] = run;
  }
  PC_REQUIRE(!flag, PACIM_ECHECK, "select: sum_r delta_r differs from the argmax gain");
}

void pc_cover_local(pacim_ctx *ctx, uint32_t s, int64_t *d_delta, int64_t *local_gain) {
  pc_ensure(ctx, ctx->sel_flag, 64);
  unsigned long long *sum = ctx->sel_flag.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(sum, 0, 8, ctx->stream));
  unsigned g = std::min<unsigned>(ctx->R_local, (unsigned)ctx->sm_count * 8);
  k_cover_local<<<g, 256, 0, ctx->stream>>>(ctx->L.as<uint32_t>(), ctx->R_local, s,
                                           ctx->csize_work.as<uint32_t>(),
                                           ctx->coff.as<uint64_t>(), ctx->perm.as<uint32_t>(),
                                           reinterpret_cast<long long *>(d_delta), sum);
  PC_CHECK_LAUNCH();
  unsigned long long h = 0;
  PC_CUDA(cudaMemcpyAsync(&h, sum, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  *local_gain = (int64_t)h;
}

void pc_argmax(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n, uint32_t *s, int64_t *g) {
  unsigned grid = pc_grid(ctx, n, SEL_THREADS, 2);
  TmpBuf part(ctx);
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
