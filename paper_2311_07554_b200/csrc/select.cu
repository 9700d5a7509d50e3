// select.cu — Step 2 of Alg. 1: the device-resident greedy loop.
//
// One persistent cooperative kernel runs all k steps (H8-H12):
//   A  argmax over v of (gain desc, id asc); seeds hold gain -1 (R5, R6)
//   B  MarkSeed: per sketch slot j, the seed's component
//      c = comp(s, j); delta_j = size_work[c]; size_work[c] <- 0      (H9)
//   C  incremental gain update (H10): every member u != s of each newly
//      covered component loses delta_j — indexed components through the
//      member index, big components (coff = PACIM_BIG) through one dense
//      pass over the store comparing slots with the covered root;
//      gain[s] <- -1
// separated by grid-wide barriers.  gain_num[i] = sum_j delta_j is checked
// against the argmax gain (the two must agree exactly).
// The multi-rank primitives (pacim_cover_local / pacim_argmax_device) reuse
// the same device phases as ordinary launches.
#include <cooperative_groups.h>

#include <cstdlib>

#include "pacim_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int SEL_THREADS = 512;
constexpr uint32_t NONE = 0xFFFFFFFFu;

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

// Per-step cover state (device, B entries each).
struct CoverState {
  const uint32_t *L;      // store rows (non-isolated vertices) x B slots
  uint32_t n, B;          // n = store rows
  const uint32_t *cid;    // vertex -> row (0xFFFFFFFF: isolated)
  const uint32_t *rmap;   // row -> vertex
  const uint64_t *coff;
  const uint32_t *perm;
  uint32_t *csw;       // working sizes, zeroed on cover
  uint64_t *list_off;  // indexed member range of slot j's covered CC
  uint32_t *list_len;  // its length (0: none)
  uint32_t *cov_root;  // root of slot j's covered big CC, or NONE
  uint32_t *cov_delta; // its size
  int *dense;          // set when some big CC was covered this step
};

// Phase B for slot j: returns delta_j.
__device__ __forceinline__ uint32_t cover_slot(const CoverState &C, uint32_t s, uint32_t j) {
  const uint32_t cs = C.cid[s];  // the seed's row
  const uint32_t sl = cs == NONE ? NONE : __ldcg(C.L + (size_t)cs * C.B + j);
  uint32_t delta = 1, len = 0, croot = NONE;
  uint64_t off = 0;
  if (cs != NONE && sl != cs) {
    const uint32_t root = (sl & PACIM_HIGH) ? cs : sl;
    const uint32_t ci = (sl & PACIM_HIGH) ? (sl & PACIM_LOW)
                                          : (__ldcg(C.L + (size_t)root * C.B + j) & PACIM_LOW);
    delta = __ldcg(C.csw + ci);
    if (delta) {
      C.csw[ci] = 0;
      off = C.coff[ci];
      if (off == PACIM_BIG) {
        croot = root;
        *C.dense = 1;
      } else {
        len = delta;
      }
    }
  }  // else: singleton {s}, covered now, no other member
  C.list_len[j] = len;
  C.list_off[j] = off;
  C.cov_root[j] = croot;
  C.cov_delta[j] = delta;
  return delta;
}

// Phase C1: target[u] -= delta_j for the members u != s of the indexed CCs,
// threads [tid, +nth) over the concatenated ranges; pre[] is per-block smem.
// The list arrays may live in global memory (written by an earlier launch or
// before a grid barrier) or in shared memory (plain loads either way).

__device__ unsigned long long apply_members(const CoverState &C, uint32_t s, long long *target,
                                            uint32_t *pre, size_t tid, size_t nth) {
  unsigned long long upd = 0;
  for (uint32_t j0 = 0; j0 < C.B; j0 += 1024) {
    const uint32_t cnt = min(1024u, C.B - j0);
    __syncthreads();
    if (threadIdx.x < 32) {  // warp-parallel exclusive prefix over cnt slots
      uint32_t carry = 0;
      for (uint32_t q0 = 0; q0 < cnt; q0 += 32) {
        uint32_t q = q0 + threadIdx.x;
        uint32_t x = q < cnt ? C.list_len[j0 + q] : 0, inc = x;
        for (int d = 1; d < 32; d <<= 1) {
          uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
          if ((int)threadIdx.x >= d) inc += y;
        }
        if (q < cnt) pre[q] = carry + inc - x;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (threadIdx.x == 0) pre[cnt] = carry;
    }
    __syncthreads();
    const uint32_t W = pre[cnt];
    for (size_t idx = tid; idx < W; idx += nth) {
      uint32_t lo = 0, hi = cnt;  // slot q with pre[q] <= idx < pre[q+1]
      while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (pre[mid] <= idx) lo = mid; else hi = mid;
      }
      const uint32_t u = C.perm[C.list_off[j0 + lo] + (idx - pre[lo])];
      if (u != s) {
        atomicAdd((unsigned long long *)&target[u],
                  (unsigned long long)(-(long long)C.list_len[j0 + lo]));
        upd++;
      }
    }
  }
  return upd;
}

// Phase C2: dense pass over the store for the covered big CCs: v is a member
// of slot j's covered CC iff its slot holds that root, or v is the root.
// Each lane keeps the covered roots of its 8 slots of a 256-slot chunk in
// registers and streams the rows.
__device__ unsigned long long apply_dense(const CoverState &C, uint32_t s, long long *target,
                                          size_t warp0, size_t nwarps) {
  const int lane = threadIdx.x & 31;
  unsigned long long upd = 0;
  for (uint32_t j0 = 0; j0 < C.B; j0 += 256) {
    uint32_t cr[8], cd[8];
    bool any = false;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const uint32_t j = j0 + lane + 32 * i;
      cr[i] = j < C.B ? C.cov_root[j] : NONE;
      cd[i] = j < C.B ? C.cov_delta[j] : 0;
      any |= cr[i] != NONE;
    }
    if (!__any_sync(0xffffffffu, any)) continue;
    for (size_t v = warp0; v < C.n; v += nwarps) {
      uint32_t x[8];
#pragma unroll
      for (int i = 0; i < 8; i++)
        x[i] = cr[i] != NONE ? __ldcs(C.L + v * C.B + j0 + lane + 32 * i) : NONE;
      long long d = 0;
#pragma unroll
      for (int i = 0; i < 8; i++)
        if (cr[i] != NONE && (x[i] == cr[i] || (uint32_t)v == cr[i])) d += cd[i];
      for (int q = 16; q; q >>= 1) d += __shfl_xor_sync(0xffffffffu, d, q);
      if (lane == 0 && d) {
        const uint32_t vid = C.rmap[v];
        if (vid != s) {
          atomicAdd((unsigned long long *)&target[vid], (unsigned long long)(-d));
          upd++;
        }
      }
    }
  }
  return upd;
}

struct SelParams {
  CoverState C;
  uint32_t nv;            // vertices (gain vector length)
  long long *gain;        // working gains
  Best *partial;          // gridDim entries
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
  const CoverState &C = P.C;
  unsigned long long upd = 0;
  for (uint32_t step = 0; step < P.k; step++) {
    // ---- A: argmax (gain desc, id asc)
    Best b{LLONG_MIN, 0xFFFFFFFFu};
    for (size_t v = tid; v < P.nv; v += nth) {
      long long g = __ldcg(P.gain + v);
      if (better(g, (uint32_t)v, b.g, b.v)) {
        b.g = g;
        b.v = (uint32_t)v;
      }
    }
    b = block_best(b, sh);
    if (threadIdx.x == 0) P.partial[blockIdx.x] = b;
    if (tid == 0) *C.dense = 0;
    grid.sync();
    Best c{LLONG_MIN, 0xFFFFFFFFu};
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      Best x;
      x.g = __ldcg(&P.partial[i].g);
      x.v = __ldcg(&P.partial[i].v);
      if (better(x.g, x.v, c.g, c.v)) c = x;
    }
    c = block_best(c, sh);
    if (threadIdx.x == 0) chosen = c;
    __syncthreads();
    const uint32_t s = chosen.v;
    // ---- B: MarkSeed on every slot
    for (size_t j = tid; j < C.B; j += nth) {
      uint32_t delta = cover_slot(C, s, (uint32_t)j);
      atomicAdd((unsigned long long *)&P.gain_num[step], (unsigned long long)delta);
    }
    grid.sync();
    // ---- C: gain updates
    upd += apply_members(C, s, P.gain, pre, tid, nth);
    if (__ldcg(C.dense)) upd += apply_dense(C, s, P.gain, tid >> 5, nth >> 5);
    if (tid == 0) {
      P.seeds[step] = s;
      P.arg_gain[step] = chosen.g;
      if (__ldcg(P.gain_num + step) != chosen.g) *P.flag = 1;
      P.gain[s] = -1;
    }
    grid.sync();
  }
  for (int d = 16; d; d >>= 1) upd += __shfl_xor_sync(0xffffffffu, upd, d);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(P.updates, upd);
}

// Two barriers per step (B <= SEL_FUSED_B): every block redundantly computes
// the seed's per-slot cover list (B cheap lookups) into shared memory, so the
// MarkSeed phase needs no barrier of its own.  The zeroing of the covered
// sizes is deferred to block 0 in the next step's argmax phase, i.e. after
// every block has read them (the cover of step i reads sizes as of step i-1).
constexpr uint32_t SEL_FUSED_B = 1024;

struct Sel2Params {
  CoverState C;           // list arrays unused (kept in shared memory)
  uint32_t nv;
  long long *gain;
  Best *partial;
  uint32_t *pending_ci;   // B: component covered in slot j by the previous step, or NONE
  uint32_t k;
  uint32_t *seeds;
  long long *gain_num;
  long long *arg_gain;
  int *flag;
  unsigned long long *updates;
};

__global__ void __launch_bounds__(SEL_THREADS) k_select2(Sel2Params P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint64_t s2[];
  const uint32_t B = P.C.B;
  uint64_t *l_off = s2;                                          // B
  uint32_t *l_len = reinterpret_cast<uint32_t *>(l_off + B);     // B
  uint32_t *c_root = l_len + B;                                  // B
  uint32_t *c_delta = c_root + B;                                // B
  uint32_t *pre = c_delta + B;                                   // 1025
  __shared__ Best sh[33];
  __shared__ Best chosen;
  __shared__ int dense;
  __shared__ unsigned long long dsum;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  CoverState C = P.C;
  C.list_off = l_off;
  C.list_len = l_len;
  C.cov_root = c_root;
  C.cov_delta = c_delta;
  unsigned long long upd = 0;
  for (uint32_t step = 0; step < P.k; step++) {
    // ---- A: argmax partials; block 0 applies the previous step's zeroing
    Best b{LLONG_MIN, 0xFFFFFFFFu};
    for (size_t v = tid; v < P.nv; v += nth) {
      long long g = __ldcg(P.gain + v);
      if (better(g, (uint32_t)v, b.g, b.v)) {
        b.g = g;
        b.v = (uint32_t)v;
      }
    }
    b = block_best(b, sh);
    if (threadIdx.x == 0) P.partial[blockIdx.x] = b;
    if (blockIdx.x == 0)
      for (uint32_t j = threadIdx.x; j < B; j += blockDim.x) {
        const uint32_t ci = P.pending_ci[j];
        if (ci != NONE) C.csw[ci] = 0;
      }
    grid.sync();
    // ---- every block: s, and the cover list of all slots
    Best c{LLONG_MIN, 0xFFFFFFFFu};
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      Best x;
      x.g = __ldcg(&P.partial[i].g);
      x.v = __ldcg(&P.partial[i].v);
      if (better(x.g, x.v, c.g, c.v)) c = x;
    }
    c = block_best(c, sh);
    if (threadIdx.x == 0) {
      chosen = c;
      dense = 0;
      dsum = 0;
    }
    __syncthreads();
    const uint32_t s = chosen.v;
    const uint32_t cs = C.cid[s];
    unsigned long long mysum = 0;
    for (uint32_t j = threadIdx.x; j < B; j += blockDim.x) {
      uint32_t delta = 1, len = 0, croot = NONE, ci = NONE;
      uint64_t off = 0;
      const uint32_t sl = cs == NONE ? NONE : __ldcg(C.L + (size_t)cs * B + j);
      if (cs != NONE && sl != cs) {
        const uint32_t root = (sl & PACIM_HIGH) ? cs : sl;
        ci = (sl & PACIM_HIGH) ? (sl & PACIM_LOW) : (__ldcg(C.L + (size_t)root * B + j) & PACIM_LOW);
        delta = __ldcg(C.csw + ci);
        if (delta) {
          off = C.coff[ci];
          if (off == PACIM_BIG) {
            croot = root;
            dense = 1;
          } else {
            len = delta;
          }
        } else {
          ci = NONE;  // already covered: nothing to zero
        }
      }
      l_off[j] = off;
      l_len[j] = len;
      c_root[j] = croot;
      c_delta[j] = delta;
      mysum += delta;
      if (blockIdx.x == 0) P.pending_ci[j] = ci;
    }
    for (int d = 16; d; d >>= 1) mysum += __shfl_xor_sync(0xffffffffu, mysum, d);
    if ((threadIdx.x & 31) == 0 && mysum) atomicAdd(&dsum, mysum);
    // ---- C: gain updates (apply_members starts with a block barrier)
    upd += apply_members(C, s, P.gain, pre, tid, nth);
    if (dense) upd += apply_dense(C, s, P.gain, tid >> 5, nth >> 5);
    if (tid == 0) {
      P.seeds[step] = s;
      P.arg_gain[step] = chosen.g;
      P.gain_num[step] = (long long)dsum;
      if ((long long)dsum != chosen.g) *P.flag = 1;
      P.gain[s] = -1;
    }
    grid.sync();
  }
  for (int d = 16; d; d >>= 1) upd += __shfl_xor_sync(0xffffffffu, upd, d);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(P.updates, upd);
}

// ------------------------------------------------ multi-rank step kernels
__global__ void k_cover_slots(CoverState C, uint32_t s, unsigned long long *sum) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < C.B; j += gridDim.x * blockDim.x)
    atomicAdd(sum, (unsigned long long)cover_slot(C, s, j));
}

__global__ void __launch_bounds__(SEL_THREADS) k_apply_members(CoverState C, uint32_t s,
                                                               long long *target) {
  __shared__ uint32_t pre[1025];
  apply_members(C, s, target, pre, (size_t)blockIdx.x * blockDim.x + threadIdx.x,
                (size_t)gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(256) k_apply_dense(CoverState C, uint32_t s, long long *target) {
  if (!__ldcg(C.dense)) return;
  apply_dense(C, s, target, ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
              ((size_t)gridDim.x * blockDim.x) >> 5);
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

static CoverState make_cover_state(pacim_ctx *ctx) {
  const uint32_t B = ctx->R_local;
  pc_ensure(ctx, ctx->sel_list, (size_t)B * 20 + 64);
  CoverState C;
  C.L = ctx->L.as<uint32_t>();
  C.n = ctx->nr;
  C.cid = ctx->cid.as<uint32_t>();
  C.rmap = ctx->rmap.as<uint32_t>();
  C.B = B;
  C.coff = ctx->coff.as<uint64_t>();
  C.perm = ctx->perm.as<uint32_t>();
  C.csw = ctx->csize_work.as<uint32_t>();
  C.list_off = ctx->sel_list.as<uint64_t>();
  C.list_len = reinterpret_cast<uint32_t *>(C.list_off + B);
  C.cov_root = C.list_len + B;
  C.cov_delta = C.cov_root + B;
  C.dense = reinterpret_cast<int *>(C.cov_delta + B);
  return C;
}

void pc_select_reset(pacim_ctx *ctx) {
  PC_CUDA(cudaMemcpyAsync(ctx->csize_work.p, ctx->csize.p, std::max<size_t>(ctx->ncomp, 1) * 4,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

void pc_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
               int64_t *sigma_num) {
  const uint32_t n = ctx->n;
  int occ = 0;
  PC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_select, SEL_THREADS, 0));
  PC_REQUIRE(occ >= 1, PACIM_ECUDA, "k_select cannot be resident");
  unsigned grid = (unsigned)ctx->sm_count * (unsigned)std::min(occ, 2);
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  pc_ensure(ctx, ctx->sel_partial, (size_t)grid * sizeof(Best));
  pc_ensure(ctx, ctx->sel_seeds, (size_t)k * 4);
  pc_ensure(ctx, ctx->sel_gain, (size_t)k * 16 + 64);
  pc_ensure(ctx, ctx->sel_flag, 64);
  SelParams P;
  P.C = make_cover_state(ctx);
  P.nv = n;
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
  P.gain = ctx->gain.as<long long>();
  P.partial = ctx->sel_partial.as<Best>();
  P.k = k;
  P.seeds = ctx->sel_seeds.as<uint32_t>();
  P.gain_num = ctx->sel_gain.as<long long>();
  P.arg_gain = P.gain_num + k;
  P.flag = ctx->sel_flag.as<int>();
  P.updates = reinterpret_cast<unsigned long long *>(P.gain_num + 2 * k);
  const uint32_t B = ctx->R_local;
  if (B <= SEL_FUSED_B && !getenv("PACIM_SELECT_3SYNC")) {
    // two grid barriers per step (the cover list is computed in every block)
    const size_t smem = (size_t)B * 20 + 1025 * 4;
    PC_CUDA(cudaFuncSetAttribute(k_select2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int occ2 = 0;
    PC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_select2, SEL_THREADS, smem));
    PC_REQUIRE(occ2 >= 1, PACIM_ECUDA, "k_select2 cannot be resident");
    const unsigned grid2 = (unsigned)ctx->sm_count * (unsigned)std::min(occ2, 2);
    pc_ensure(ctx, ctx->sel_partial, (size_t)grid2 * sizeof(Best) + (size_t)B * 4);
    Sel2Params Q;
    Q.C = P.C;
    Q.nv = n;
    Q.gain = P.gain;
    Q.partial = ctx->sel_partial.as<Best>();
    Q.pending_ci = reinterpret_cast<uint32_t *>(Q.partial + grid2);
    PC_CUDA(cudaMemsetAsync(Q.pending_ci, 0xFF, (size_t)B * 4, ctx->stream));
    Q.k = k;
    Q.seeds = P.seeds;
    Q.gain_num = P.gain_num;
    Q.arg_gain = P.arg_gain;
    Q.flag = P.flag;
    Q.updates = P.updates;
    void *args2[] = {&Q};
    PC_CUDA(cudaLaunchCooperativeKernel((void *)k_select2, grid2, SEL_THREADS, args2, smem,
                                        ctx->stream));
  } else {
    void *args[] = {&P};
    PC_CUDA(cudaLaunchCooperativeKernel((void *)k_select, grid, SEL_THREADS, args, 0, ctx->stream));
  }

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
  CoverState C = make_cover_state(ctx);
  pc_ensure(ctx, ctx->sel_flag, 64);
  unsigned long long *sum = ctx->sel_flag.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(sum, 0, 8, ctx->stream));
  PC_CUDA(cudaMemsetAsync(C.dense, 0, 4, ctx->stream));
  const uint32_t B = ctx->R_local;
  k_cover_slots<<<(B + 255) / 256, 256, 0, ctx->stream>>>(C, s, sum);
  PC_CHECK_LAUNCH();
  long long *t = reinterpret_cast<long long *>(d_delta);
  k_apply_members<<<pc_grid(ctx, (size_t)1 << 22, SEL_THREADS, 2), SEL_THREADS, 0, ctx->stream>>>(
      C, s, t);
  PC_CHECK_LAUNCH();
  k_apply_dense<<<pc_grid(ctx, (size_t)ctx->n * 32, 256, 8), 256, 0, ctx->stream>>>(C, s, t);
  PC_CHECK_LAUNCH();
  unsigned long long h = 0;
  PC_CUDA(cudaMemcpyAsync(&h, sum, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  *local_gain = (int64_t)h;
}

void pc_argmax(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n, uint32_t *s, int64_t *g) {
  unsigned grid = pc_grid(ctx, n, SEL_THREADS, 2);
  DevBuf &part = ctx->sel_partial;  // persistent: no allocation per step
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
