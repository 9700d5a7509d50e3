// dist.cu — multi-GPU sketch sharding behind the C ABI.
//
// One process per GPU.  Rank g builds the sketches r = g (mod P) over a
// replicated CSR (pacim_build_sketches with shard_rank = g, shard_world = P);
// with a communicator (pacim_init_comm: NCCL, called from C++) the build ends
// with ONE all-reduce of gain0 (int64, H7) — and of the per-vertex hot sums
// of the hub's giant CCs — so every rank holds the global gain vector.
//
// pacim_select_seeds on a sharded build (sketches are independent,
// the greedy step sums over them):
//   fast path (compact store), per step, all enqueued on the ctx stream with
//   no host synchronisation (optionally one CUDA graph for all k steps):
//     k_dist_cover  every rank: NextSeed over the replicated gains (cached
//                   chunk maxima, identical on all ranks), MarkSeed on its own
//                   sketches, the members' deltas (v, |C|) into a fixed-size
//                   list; big CCs (no member list) are flagged
//     k_dist_head   the step header: list length, local sum of delta_r,
//                   overflow, and whether the step's big CCs are exactly this
//                   rank's hub giants
//     ncclAllGather header + list (one collective per step)
//     k_dist_apply  every rank applies every rank's list (and, in the step
//                   that covers the hub's giants on every rank, the all-reduced
//                   hot sums) to its replica; checks sum delta = argmax gain
//     k_dist_chunks the chunk maxima that lost their argmax
//   A list overflow or a big CC that is not a hub giant sets a replay flag
//   (seen by every rank: it is in the gathered headers); the host then
//   re-runs the selection on the robust path.
//   robust path (any store, and replays): per step the argmax read back,
//   MarkSeed + member deltas into a dense int64 delta vector, one
//   ncclAllReduce of it, applied — correct whatever the CC sizes.
// Integer sums are associative: any partition gives the one-GPU sequence.
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "pacim_internal.cuh"

namespace cg = cooperative_groups;

#define PC_NCCL(call)                                                               \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess)                                                          \
      throw PacimError{PACIM_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

namespace {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t COV = 0x40000000u;
constexpr uint32_t SIZE = 0x3FFFFFFFu;
constexpr unsigned FULL = 0xffffffffu;
constexpr int DT = 512;                 // threads per block of the step kernels
constexpr uint32_t MAX_CHUNKS = 4096;
// header words (u64) of a rank's step message
enum { H_CNT = 0, H_DSUM, H_FLAGS, H_PAD, H_WORDS };
enum { F_OVER = 1, F_DENSE = 2, F_EXACT = 4 };
// device state words (u64)
enum { D_S = 0, D_SG, D_REPLAY, D_CHECK, D_DCNT, D_WORDS = 8 };

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

struct DSel {
  // compact store of this rank (store_cs.cu): E = {P, next} words, vid
  const uint2 *rec;
  uint32_t MW;
  uint32_t *E;
  const uint32_t *vid, *cid;
  uint32_t B, nv, list_t;
  const uint32_t *hot_root;
  // replicated gains + argmax cache
  long long *gain;
  Best *cmax;
  uint32_t *cdirty, *dlist;
  uint32_t csh, nchunks;
  const int64_t *ghot;     // all-reduced hot sums (null: none)
  // covered CCs (restored before the next selection)
  unsigned long long *cov_list, *cov_cnt, cov_cap;
  uint32_t *cov_root;      // [B] big CC covered in slot j this step
  // messages
  unsigned long long *send;  // H_WORDS + cap
  const unsigned long long *recv;  // world x (H_WORDS + cap)
  unsigned long long cap;
  int world;
  unsigned long long *st;  // D_WORDS
  uint32_t *seeds;
  long long *gain_num;
};

__device__ __forceinline__ void mark_dirty(const DSel &S, uint32_t c) {
  if (atomicExch(S.cdirty + c, 1u) == 0u)
    S.dlist[atomicAdd(reinterpret_cast<unsigned long long *>(S.st + D_DCNT), 1ull)] = c;
}

// Step part 1 (cooperative): every block takes NextSeed from the chunk
// maxima (identical on every rank); MarkSeed on this rank's slots, a warp per
// slot: lane 0 walks the newly covered CC's member list into a shared buffer,
// the warp appends (v, |C|) to the send list; then, after a grid barrier,
// block 0 writes the step header: list overflow; list-less CCs covered;
// EXACT = those are exactly this rank's hub CCs (both sets may be empty) —
// when some rank covers list-less CCs, the all-reduced hot sums are the
// update iff every rank is EXACT.
constexpr uint32_t WBUF = 128;
__global__ void __launch_bounds__(DT, 1) k_dist_cover(DSel S, uint32_t step) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Best sh[33];
  __shared__ uint32_t wbuf[DT / 32][WBUF];
  __shared__ int dense, exact;
  Best c{LLONG_MIN, NONE};
  for (uint32_t i = threadIdx.x; i < S.nchunks; i += blockDim.x) {
    Best x;
    x.g = __ldcg(&S.cmax[i].g);
    x.v = __ldcg(&S.cmax[i].v);
    if (better(x.g, x.v, c.g, c.v)) c = x;
  }
  c = block_best(c, sh);
  const uint32_t s = c.v;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) {
    S.st[D_S] = s;
    S.st[D_SG] = (unsigned long long)c.g;
    S.st[D_DCNT] = 0;
    S.seeds[step] = s;
  }
  const int lane = threadIdx.x & 31;
  const size_t gwarp = tid >> 5, nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  uint32_t *buf = wbuf[threadIdx.x >> 5];
  const uint32_t srow = S.cid ? S.cid[s] : s;
  unsigned long long dsum = 0;
  for (size_t j = gwarp; j < S.B; j += nwarps) {
    uint32_t d = 1, mr = NONE;
    if (lane == 0) {
      S.cov_root[j] = NONE;
      if (srow != NONE && ((S.rec[(size_t)srow * S.MW + (j >> 5)].y >> (j & 31)) & 1u)) {
        const uint32_t e = pc_cs_pos(S.rec, S.MW, srow, (uint32_t)j);
        const uint32_t x0 = __ldcg(S.E + 2 * (size_t)e);
        const uint32_t root = (x0 & PACIM_HIGH) ? e : x0;
        const uint32_t x = atomicOr(S.E + 2 * (size_t)root, COV);
        if (x & COV) {
          d = 0;
        } else {
          d = x & SIZE;
          const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
          if (at < S.cov_cap) S.cov_list[at] = root;
          if (d > S.list_t || root == S.hot_root[j])
            S.cov_root[j] = root;  // no member list
          else
            mr = root;
        }
      }
    }
    d = __shfl_sync(FULL, d, 0);
    mr = __shfl_sync(FULL, mr, 0);
    dsum += d;
    if (mr == NONE) continue;
    uint32_t e = mr, left = d;
    while (left) {  // the members, a buffer of entries at a time
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
      for (uint32_t t0 = 0; t0 < cnt; t0 += 32) {
        const uint32_t t = t0 + lane;
        uint32_t v = NONE;
        if (t < cnt) v = __ldg(S.vid + buf[t]);
        const bool put = t < cnt && v != s;
        const uint32_t m = __ballot_sync(FULL, put);
        unsigned long long at = 0;
        if (lane == 0 && m) at = atomicAdd(S.send + H_CNT, (unsigned long long)__popc(m));
        at = __shfl_sync(FULL, at, 0) + __popc(m & ((1u << lane) - 1));
        if (put && at < S.cap) S.send[H_WORDS + at] = ((unsigned long long)v << 32) | d;
      }
      __syncwarp();
    }
  }
  if (lane == 0 && dsum) atomicAdd(S.send + H_DSUM, dsum);
  grid.sync();
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      dense = 0;
      exact = 1;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < S.B; j += blockDim.x) {
      const uint32_t cr = S.cov_root[j];
      if (cr != NONE) dense = 1;
      if (cr != S.hot_root[j]) exact = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long f = 0;
      if (S.send[H_CNT] > S.cap) f |= F_OVER;
      if (dense) f |= F_DENSE;
      if (exact) f |= F_EXACT;
      S.send[H_FLAGS] = f;
    }
  }
}

// Step part 2 (cooperative): every rank applies every rank's list to its
// replica; after a grid barrier the chunk maxima that lost their argmax are
// rescanned (a block per chunk) and the send header cleared
__device__ void refresh_dirty(const DSel &S, bool all, Best *sh) {
  const uint32_t nd = all ? S.nchunks : (uint32_t)__ldcg(S.st + D_DCNT);
  for (uint32_t t = blockIdx.x; t < nd; t += gridDim.x) {
    const uint32_t c = all ? t : __ldcg(S.dlist + t);
    const size_t v0 = (size_t)c << S.csh, v1 = min((size_t)S.nv, v0 + ((size_t)1 << S.csh));
    Best b{LLONG_MIN, NONE};
    for (size_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
      const long long g = __ldcg(S.gain + v);
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

__global__ void __launch_bounds__(DT, 1) k_dist_apply(DSel S, uint32_t step) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Best sh[33];
  const uint32_t s = (uint32_t)S.st[D_S];
  const long long sg = (long long)S.st[D_SG];
  // consensus from the gathered headers (identical on every rank)
  bool replay = false, any_dense = false, all_exact = true;
  long long gsum = 0;
  for (int p = 0; p < S.world; p++) {
    const unsigned long long *h = S.recv + (size_t)p * (H_WORDS + S.cap);
    const unsigned long long f = h[H_FLAGS];
    gsum += (long long)h[H_DSUM];
    if (f & F_OVER) replay = true;
    if (f & F_DENSE) any_dense = true;
    if (!(f & F_EXACT)) all_exact = false;
  }
  // list-less CCs: only the step that covers every rank's hub CCs at once has
  // its update precomputed (the all-reduced hot sums)
  if (any_dense && (!all_exact || !S.ghot)) replay = true;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  if (tid == 0) {
    if (replay) S.st[D_REPLAY] = 1;
    if (gsum != sg) S.st[D_CHECK] = 1;
    S.gain_num[step] = gsum;
    S.gain[s] = -1;  // s leaves the candidate set (R6)
    mark_dirty(S, s >> S.csh);
  }
  if (!replay) {
    if (any_dense && S.ghot) {
      for (size_t v = tid; v < S.nv; v += nth) {
        const long long h = S.ghot[v];
        if (h && v != s) {
          atomicAdd(reinterpret_cast<unsigned long long *>(S.gain + v), (unsigned long long)(-h));
          const uint32_t c = (uint32_t)(v >> S.csh);
          if (__ldcg(&S.cmax[c].v) == v) mark_dirty(S, c);
        }
      }
    }
    for (int p = 0; p < S.world; p++) {
      const unsigned long long *h = S.recv + (size_t)p * (H_WORDS + S.cap);
      const unsigned long long cnt = min(h[H_CNT], S.cap);
      for (size_t t = tid; t < cnt; t += nth) {
        const unsigned long long x = h[H_WORDS + t];
        const uint32_t v = (uint32_t)(x >> 32);
        const long long d = (long long)(uint32_t)x;
        atomicAdd(reinterpret_cast<unsigned long long *>(S.gain + v), (unsigned long long)(-d));
        const uint32_t c = v >> S.csh;
        if (__ldcg(&S.cmax[c].v) == v) mark_dirty(S, c);
      }
    }
  }
  grid.sync();
  refresh_dirty(S, false, sh);
  if (blockIdx.x == 0 && threadIdx.x < H_WORDS) S.send[threadIdx.x] = 0;
}

// the initial chunk maxima (all chunks) and a cleared send header
__global__ void __launch_bounds__(DT) k_dist_chunks(DSel S) {
  __shared__ Best sh[33];
  refresh_dirty(S, true, sh);
  if (blockIdx.x == 0 && threadIdx.x < H_WORDS) S.send[threadIdx.x] = 0;
}

__global__ void k_dist_uncover(uint32_t *E, const unsigned long long *list, unsigned long long cnt) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (size_t)gridDim.x * blockDim.x)
    atomicAnd(E + 2 * list[i], ~COV);
}

__global__ void k_dist_set(long long *gain, uint32_t s, long long x) { gain[s] = x; }

__global__ void k_dist_add(long long *gain, long long *delta, uint32_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const long long x = delta[i];
    if (x) {
      gain[i] += x;
      delta[i] = 0;
    }
  }
}

}  // namespace

// ------------------------------------------------------------------ host
static ncclComm_t comm_of(pacim_ctx *ctx) { return reinterpret_cast<ncclComm_t>(ctx->comm); }

// ------------------------------------------------ edge-partitioned build
// Every rank hashing every edge for its own sketches costs each rank the
// whole edge stream (c4, 32 sketches per rank: a 16 ms mask pass of a 25 ms
// build).  Instead rank g tests its 1/P of the upper edges against all R
// sketches (pc_ep_edges), groups the live (edge, sketch) pairs by the
// sketch's owner (r mod P, the sharding of everything downstream), and the
// ranks exchange them (ncclSend / ncclRecv; the rank's own part by a device
// copy).  What each rank receives is exactly the live pairs of its sketches;
// their bits go into the compact store's masks and the union pass reads
// them (pc_cs_list_unite).  The exchange is the only collective; every
// pair moves once.
namespace {
constexpr uint32_t EP_TILE = 4096;  // pairs per block of the owner histogram / scatter

// per-owner counts of the pair list (holes ~0 skipped); map[g] = owner << 8 | local slot
__global__ void __launch_bounds__(256) k_ep_count(const unsigned long long *__restrict__ pl,
                                                  unsigned long long cnt,
                                                  const uint32_t *__restrict__ map, uint32_t P,
                                                  unsigned long long *hist) {
  __shared__ uint32_t h[256];
  for (uint32_t o = threadIdx.x; o < P; o += blockDim.x) h[o] = 0;
  __syncthreads();
  for (unsigned long long t0 = (unsigned long long)blockIdx.x * EP_TILE; t0 < cnt;
       t0 += (unsigned long long)gridDim.x * EP_TILE) {
    const unsigned long long t1 = min(cnt, t0 + EP_TILE);
    for (unsigned long long i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
      const unsigned long long x = pl[i];
      if (x != ~0ull) atomicAdd(&h[map[x & 255u] >> 8], 1u);
    }
  }
  __syncthreads();
  for (uint32_t o = threadIdx.x; o < P; o += blockDim.x)
    if (h[o]) atomicAdd(hist + o, (unsigned long long)h[o]);
}

// the pairs into their owner's segment (cursor[o] starts at its offset),
// slot field = the owner's local slot; one global add per (tile, owner)
__global__ void __launch_bounds__(256) k_ep_scatter(const unsigned long long *__restrict__ pl,
                                                    unsigned long long cnt,
                                                    const uint32_t *__restrict__ map, uint32_t P,
                                                    unsigned long long *cursor,
                                                    unsigned long long *out) {
  __shared__ uint32_t h[256];
  __shared__ unsigned long long base[256];
  for (unsigned long long t0 = (unsigned long long)blockIdx.x * EP_TILE; t0 < cnt;
       t0 += (unsigned long long)gridDim.x * EP_TILE) {
    const unsigned long long t1 = min(cnt, t0 + EP_TILE);
    for (uint32_t o = threadIdx.x; o < P; o += blockDim.x) h[o] = 0;
    __syncthreads();
    for (unsigned long long i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
      const unsigned long long x = pl[i];
      if (x != ~0ull) atomicAdd(&h[map[x & 255u] >> 8], 1u);
    }
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < P; o += blockDim.x) {
      base[o] = h[o] ? atomicAdd(cursor + o, (unsigned long long)h[o]) : 0ull;
      h[o] = 0;
    }
    __syncthreads();
    for (unsigned long long i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
      const unsigned long long x = pl[i];
      if (x == ~0ull) continue;
      const uint32_t mo = map[x & 255u], o = mo >> 8;
      out[base[o] + atomicAdd(&h[o], 1u)] = (x & ~255ull) | (mo & 255u);
    }
    __syncthreads();
  }
}

// the received pairs' bits in both endpoints' row masks (rec .y words)
__global__ void k_ep_mask(const unsigned long long *__restrict__ pl, unsigned long long cnt,
                          uint32_t *rec_words, uint32_t MW) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long x = pl[i];
    const uint32_t u = (uint32_t)(x >> 36), v = (uint32_t)(x >> 8) & 0x0FFFFFFFu, j = (uint32_t)x & 255u;
    atomicOr(rec_words + ((size_t)u * MW + (j >> 5)) * 2 + 1, 1u << (j & 31));
    atomicOr(rec_words + ((size_t)v * MW + (j >> 5)) * 2 + 1, 1u << (j & 31));
  }
}
}  // namespace

unsigned long long pc_cs_ep_pairs(pacim_ctx *ctx, uint32_t MW, unsigned long long *ctr) {
  const uint32_t R = ctx->R, P = ctx->world, rank = ctx->rank;
  if (!pc_dist_active(ctx) || ctx->lean || (ctx->ucsr && !ctx->elist_ok) || ctx->hash_rule || R > 256 || ctx->nr >= (1u << 28) ||
      (getenv("PACIM_EP") && !atoi(getenv("PACIM_EP"))) || (P == 1 && !getenv("PACIM_EP")))
    return ~0ull;  // (at one rank only on request: the plain list build is the same work)
  // global slot table (all R sketches, sorted by hi32(hash(r)), then r) and
  // for each global slot its owner and the owner's local slot (its rank
  // among the owner's sketches in the same order: pc_slot_table's)
  std::vector<std::pair<uint64_t, uint32_t>> hs(R);
  for (uint32_t r = 0; r < R; r++) hs[r] = {pc_mix64(((1ull << 63) | (uint64_t)r) ^ ctx->K), r};
  std::sort(hs.begin(), hs.end(), [](const std::pair<uint64_t, uint32_t> &a,
                                     const std::pair<uint64_t, uint32_t> &b) {
    return (a.first >> 32) != (b.first >> 32) ? (a.first >> 32) < (b.first >> 32) : a.second < b.second;
  });
  const uint32_t NT = 1u << PACIM_TB;
  std::vector<uint32_t> tab32((size_t)2 * R + (NT + 2) / 2, 0);
  uint32_t *shr = tab32.data();
  uint16_t *tab = reinterpret_cast<uint16_t *>(shr + R);
  uint32_t *map = shr + R + (NT + 2) / 2;
  std::vector<uint32_t> seen(P, 0);
  for (uint32_t g = 0; g < R; g++) {
    shr[g] = (uint32_t)(hs[g].first >> 32);
    const uint32_t o = hs[g].second % P;
    map[g] = o << 8 | seen[o]++;
  }
  for (uint32_t p = 0, g = 0; p <= NT; p++) {
    while (g < R && (shr[g] >> (32 - PACIM_TB)) < p) g++;
    tab[p] = (uint16_t)g;
  }
  PC_REQUIRE(seen[rank] == ctx->R_local, PACIM_ECHECK, "edge-partitioned build: owner map");
  pc_ensure(ctx, ctx->ep_tab, tab32.size() * 4);
  PC_CUDA(cudaMemcpyAsync(ctx->ep_tab.p, tab32.data(), tab32.size() * 4, cudaMemcpyHostToDevice,
                          ctx->stream));
  const uint32_t *d_shr = ctx->ep_tab.as<uint32_t>();
  const uint16_t *d_tab = reinterpret_cast<const uint16_t *>(d_shr + R);
  const uint32_t *d_map = d_shr + R + (NT + 2) / 2;
  // counters: [0] list slots reserved, [1, 1+P) per-owner counts, then
  // cursors (P), then all ranks' counts (P x P)
  pc_ensure(ctx, ctx->ep_cnt, (1 + 2 * (size_t)P + (size_t)P * P) * 8);
  unsigned long long *c = ctx->ep_cnt.as<unsigned long long>();
  unsigned long long *cown = c + 1, *cur = cown + P, *call = cur + P;
  // this rank's 1/P of the upper edges, all sketches, into the pair list
  const uint64_t m = ctx->m, e0 = m * rank / P, e1 = m * (rank + 1) / P;
  const bool same = ctx->ep_gen == ctx->hint_gen && ctx->ep_K == ctx->K;
  unsigned long long cap = same ? ctx->ep_hint + ctx->ep_hint / 16 + (1ull << 22) : 0;
  if (const char *e = getenv("PACIM_EP_CAP")) cap = std::max(1LL, atoll(e));  // tests: overflow
  if (!cap) {
    size_t fr = 0, tot = 0;
    pc_mem_info(ctx, &fr, &tot);
    fr += ctx->cs_plist.bytes;
    cap = std::min<unsigned long long>(fr / 6 / 8, 1ull << 33);
  }
  // phase marks (PACIM_BUILD_TIMES=1: printed to stderr)
  const bool times = getenv("PACIM_BUILD_TIMES") != nullptr;
  cudaEvent_t ev[5] = {};
  if (times)
    for (auto &e : ev) PC_CUDA(cudaEventCreate(&e));
  if (times) PC_CUDA(cudaEventRecord(ev[0], ctx->stream));
  unsigned long long reserved = 0;
  for (int attempt = 0; attempt < 2; attempt++) {
    if (ctx->cs_plist.bytes < cap * 8) {
      pc_free(ctx, ctx->cs_plist);
      pc_ensure(ctx, ctx->cs_plist, cap * 8);
    }
    PC_CUDA(cudaMemsetAsync(c, 0, (1 + 2 * (size_t)P) * 8, ctx->stream));
    // (its live count, pairs of every rank's sketches, goes to a scratch
    // counter: the rank's own live pairs are what it receives)
    pc_ep_edges(ctx, e0, e1, d_shr, d_tab, R, ctx->cs_plist.as<unsigned long long>(), c, cap,
                ctr + 20);
    PC_CUDA(cudaMemcpyAsync(&reserved, c, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (reserved <= cap) break;
    PC_REQUIRE(attempt == 0, PACIM_ECHECK, "edge-partitioned build: pair list overflow twice");
    cap = reserved;  // exact: every warp reserved its chunks (the pass is repeated)
  }
  ctx->ep_hint = reserved;
  ctx->ep_gen = ctx->hint_gen;
  ctx->ep_K = ctx->K;
  if (times) PC_CUDA(cudaEventRecord(ev[1], ctx->stream));
  // group by owner
  const unsigned long long *pl = ctx->cs_plist.as<unsigned long long>();
  const unsigned tg = pc_grid(ctx, (reserved + EP_TILE - 1) / EP_TILE * 256, 256, 4);
  k_ep_count<<<tg, 256, 0, ctx->stream>>>(pl, reserved, d_map, P, cown);
  PC_CHECK_LAUNCH();
  std::vector<unsigned long long> sc(P), so(P + 1, 0);
  PC_CUDA(cudaMemcpyAsync(sc.data(), cown, (size_t)P * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  for (uint32_t o = 0; o < P; o++) so[o + 1] = so[o] + sc[o];
  pc_ensure(ctx, ctx->ep_send, std::max<unsigned long long>(so[P], 1) * 8);
  unsigned long long *send = ctx->ep_send.as<unsigned long long>();
  PC_CUDA(cudaMemcpyAsync(cur, so.data(), (size_t)P * 8, cudaMemcpyHostToDevice, ctx->stream));
  k_ep_scatter<<<tg, 256, 0, ctx->stream>>>(pl, reserved, d_map, P, cur, send);
  PC_CHECK_LAUNCH();
  if (times) PC_CUDA(cudaEventRecord(ev[2], ctx->stream));
  // every rank's per-owner counts -> what this rank receives from each
  std::vector<unsigned long long> all((size_t)P * P);
  PC_NCCL(ncclAllGather(cown, call, P, ncclUint64, comm_of(ctx), ctx->stream));
  PC_CUDA(cudaMemcpyAsync(all.data(), call, (size_t)P * P * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<unsigned long long> ro(P + 1, 0);
  for (uint32_t q = 0; q < P; q++) ro[q + 1] = ro[q] + all[(size_t)q * P + rank];
  const unsigned long long total = ro[P];
  PC_REQUIRE(all[(size_t)rank * P + rank] == sc[rank], PACIM_ECHECK, "edge-partitioned build: counts");
  // the receive buffer is the pair list (its pairs were scattered to send)
  if (ctx->cs_plist.bytes < std::max<unsigned long long>(total, 1) * 8) {
    pc_free(ctx, ctx->cs_plist);
    pc_ensure(ctx, ctx->cs_plist, std::max<unsigned long long>(total, 1) * 8);
  }
  unsigned long long *recv = ctx->cs_plist.as<unsigned long long>();
  if (sc[rank])
    PC_CUDA(cudaMemcpyAsync(recv + ro[rank], send + so[rank], sc[rank] * 8, cudaMemcpyDeviceToDevice,
                            ctx->stream));
  if (P > 1) {
    PC_NCCL(ncclGroupStart());
    for (uint32_t q = 0; q < P; q++) {
      if (q == rank) continue;
      if (sc[q]) PC_NCCL(ncclSend(send + so[q], sc[q], ncclUint64, (int)q, comm_of(ctx), ctx->stream));
      const unsigned long long rq = ro[q + 1] - ro[q];
      if (rq) PC_NCCL(ncclRecv(recv + ro[q], rq, ncclUint64, (int)q, comm_of(ctx), ctx->stream));
    }
    PC_NCCL(ncclGroupEnd());
  }
  if (times) PC_CUDA(cudaEventRecord(ev[3], ctx->stream));
  // the pairs' bits in the row masks (the compact store's entries)
  if (total)
    k_ep_mask<<<pc_grid(ctx, total, 256, 8), 256, 0, ctx->stream>>>(recv, total,
                                                                  ctx->cs_rec.as<uint32_t>(), MW);
  PC_CHECK_LAUNCH();
  ctx->launches += 3;
  if (times) {
    PC_CUDA(cudaEventRecord(ev[4], ctx->stream));
    PC_CUDA(cudaEventSynchronize(ev[4]));
    float t[4];
    for (int i = 0; i < 4; i++) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    fprintf(stderr,
            "ep pairs ms: pass %.3f (edges %llu of %llu, list %llu) group %.3f (%llu pairs) exchange "
            "%.3f (recv %llu) masks %.3f\n",
            t[0], (unsigned long long)(e1 - e0), (unsigned long long)m, reserved, t[1], so[P], t[2],
            total, t[3]);
    for (auto &e : ev) cudaEventDestroy(e);
  }
  return total;
}

void pc_nccl_unique_id(void *out) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  PC_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
}

void pc_init_comm(pacim_ctx *ctx, int rank, int world, const void *id) {
  pc_free_comm(ctx);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  PC_NCCL(ncclCommInitRank(&c, world, uid, rank));
  ctx->comm = c;
  ctx->comm_rank = rank;
  ctx->comm_world = world;
}

void pc_free_comm(pacim_ctx *ctx) {
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);  // a launched select graph
  if (ctx->dist_graph) {
    cudaGraphExecDestroy(reinterpret_cast<cudaGraphExec_t>(ctx->dist_graph));
    ctx->dist_graph = nullptr;
  }
  if (ctx->dist_cap_stream) {
    cudaStreamDestroy(ctx->dist_cap_stream);
    ctx->dist_cap_stream = nullptr;
  }
  if (ctx->comm) {
    cudaStreamSynchronize(ctx->stream);
    ncclCommDestroy(comm_of(ctx));
  }
  ctx->comm = nullptr;
  ctx->comm_rank = 0;
  ctx->comm_world = 1;
}

void pc_dist_restore(pacim_ctx *ctx) {
  if (ctx->cs && ctx->dist_cov_valid && ctx->dist_cov_n) {
    k_dist_uncover<<<pc_grid(ctx, ctx->dist_cov_n, 256), 256, 0, ctx->stream>>>(
        ctx->cs_E.as<uint32_t>(), ctx->dist_cov_old.as<unsigned long long>(), ctx->dist_cov_n);
    PC_CHECK_LAUNCH();
  }
  ctx->dist_cov_valid = false;
  ctx->dist_cov_n = 0;
}

// the sharded paths run when the build's shard matches the communicator; at
// world 1 only on request (PACIM_FORCE_DIST=1: the one-GPU test of the same code)
bool pc_dist_active(const pacim_ctx *ctx) {
  return ctx->comm && ctx->comm_world == (int)ctx->world && ctx->comm_rank == (int)ctx->rank &&
         (ctx->world > 1 || getenv("PACIM_FORCE_DIST") != nullptr);
}

// End of a sharded build: gain0 all-reduced (H7 summed over the ranks'
// sketches) and, if any rank has hub giants, the hot sums too.  Recorded
// in t_build ("including the all-reduce at P > 1").
void pc_dist_build_finish(pacim_ctx *ctx) {
  if (!pc_dist_active(ctx)) return;
  cudaEvent_t a, b;
  PC_CUDA(cudaEventCreate(&a));
  PC_CUDA(cudaEventCreate(&b));
  PC_CUDA(cudaEventRecord(a, ctx->stream));
  TmpBuf flag(ctx);
  pc_ensure(ctx, flag, 8);
  const int local = (!ctx->compressed && ctx->hot_any) ? 1 : 0;
  PC_CUDA(cudaMemcpyAsync(flag.p, &local, 4, cudaMemcpyHostToDevice, ctx->stream));
  PC_NCCL(ncclAllReduce(flag.p, flag.p, 1, ncclInt32, ncclMax, comm_of(ctx), ctx->stream));
  PC_NCCL(ncclAllReduce(ctx->gain0.p, ctx->gain0.p, ctx->n, ncclInt64, ncclSum, comm_of(ctx),
                        ctx->stream));
  int any = 0;
  PC_CUDA(cudaMemcpyAsync(&any, flag.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->dist_hot = any != 0;
  if (any) {  // the global hot sums, beside this rank's own (its covers use those)
    pc_ensure(ctx, ctx->dist_ghot, (size_t)ctx->n * 8);
    if (local)
      PC_CUDA(cudaMemcpyAsync(ctx->dist_ghot.p, ctx->hotsum.p, (size_t)ctx->n * 8,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    else
      PC_CUDA(cudaMemsetAsync(ctx->dist_ghot.p, 0, (size_t)ctx->n * 8, ctx->stream));
    PC_NCCL(ncclAllReduce(ctx->dist_ghot.p, ctx->dist_ghot.p, ctx->n, ncclInt64, ncclSum,
                          comm_of(ctx), ctx->stream));
  }
  PC_CUDA(cudaEventRecord(b, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ctx->stats.t_build_ms += ms;
  ctx->stats.t_gain_ms += ms;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}

// robust path: per step the argmax on the host, a dense delta vector, one
// all-reduce; works on every store (dense, compact, compressed)
static void dist_select_robust(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num) {
  const uint32_t n = ctx->n;
  TmpBuf gb(ctx), db(ctx), sb(ctx);
  pc_ensure(ctx, gb, (size_t)n * 8);
  pc_ensure(ctx, db, (size_t)n * 8);
  pc_ensure(ctx, sb, 16);
  int64_t *gain = gb.as<int64_t>(), *delta = db.as<int64_t>();
  PC_CUDA(cudaMemcpyAsync(gain, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  PC_CUDA(cudaMemsetAsync(delta, 0, (size_t)n * 8, ctx->stream));
  if (ctx->compressed) {
    pc_select_reset_compressed(ctx);
  } else {
    pc_select_reset(ctx);  // restores the previous selection's flags
    if (k > ctx->sel_k_cap) {  // covered list for k steps
      ctx->sel_k_cap = k;
      ctx->sel_list_valid = false;
      pc_select_reset(ctx);
    }
  }
  for (uint32_t i = 0; i < k; i++) {
    uint32_t s = 0;
    int64_t g = 0, loc = 0;
    pc_argmax(ctx, gain, n, &s, &g);
    if (ctx->compressed) {
      pc_cover_compressed(ctx, s, delta, &loc);
      PC_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
      pc_cover_local(ctx, s, delta, &loc);
    }
    PC_CUDA(cudaMemcpyAsync(sb.p, &loc, 8, cudaMemcpyHostToDevice, ctx->stream));
    PC_NCCL(ncclGroupStart());
    PC_NCCL(ncclAllReduce(delta, delta, n, ncclInt64, ncclSum, comm_of(ctx), ctx->stream));
    PC_NCCL(ncclAllReduce(sb.p, sb.p, 1, ncclInt64, ncclSum, comm_of(ctx), ctx->stream));
    PC_NCCL(ncclGroupEnd());
    k_dist_add<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(
        reinterpret_cast<long long *>(gain), reinterpret_cast<long long *>(delta), n);
    k_dist_set<<<1, 1, 0, ctx->stream>>>(reinterpret_cast<long long *>(gain), s, -1);
    PC_CHECK_LAUNCH();
    int64_t gsum = 0;
    PC_CUDA(cudaMemcpyAsync(&gsum, sb.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    PC_REQUIRE(gsum == g, PACIM_ECHECK, "sharded select: sum of delta_r differs from the argmax gain");
    seeds[i] = s;
    gain_num[i] = g;
  }
}

// fast path on the compact store: no host synchronisation per step
static bool dist_select_fast(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num) {
  const uint32_t n = ctx->n, B = ctx->R_local;
  const int world = ctx->comm_world;
  const unsigned long long cap =
      getenv("PACIM_DIST_CAP") ? (unsigned long long)std::max(1LL, atoll(getenv("PACIM_DIST_CAP")))
                               : (1ull << 14);
  DSel S{};  // zeroed, padding included: its bytes are the graph's cache key
  S.rec = ctx->cs_rec.as<uint2>();
  S.MW = ctx->cs_MW;
  S.E = ctx->cs_E.as<uint32_t>();
  S.vid = ctx->cs_vid.as<uint32_t>();
  S.cid = ctx->lean ? nullptr : ctx->cid.as<uint32_t>();
  S.B = B;
  S.nv = n;
  S.list_t = ctx->cs_list_t;
  S.hot_root = ctx->d_hot.as<uint32_t>();
  S.ghot = ctx->dist_hot ? ctx->dist_ghot.as<int64_t>() : nullptr;
  uint32_t csh = 10;
  while (((uint64_t)n + (1ull << csh) - 1) >> csh > MAX_CHUNKS) csh++;
  S.csh = csh;
  S.nchunks = (uint32_t)(((uint64_t)n + (1ull << csh) - 1) >> csh);
  S.cap = cap;
  S.world = world;
  S.cov_cap = (unsigned long long)k * B;
  const size_t msg = (H_WORDS + cap) * 8;
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  S.gain = ctx->gain.as<long long>();
  // one scratch allocation: chunk cache, covered list, messages, state
  const size_t o_cmax = 0;
  const size_t o_dirty = o_cmax + (size_t)S.nchunks * sizeof(Best);
  const size_t o_dlist = o_dirty + (size_t)S.nchunks * 4;
  const size_t o_cov = (o_dlist + (size_t)S.nchunks * 4 + 15) & ~(size_t)15;
  const size_t o_covr = o_cov + 8 + S.cov_cap * 8;
  const size_t o_send = (o_covr + (size_t)B * 4 + 15) & ~(size_t)15;
  const size_t o_recv = o_send + msg;
  const size_t o_st = o_recv + msg * world;
  const size_t o_out = o_st + D_WORDS * 8;
  const size_t bytes = o_out + (size_t)k * 12 + 64;
  pc_ensure(ctx, ctx->dist_buf, bytes);
  char *base = ctx->dist_buf.as<char>();
  S.cmax = reinterpret_cast<Best *>(base + o_cmax);
  S.cdirty = reinterpret_cast<uint32_t *>(base + o_dirty);
  S.dlist = reinterpret_cast<uint32_t *>(base + o_dlist);
  S.cov_cnt = reinterpret_cast<unsigned long long *>(base + o_cov);
  S.cov_list = S.cov_cnt + 1;
  S.cov_root = reinterpret_cast<uint32_t *>(base + o_covr);
  S.send = reinterpret_cast<unsigned long long *>(base + o_send);
  S.recv = reinterpret_cast<unsigned long long *>(base + o_recv);
  S.st = reinterpret_cast<unsigned long long *>(base + o_st);
  S.gain_num = reinterpret_cast<long long *>(base + o_out);
  S.seeds = reinterpret_cast<uint32_t *>(base + o_out + (size_t)k * 8);
  // restore the covered flags of earlier selections on this store
  pc_dist_restore(ctx);
  pc_cs_select_reset(ctx);
  PC_CUDA(cudaMemsetAsync(base, 0, o_recv, ctx->stream));  // cache, flags, lists, send
  PC_CUDA(cudaMemsetAsync(S.st, 0, D_WORDS * 8, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(S.gain, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  const unsigned grid = (unsigned)ctx->sm_count;
  k_dist_chunks<<<grid, DT, 0, ctx->stream>>>(S);
  PC_CHECK_LAUNCH();
  cudaEvent_t e0, e1;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  auto enqueue_loop = [&](cudaStream_t st) {
    for (uint32_t i = 0; i < k; i++) {
      uint32_t step = i;
      void *args[] = {&S, &step};
      PC_CUDA(cudaLaunchCooperativeKernel((void *)k_dist_cover, grid, DT, args, 0, st));
      PC_NCCL(ncclAllGather(S.send, const_cast<unsigned long long *>(S.recv), H_WORDS + cap,
                            ncclUint64, comm_of(ctx), st));
      PC_CUDA(cudaLaunchCooperativeKernel((void *)k_dist_apply, grid, DT, args, 0, st));
    }
  };
  if (getenv("PACIM_DIST_NOGRAPH")) {
    enqueue_loop(ctx->stream);
  } else {
    // the loop as one CUDA graph (2k cooperative kernels + k all-gathers:
    // ~70 us of launches per step otherwise), captured on a side stream and
    // launched on the ctx stream; re-captured when its arguments change
    std::vector<unsigned char> key(sizeof(S) + 16);
    memcpy(key.data(), &S, sizeof(S));
    const uint64_t kw[2] = {(uint64_t)k, (uint64_t)(uintptr_t)ctx->comm};
    memcpy(key.data() + sizeof(S), kw, 16);
    if (!ctx->dist_graph || key != ctx->dist_graph_key) {
      if (ctx->dist_graph) {
        cudaGraphExecDestroy(reinterpret_cast<cudaGraphExec_t>(ctx->dist_graph));
        ctx->dist_graph = nullptr;
      }
      if (!ctx->dist_cap_stream)
        PC_CUDA(cudaStreamCreateWithFlags(&ctx->dist_cap_stream, cudaStreamNonBlocking));
      cudaGraph_t g = nullptr;
      PC_CUDA(cudaStreamBeginCapture(ctx->dist_cap_stream, cudaStreamCaptureModeRelaxed));
      try {
        enqueue_loop(ctx->dist_cap_stream);
      } catch (...) {
        cudaStreamEndCapture(ctx->dist_cap_stream, &g);  // leave capture mode
        if (g) cudaGraphDestroy(g);
        throw;
      }
      PC_CUDA(cudaStreamEndCapture(ctx->dist_cap_stream, &g));
      cudaGraphExec_t ge = nullptr;
      PC_CUDA(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphDestroy(g);
      ctx->dist_graph = ge;
      ctx->dist_graph_key = key;
    }
    PC_CUDA(cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(ctx->dist_graph), ctx->stream));
  }
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  unsigned long long st[D_WORDS], covn = 0;
  std::vector<long long> hg(k);
  PC_CUDA(cudaMemcpyAsync(st, S.st, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(&covn, S.cov_cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(seeds, S.seeds, (size_t)k * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(hg.data(), S.gain_num, (size_t)k * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms = ms;
  ctx->stats.kernel_launches_select = 2 * k + 1;
  // keep the covered list so the next selection can restore the flags
  PC_REQUIRE(covn <= S.cov_cap, PACIM_ECHECK, "sharded select: covered list overflowed");
  pc_ensure(ctx, ctx->dist_cov_old, std::max<size_t>(covn, 1) * 8);
  PC_CUDA(cudaMemcpyAsync(ctx->dist_cov_old.p, S.cov_list, covn * 8, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  ctx->dist_cov_n = covn;
  ctx->dist_cov_valid = true;
  if (st[D_REPLAY]) return false;
  PC_REQUIRE(!st[D_CHECK], PACIM_ECHECK, "sharded select: sum of delta_r differs from the argmax gain");
  for (uint32_t i = 0; i < k; i++) gain_num[i] = hg[i];
  return true;
}

void pc_dist_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num) {
  PC_REQUIRE(pc_dist_active(ctx), PACIM_ESTATE,
             "sharded build: pacim_init_comm(rank, world) with the build's shard first");
  PC_REQUIRE(ctx->selector == 0 || ctx->selector == 3, PACIM_ENOTIMPL,
             "sharded select: the incremental selector only (auto selects it)");
  ctx->stats.select_dist_replays = 0;
  if (ctx->cs && !getenv("PACIM_DIST_ROBUST")) {
    if (dist_select_fast(ctx, k, seeds, gain_num)) return;
    ctx->stats.select_dist_replays = 1;
  }
  pc_dist_restore(ctx);  // the fast path's covered flags
  cudaEvent_t e0, e1;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  dist_select_robust(ctx, k, seeds, gain_num);
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms += ms;
}
