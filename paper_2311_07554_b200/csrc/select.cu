// select.cu — Step 2 of Alg. 1: the device-resident greedy loop
// over the uncompressed store (H8-H12).
//
// One persistent cooperative kernel runs all k steps:
//   A  NextSeed: argmax of (gain desc, id asc) over v (R5, R6) through a
//      two-level tournament array (the Win-Tree layout of P:2658-2664,
//      flattened): per-chunk maxima; a chunk is rescanned only when the
//      vertex holding its maximum lost gain (gains only decrease, so a drop
//      anywhere else cannot change the chunk's (max, argmax)).
//   B  MarkSeed: one warp per sketch slot j reads the seed's CC
//      from its root slot (HIGH | size): delta_j = size unless the CC is
//      already covered (bit 30), then marks it covered.
//   C  incremental gain update (R17): the members of every newly covered CC
//      lose delta_j.  Small CCs are enumerated by the slot's warp with a
//      shared-memory queue (warp_bfs).  The others are enumerated by ONE
//      asynchronous traversal shared by all slots: a row carries the set of
//      slots it was newly reached in (a bitmask), its adjacency is read and
//      each edge hashed once, and only the edge's candidate slots (the bucket
//      table of the build) that are in the mask are tested, a 32-slot word at
//      a time.  Work items sit in a queue served by every warp of the grid —
//      no barrier per BFS level; the traversal ends at quiescence (every
//      pushed item expanded, no producer left).  A row of degree > CH splits
//      its adjacency into CH-edge chunk items (carrying one 32-slot mask word
//      each), so hubs are expanded by many warps at once.  CCs larger than
//      big_t are covered by one dense pass over the store.
// The covered bits are cleared before the next selection (the list of
// covered root slots is kept).  gain_num[i] = sum_j delta_j; the host checks
// it against the argmax gain.
#include <cooperative_groups.h>
#include <cstddef>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "pacim_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int SEL_THREADS = 512;
constexpr int SEL_WARPS = SEL_THREADS / 32;
constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t COV = 0x40000000u;   // covered bit of a root slot
constexpr uint32_t SIZE = 0x3FFFFFFFu;  // CC size bits of a root slot
constexpr uint32_t MAX_CHUNKS = 4096;   // argmax cache: chunk maxima
constexpr uint32_t MAX_BW = 32;         // slot-mask words per row: select supports B <= 1024
constexpr uint32_t CH_DEFAULT = 256;    // edges per chunk item
constexpr unsigned long long FULL = 0xffffffffu;

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

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acq32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t exch_release(uint32_t *p, uint32_t x) {
  uint32_t v;
  asm volatile("atom.release.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "r"(x) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t exch_acq_rel(uint32_t *p, uint32_t x) {
  uint32_t v;
  asm volatile("atom.acq_rel.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "r"(x) : "memory");
  return v;
}
__device__ __forceinline__ void add_release(unsigned long long *p, unsigned long long x) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}

// queue control words (u64 tickets, each in its own 128-B line)
// Queue tickets (tail / head / done) in their own 128-B lines.  QC_PROD + 16
// * parity: producers of B still running in a step of that parity.
enum { QC_TAIL = 0, QC_HEAD = 16, QC_DONE = 32, QC_PROD = 48, QC_WORDS = 80 };
// diagnostics (u64): steps, dense steps, warp-BFS slots, deferred slots,
// row items, chunk items, chunks expanded inline (queue guard)
enum { DG_STEPS = 0, DG_DENSE, DG_WARP, DG_DEFER, DG_ROWS, DG_CHUNKS, DG_INLINE, DG_ABORT,
       DG_EDGES, DG_HOT, DG_WORDS = 10 };
constexpr unsigned long long WATCHDOG_NS = 20000000000ull;  // a 20 s wait is a bug: abort

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Work-queue slot (bounded MPMC ring with per-slot sequence numbers): the
// producer of ticket t waits for seq == t, writes, sets seq = t + 1; the
// consumer of ticket t waits for seq == t + 1, reads, sets seq = t + Q.
// cw = chunk << 6 | mask word; chunk == CW_ROW marks a row item (its slots
// are taken from the row's pending mask).
struct Item {
  uint32_t seq, row, cw, bits;
};
constexpr uint32_t CW_ROW = 0xFFFFFFFFu;

struct Sel {
  Ep ep;  // slot epochs of the store (build.cu): every slot read through ep_rd
  // graph (traversals over live edges)
  const uint64_t *off;
  const uint32_t *nbr;
  uint64_t K, t32;
  const uint32_t *tcsr;  // per-edge models: T32 - toff per CSR entry
  int wic;                // per-edge thresholds (WIC or Uniform)
  uint32_t toff;
  const uint32_t *g_shr;   // hi32(hash(r)) of slot j (sorted)
  const uint64_t *hr64;    // hash(r) of slot j (R20 decorrelated rule)
  int decor;               // R20: live <=> hi32(mix64(hash(r) ^ hash(e))) < T32
  const uint16_t *g_tab;   // candidate bucket table of the sorted slots
  // store
  uint32_t *L;
  const uint32_t *smap;    // slot -> f << 16 | c of its store window (pc_addr)
  int onew;                // one window [0, B): address row * B + j
  uint32_t nr, B, BW, nv;  // rows, slots, mask words per row, vertices
  const uint32_t *cid, *rmap;
  // per step
  long long *target;       // gain vector (single rank) or delta vector (multi-rank)
  uint32_t *dl;            // B: delta_j of a CC enumerated by traversal (0: none)
  uint32_t *cov_root;      // B: root row of a big CC covered in slot j, or NONE
  uint32_t *cov_delta;     // B
  int *dense;              // [2] by step parity: a big CC was covered
  unsigned long long *cov_list, *cov_cnt;  // covered root-slot indices (restored later)
  unsigned long long cov_cap;
  uint32_t big_t;
  int warp_ok;             // small CCs may use warp_bfs
  uint32_t warp_max;       // ... up to this many vertices (<= QCAP)
  const int64_t *hotsum;   // per vertex: sizes of the giant hot CCs containing it (or null)
  const uint32_t *hot_root, *hot_size;  // per slot: the hub's root row and CC size
  int trav_only;           // no store: dl[] preset per slot, only the member traversal
  // asynchronous traversal
  uint32_t *vis;           // rows x BW: slots in which the row was visited this step
  uint32_t *pend;          // rows x BW: slots reached but not yet expanded (light rows)
  uint32_t *inq;           // rows: row is in the queue
  Item *ring;              // work queue (rows, chunk items), Q = qmask + 1 slots
  unsigned long long qmask, qguard;  // chunk items are queued only below qguard outstanding
  unsigned long long *qc;  // QC_* words
  const uint32_t *hidx;    // rows: hub index or NONE (HLA valid iff hla_off != nullptr)
  const unsigned long long *hla_off;  // [nhub * B + 1] segment offsets by (hub, slot)
  const uint32_t *hla_row; // the rows joined to the hub by an edge live in the slot
  uint32_t ch;             // edges per chunk item
  uint32_t lkeep;          // rows a warp keeps for itself (local continuation), <= LCAP
  uint32_t max_sleep;      // ns: backoff cap of idle queue pollers
  uint32_t *touched;       // [2][rows]: rows visited in a step of parity par (each once)
  uint32_t *tflag;         // [rows]: row is in a touched list
  uint32_t *tcnt;          // [2]
  // argmax cache (single rank): marks of step i go to dlist[i & 1], consumed
  // at the end of step i; the buffer is re-armed at the end of step i + 1
  Best *cmax;
  uint32_t *cdirty, *dlist, *dcnt;  // dlist[2][nchunks], dcnt[2]
  uint32_t par, csh, nchunks;
  int track;
  unsigned long long *diag;
  DeltaList dlst;          // multi-rank sparse deltas (v == nullptr: off)
  uint32_t tlstep;
  unsigned long long *ilog;  // optional item log: [0] count, then {start, end, step, edges} x cap
  unsigned long long ilog_cap;
  unsigned long long *tl;  // optional timeline: 8 %globaltimer stamps per step (block 0, thread 0)
};

__device__ __forceinline__ void stamp(const Sel &S, uint32_t step, int i) {
  if (S.tl && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    S.tl[(size_t)step * 8 + i] = t;
  }
}

__device__ __forceinline__ void mark_dirty(const Sel &S, uint32_t c) {
  if (atomicExch(S.cdirty + c, 1u) == 0u)
    S.dlist[(size_t)S.par * S.nchunks + atomicAdd(S.dcnt + S.par, 1u)] = c;
}

// remember a row whose visited bits must be cleared before the next step
__device__ __forceinline__ void touch(const Sel &S, uint32_t row) {
  if (atomicExch(S.tflag + row, 1u) == 0u)
    S.touched[(size_t)S.par * S.nr + atomicAdd(S.tcnt + S.par, 1u)] = row;
}

__device__ __forceinline__ void sub_gain(const Sel &S, uint32_t u, long long d) {
  atomicAdd((unsigned long long *)&S.target[u], (unsigned long long)(-d));
  S.dlst.add(u, -d);
  if (S.track) {
    const uint32_t c = u >> S.csh;
    if (__ldcg(&S.cmax[c].v) == u) mark_dirty(S, c);  // only the chunk's argmax matters
  }
}

__device__ __forceinline__ void q_write(Item *ring, unsigned long long mask, unsigned long long t,
                                        uint32_t row, uint32_t cw, uint32_t bits) {
  Item *it = ring + (t & mask);
  while (ld_acq32(&it->seq) != (uint32_t)t) __nanosleep(32);  // freed by its last consumer
  it->row = row;
  it->cw = cw;
  it->bits = bits;
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&it->seq), "r"((uint32_t)(t + 1))
               : "memory");
}

// The warp's local stack of rows it discovered and expands itself (no queue
// hand-off); rows beyond the first `lkeep` go to the shared queue.
struct LStack {
  uint32_t *row, *x, *cnt;  // shared memory of the warp
  uint32_t keep;
  uint32_t *trow, *tn;      // rows expanded, touched in batches of 32 (off the hop's path)
};
constexpr uint32_t LCAP = 16;

// the warp's pending touches, one lane per row (before the item is done)
__device__ __forceinline__ void flush_touches(const Sel &S, const LStack *ls) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const uint32_t n = *ls->tn;
  if ((uint32_t)lane < n) touch(S, ls->trow[lane]);
  __syncwarp();
  if (lane == 0) *ls->tn = 0;
  __syncwarp();
}

// (row wr of vertex w, mask word wd) newly reached in the slots nb: schedule
// its expansion (one queue entry per row at a time; bits arriving meanwhile
// merge into it)
__device__ __forceinline__ void reach(const Sel &S, uint32_t wr, uint32_t w, uint32_t wd,
                                      uint32_t nb, const LStack *ls) {
  atomicOr(S.pend + (size_t)wr * S.BW + wd, nb);
  // release: a consumer that clears the flag after this exchange (acq_rel)
  // sees the bits
  if (exch_release(S.inq + wr, 1u) == 0u) {
    if (ls) {
      const uint32_t at = atomicAdd(ls->cnt, 1u);
      if (at < ls->keep) {
        ls->row[at] = wr;
        ls->x[at] = w;
        return;
      }
    }
    q_write(S.ring, S.qmask, atomicAdd(S.qc + QC_TAIL, 1ull), wr, CW_ROW, 0);
  }
}

// Phase B for slot j (one thread): MarkSeed and classification.
__device__ __forceinline__ uint32_t cover_slot(const Sel &S, uint32_t srow, uint32_t j) {
  uint32_t delta = 1;
  S.dl[j] = 0;
  S.cov_root[j] = NONE;
  if (srow == NONE) return delta;  // isolated seed: singleton in every sketch
  const uint32_t sl =
      ep_rd(S.L[S.onew ? (size_t)srow * S.B + j : pc_addr(S.smap, S.nr, srow, j)], S.ep);
  if (sl == (PACIM_HIGH | 1u)) return delta;  // singleton {s} (root of size 1)
  const uint32_t root = (sl & PACIM_HIGH) ? srow : sl;
  const size_t ra = S.onew ? (size_t)root * S.B + j : pc_addr(S.smap, S.nr, root, j);
  uint32_t *rs = S.L + ra;
  // (a root of >= 2 members: its slot is of this build's epoch)
  const uint32_t x = ep_rd(atomicOr(rs, COV), S.ep);  // covered from now on
  if (x & COV) return 0;                              // covered by an earlier seed
  delta = x & SIZE;
  const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
  if (at < S.cov_cap) S.cov_list[at] = ra;
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

// Warp-local BFS of the seed's CC in slot j (<= QCAP vertices) with a
// shared-memory queue and visited set; applies the gain updates.  Returns
// false, before updating anything, if it meets a vertex of degree > WARP_DEG
// (the shared traversal then takes the slot and reads that adjacency once
// for all slots).
constexpr uint32_t QCAP = 512;
constexpr uint32_t HCAP = 1024;
constexpr uint64_t WARP_DEG = 1024;
// + mask, nonzero-word list (u8), local stack (rows, vertices, count)
constexpr uint32_t WARP_WORDS = QCAP + HCAP + 1 + MAX_BW + MAX_BW / 4 + 2 * 16 + 1 + 33;

// shared-memory words of the slot tables (shr[B] + tab[2^TB + 1] u16), 16-B aligned
__host__ __device__ __forceinline__ uint32_t table_words(uint32_t B) {
  return (((uint32_t)B * 4 + ((1u << PACIM_TB) + 1) * 2 + 15) & ~15u) / 4;
}

__device__ bool warp_bfs(const Sel &S, uint32_t s, uint32_t j, uint32_t delta, uint32_t *q,
                         uint32_t *hs, uint32_t *tail, const uint32_t *shr) {
  const int lane = threadIdx.x & 31;
  const uint32_t hr = shr[j];
  const uint64_t hrj = S.decor ? __ldg(S.hr64 + j) : 0;
  for (uint32_t i = lane; i < HCAP; i += 32) hs[i] = NONE;
  __syncwarp();
  if (lane == 0) {
    q[0] = s;
    hs[(s * 2654435761u) & (HCAP - 1)] = s;
    *tail = 1;
  }
  __syncwarp();
  // level-synchronous within the warp: the (vertex, edge) pairs of up to 32
  // queued vertices are spread over the lanes, so the latency is the CC's
  // depth, not its size
  for (uint32_t head = 0; head < *tail;) {
    const uint32_t lvl_end = *tail;
    for (uint32_t base = head; base < lvl_end; base += 32) {
      const uint32_t idx = base + lane;
      const uint32_t x = idx < lvl_end ? q[idx] : 0u;
      uint64_t e0 = 0, deg = 0;
      if (idx < lvl_end) {
        e0 = S.off[x];
        deg = S.off[x + 1] - e0;
      }
      if (__any_sync(FULL, deg > WARP_DEG)) return false;  // a hub: the shared traversal
      uint32_t pre = (uint32_t)deg;  // inclusive scan of the degrees
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, pre, d);
        if (lane >= d) pre += y;
      }
      const uint32_t total = __shfl_sync(FULL, pre, 31);
      pre -= (uint32_t)deg;  // exclusive
      // WU rounds of 32 pairs at a time: their CSR (and threshold) loads are
      // issued back to back, then the pairs are tested and inserted
      constexpr int WU = 4;
      for (uint32_t c = 0; c < total; c += 32 * WU) {
        uint32_t wv[WU], xv[WU];
        uint64_t tv[WU];
#pragma unroll
        for (int u = 0; u < WU; u++) {
          const uint32_t t = c + 32 * u + lane;
          uint32_t a = 0;  // the lane (vertex) owning pair t: largest a with pre[a] <= t
#pragma unroll
          for (int b = 16; b; b >>= 1) {
            const uint32_t pa = __shfl_sync(FULL, pre, a + b);
            if (pa <= t) a += b;
          }
          xv[u] = __shfl_sync(FULL, x, a);
          const uint64_t ea = __shfl_sync(FULL, e0, a);
          const uint32_t pra = __shfl_sync(FULL, pre, a);
          wv[u] = NONE;
          tv[u] = S.t32;
          if (t < total) {
            const uint64_t e = ea + (t - pra);
            wv[u] = S.nbr[e];
            if (S.wic) tv[u] = (uint64_t)S.tcsr[e] + S.toff;  // R4 / R19
          }
        }
#pragma unroll
        for (int u = 0; u < WU; u++) {
          const uint32_t w = wv[u], xa = xv[u];
          if (w == NONE) continue;
          const uint64_t lo = xa < w ? xa : w, hi = xa < w ? w : xa;
          const uint64_t he64 = pc_mix64(((lo << 32) | hi) ^ S.K);
          const uint32_t he = (uint32_t)(he64 >> 32);
          const uint64_t T = tv[u];
          if (S.decor) {  // R20
            if (T < (1ull << 32) && (pc_mix64(hrj ^ he64) >> 32) >= T) continue;
          } else if ((uint64_t)(hr ^ he) >= T) {
            continue;  // R3
          }
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
      }
      __syncwarp();
    }
    head = lvl_end;
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

// Expand CSR entry e of vertex x for the slots in mask M (BW words): hash
// the edge once (R2), enumerate its candidate slots from the bucket table
// (exact: the top clz(T-1) bits of hash(r) and hash(e) must agree), test
// the masked candidates 32 at a time (R3 live test), and for the slots in
// which the neighbour is new: one gain update with the sum of their deltas
// and one scheduling of its expansion.
__device__ __forceinline__ void expand_edge(const Sel &S, uint32_t x, uint32_t w, uint64_t T,
                                            const uint32_t *M, uint32_t s, const uint32_t *shr,
                                            const uint16_t *tab, const uint32_t *sdl,
                                            const LStack *ls) {
  const uint64_t a = x < w ? x : w, b = x < w ? w : x;
  if (T == 0) return;
  const uint64_t he64 = pc_mix64(((a << 32) | b) ^ S.K);
  const uint32_t he = (uint32_t)(he64 >> 32);
  const uint32_t wb = __clz((uint32_t)(T - 1));
  uint32_t lo, hi;
  if (S.decor) {  // R20: every slot is a candidate
    lo = 0;
    hi = S.B;
  } else if (wb >= PACIM_TB) {
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
  if (lo >= hi) return;
  // every candidate is live when T is the full bucket width 2^(32 - wb) and
  // the table resolves all wb bits
  const bool all_live = S.decor ? T >= (1ull << 32) : (wb <= PACIM_TB && T == (1ull << (32 - wb)));
  uint32_t wr = NONE;
  const uint32_t w0 = lo >> 5, w1 = (hi - 1) >> 5;
  for (uint32_t wd = w0; wd <= w1; wd++) {
    uint32_t rb = 0xFFFFFFFFu;
    if (wd == w0) rb &= 0xFFFFFFFFu << (lo & 31);
    if (wd == w1) rb &= 0xFFFFFFFFu >> (31 - ((hi - 1) & 31));
    const uint32_t bits = M[wd] & rb;
    if (!bits) continue;
    uint32_t live = bits;
    if (!all_live) {
      live = 0;
      for (uint32_t t = bits; t; t &= t - 1) {
        const uint32_t bit = __ffs(t) - 1;
        const uint32_t j = wd * 32 + bit;
        const bool lv = S.decor ? (pc_mix64(__ldg(S.hr64 + j) ^ he64) >> 32) < T
                                : (uint64_t)(shr[j] ^ he) < T;
        if (lv) live |= 1u << bit;
      }
      if (!live) continue;
    }
    uint32_t cm = NONE;
    if (wr == NONE) {
      wr = S.cid[w];
      if (S.track) cm = __ldcg(&S.cmax[w >> S.csh].v);  // in flight with the row lookup
    }
    const uint32_t old = atomicOr(S.vis + (size_t)wr * S.BW + wd, live);
    const uint32_t nb = live & ~old;
    if (!nb) continue;
    long long d = 0;
    for (uint32_t t = nb; t; t &= t - 1) d += sdl[wd * 32 + __ffs(t) - 1];
    if (w != s) {
      atomicAdd((unsigned long long *)&S.target[w], (unsigned long long)(-d));
      S.dlst.add(w, -d);
      if (S.track) {  // only the chunk's argmax matters (gains only decrease)
        if (cm == NONE) cm = __ldcg(&S.cmax[w >> S.csh].v);
        if (cm == w) mark_dirty(S, w >> S.csh);
      }
    }
    reach(S, wr, w, wd, nb, ls);  // the row is touched when it is expanded
  }
}

// Expand CSR entries [ea, eb) of vertex x (lanes strided): the neighbour and
// threshold loads of EU entries per lane are issued before any of them is
// tested, so a 256-entry chunk costs about one memory latency, not eight.
constexpr int EU = 8;
__device__ __forceinline__ void load_batch(const Sel &S, uint64_t base, uint64_t eb,
                                           uint32_t (&w)[EU], uint32_t (&tm)[EU]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < EU; u++) {
    const uint64_t e = base + lane + 32 * u;
    w[u] = e < eb ? __ldcs(S.nbr + e) : NONE;
    tm[u] = (e < eb && S.wic) ? __ldcs(S.tcsr + e) : 0u;
  }
}
// pre (optional): the batch at ea already loaded, bounded by pe >= eb
__device__ __forceinline__ void expand_range(const Sel &S, uint32_t x, uint64_t ea, uint64_t eb,
                                             const uint32_t *M, uint32_t s, const uint32_t *shr,
                                             const uint16_t *tab, const uint32_t *sdl,
                                             const LStack *ls, uint32_t (*pw)[EU] = nullptr,
                                             uint32_t (*ptm)[EU] = nullptr) {
  const int lane = threadIdx.x & 31;
  for (uint64_t base = ea; base < eb; base += 32 * EU) {
    uint32_t w[EU], tm[EU];
    if (pw && base == ea) {
#pragma unroll
      for (int u = 0; u < EU; u++) {
        w[u] = base + lane + 32 * u < eb ? (*pw)[u] : NONE;
        tm[u] = (*ptm)[u];
      }
    } else {
      load_batch(S, base, eb, w, tm);
    }
#pragma unroll
    for (int u = 0; u < EU; u++) {
      if (w[u] == NONE) continue;
      const uint64_t T = S.wic ? (uint64_t)tm[u] + S.toff : S.t32;  // R3 / R4 / R19
      expand_edge(S, x, w[u], T, M, s, shr, tab, sdl, ls);
    }
  }
}

// row r newly reached from a hub in slot j (mask word wd, bit)
__device__ __forceinline__ void hub_visit(const Sel &S, uint32_t r, uint32_t j, uint32_t s,
                                          const uint32_t *sdl, const LStack *ls) {
  const uint32_t wd = j >> 5, bit = 1u << (j & 31);
  const uint32_t old = atomicOr(S.vis + (size_t)r * S.BW + wd, bit);
  if (old & bit) return;
  const uint32_t w = S.rmap[r];
  if (w != s) sub_gain(S, w, sdl[j]);
  reach(S, r, w, wd, bit, ls);
}

// Expand hub h for the pending slots in wm through the live hub adjacency:
// lane l takes slot 32 * wd + l of each nonzero mask word; segments longer
// than 32 rows are walked by the whole warp.
__device__ void expand_hub(const Sel &S, uint32_t h, const uint32_t *wm, uint32_t s,
                           const uint32_t *sdl, const LStack *ls) {
  const int lane = threadIdx.x & 31;
  for (uint32_t wd = 0; wd < S.BW; wd++) {
    const uint32_t m = wm[wd];
    if (!m) continue;
    const uint32_t j = wd * 32 + lane;
    unsigned long long a = 0, z = 0;
    if ((m >> lane) & 1u) {
      const unsigned long long key = (unsigned long long)h * S.B + j;
      a = __ldg(S.hla_off + key);
      z = __ldg(S.hla_off + key + 1);
    }
    const bool longseg = z - a > 32;
    if (!longseg)
      for (unsigned long long i = a; i < z; i++) hub_visit(S, __ldg(S.hla_row + i), j, s, sdl, ls);
    for (uint32_t lm = __ballot_sync(FULL, longseg); lm; lm &= lm - 1) {
      const int src = __ffs(lm) - 1;
      const unsigned long long la = __shfl_sync(FULL, a, src), lz = __shfl_sync(FULL, z, src);
      const uint32_t lj = wd * 32 + src;
      for (unsigned long long i = la + lane; i < lz; i += 32)
        hub_visit(S, __ldg(S.hla_row + i), lj, s, sdl, ls);
    }
  }
}

// Expand one item: a row (its pending slots taken; rows of degree > CH also
// queue their chunks 1.. as chunk items) or a chunk item.  Returns the CSR
// entries tested.
__device__ uint64_t process_item(const Sel &S, uint32_t s, uint32_t row, uint32_t x, uint32_t cw,
                                 uint32_t bits, uint32_t *wm, uint8_t *wl, const uint32_t *shr,
                                 const uint16_t *tab, const uint32_t *sdl, const LStack *ls,
                                 unsigned long long &nrow, unsigned long long &nchunk,
                                 unsigned long long &ninl) {
  const int lane = threadIdx.x & 31;
  uint64_t c_lo, c_hi;  // chunks expanded by this warp
  uint64_t e0, e1, nch;
  uint32_t pw[EU], ptm[EU];
  bool pre = false;
  if (cw == CW_ROW) {
    nrow++;
    e0 = S.off[x];  // issued before the flag exchange (independent)
    e1 = S.off[x + 1];
    // take the row's pending slots (clear the queue flag first: bits added
    // after this point re-queue the row)
    if (lane == 0) exch_acq_rel(S.inq + row, 0u);
    __syncwarp();
    const uint32_t m = lane < S.BW ? atomicExch(S.pend + (size_t)row * S.BW + lane, 0u) : 0u;
    // the first adjacency batch in flight with the exchange (CSR: immutable)
    load_batch(S, e0, min(e1, e0 + 32 * EU), pw, ptm);
    if (lane < S.BW) wm[lane] = m;
    const uint32_t nzb = __ballot_sync(FULL, m != 0);
    const uint32_t nnz = __popc(nzb);
    if (m) wl[__popc(nzb & ((1u << lane) - 1))] = lane;
    // its visited bits are cleared before the next step: touched in the
    // warp's batch (flushed before the item is done)
    __syncwarp();
    if (*ls->tn == 32) flush_touches(S, ls);  // warp-uniform
    if (lane == 0) ls->trow[(*ls->tn)++] = row;
    __syncwarp();
    pre = true;
    nch = (e1 - e0 + S.ch - 1) / S.ch;
    c_lo = 0;
    c_hi = nnz ? nch : 0;
    if (S.hla_off && nnz) {
      const uint32_t h = S.hidx[row];
      if (h != NONE) {  // a hub: its live edges from the build, no hashing
        expand_hub(S, h, wm, s, sdl, ls);
        return 0;
      }
    }
    // chunks 1..nch-1: one item per (chunk, nonzero word), queued in batches
    // of 32 while the queue has room, else expanded here
    const uint64_t nitems = nch > 1 ? (nch - 1) * nnz : 0;
    uint64_t done_items = 0;
    while (done_items < nitems) {
      unsigned long long t0 = 0;
      const uint32_t nb = (uint32_t)(nitems - done_items < 32 ? nitems - done_items : 32);
      int ok = 0;
      if (lane == 0) {
        const unsigned long long out = ld_acq(S.qc + QC_TAIL) - ld_acq(S.qc + QC_DONE);
        if (out + nb < S.qguard) {
          ok = 1;
          t0 = atomicAdd(S.qc + QC_TAIL, (unsigned long long)nb);
        }
      }
      if (!__shfl_sync(FULL, ok, 0)) break;
      t0 = __shfl_sync(FULL, t0, 0);
      if (lane < nb) {
        const uint64_t it = done_items + lane;
        const uint32_t wd = wl[it % nnz];
        q_write(S.ring, S.qmask, t0 + lane, row, (uint32_t)((1 + it / nnz) << 6) | wd, wm[wd]);
      }
      done_items += nb;
    }
    if (nitems) {
      if (done_items < nitems) {
        ninl++;  // the queue is full: expand the rest here (with the full mask;
                 // repeated tests of already visited slots are no-ops)
        expand_range(S, x, e0, min(e1, e0 + S.ch), wm, s, shr, tab, sdl, ls, &pw, &ptm);
        pre = false;
        c_lo = 1 + done_items / nnz;
        c_hi = nch;
      } else {
        c_hi = 1;
      }
    }
  } else {
    nchunk++;
    x = S.rmap[row];
    e0 = S.off[x];
    e1 = S.off[x + 1];
    for (uint32_t q = lane; q < S.BW; q += 32) wm[q] = 0;
    __syncwarp();
    if (lane == 0) wm[cw & 63] = bits;
    __syncwarp();
    c_lo = cw >> 6;
    c_hi = c_lo + 1;
  }
  const uint64_t ea = min(e1, e0 + c_lo * S.ch), eb = min(e1, e0 + c_hi * S.ch);
  if (pre && ea == e0)
    expand_range(S, x, ea, eb, wm, s, shr, tab, sdl, ls, &pw, &ptm);
  else
    expand_range(S, x, ea, eb, wm, s, shr, tab, sdl, ls);
  return eb > ea ? eb - ea : 0;
}

// Queue phase: every warp pops items and expands them until quiescence.
// Returns the final tail (identical in every warp).  wm / wl: the warp's
// shared words for the item's mask and the list of its nonzero words; sdl:
// the block's copy of the slots' deltas (final once every B is done).
__device__ unsigned long long queue_phase(const Sel &S, uint32_t s, uint32_t *wm, uint8_t *wl,
                                          const uint32_t *shr, const uint16_t *tab,
                                          uint32_t *sdl, const unsigned long long *prod,
                                          const LStack *ls) {
  const int lane = threadIdx.x & 31;
  // wait for every producer of B; if nothing was queued the traversal is
  // already over (quiescent: no producer, nothing queued), else snapshot the
  // deltas
  __shared__ unsigned long long quiet_tail;
  if (threadIdx.x == 0) {
    unsigned ns = 32;
    const unsigned long long t0 = gtime();
    while (ld_acq(prod) != 0) {
      __nanosleep(ns);
      ns = ns < 256 ? ns * 2 : 256;
      if (gtime() - t0 > WATCHDOG_NS) {
        atomicExch(S.diag + DG_ABORT, 1ull);
        break;
      }
    }
    const unsigned long long done = ld_acq(S.qc + QC_DONE);
    const unsigned long long tail = ld_acq(S.qc + QC_TAIL);
    quiet_tail = done == tail ? tail : ~0ull;
  }
  __syncthreads();
  if (S.tl && blockIdx.x == 0 && threadIdx.x == 0) S.tl[(size_t)S.tlstep * 8 + 3] = gtime();
  const unsigned long long qt = quiet_tail;
  if (qt != ~0ull) return qt;
  for (uint32_t j = threadIdx.x; j < S.B; j += blockDim.x) sdl[j] = __ldcg(S.dl + j);
  __syncthreads();
  unsigned long long nrow = 0, nchunk = 0, ninl = 0, nedg = 0;
  for (;;) {
    unsigned long long i = 0, tend = 0;
    uint32_t row = NONE, cw = 0, bits = 0;
    int fin = 0;
    if (lane == 0) {
      unsigned ns = 32;
      bool have = false;
      const unsigned long long t0 = gtime();
      for (;;) {
        const unsigned long long tail = ld_acq(S.qc + QC_TAIL);
        if (!have && ld_rlx(S.qc + QC_HEAD) < tail) {  // reserve only when work is queued
          i = atomicAdd(S.qc + QC_HEAD, 1ull);
          have = true;
          ns = 32;
        }
        if (have) {
          Item *it = S.ring + (i & S.qmask);
          if (ld_acq32(&it->seq) == (uint32_t)(i + 1)) {  // item i is written
            row = it->row;
            cw = it->cw;
            bits = it->bits;
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&it->seq),
                         "r"((uint32_t)(i + S.qmask + 1))
                         : "memory");
            break;
          }
        }
        if (!have || i >= tail) {
          const unsigned long long done = ld_acq(S.qc + QC_DONE);
          const unsigned long long t2 = ld_acq(S.qc + QC_TAIL);
          if (done == t2 && (!have || i >= t2)) {  // quiescent: nothing queued, nobody expanding
            fin = 1;
            tend = t2;
            break;
          }
        }
        if (gtime() - t0 > WATCHDOG_NS || ld_rlx(S.diag + DG_ABORT)) {
          atomicExch(S.diag + DG_ABORT, 1ull);
          fin = 1;  // the host reports the abort
          break;
        }
        __nanosleep(ns);
        ns = ns < S.max_sleep ? ns * 2 : S.max_sleep;  // idle pollers stay off the hot lines
      }
    }
    fin = __shfl_sync(FULL, fin, 0);
    if (fin) {
      if (lane == 0 && S.diag) {
        atomicAdd(S.diag + DG_ROWS, nrow);
        atomicAdd(S.diag + DG_CHUNKS, nchunk);
        atomicAdd(S.diag + DG_INLINE, ninl);
        atomicAdd(S.diag + DG_EDGES, nedg);
      }
      return __shfl_sync(FULL, tend, 0);
    }
    row = __shfl_sync(FULL, row, 0);
    cw = __shfl_sync(FULL, cw, 0);
    bits = __shfl_sync(FULL, bits, 0);
    const unsigned long long it_t0 = S.ilog ? gtime() : 0;
    // the popped item, then the rows this warp discovered and kept (local
    // continuation: no queue hand-off); the item is done when both are
    if (lane == 0) *ls->cnt = 0;
    __syncwarp();
    uint32_t xr = cw == CW_ROW ? S.rmap[row] : NONE;  // chunk items look up x below
    uint64_t nedges = 0;
    for (int first = 1;; first = 0) {
      nedges += process_item(S, s, row, xr, cw, bits, wm, wl, shr, tab, sdl, ls, nrow, nchunk, ninl);
      __syncwarp();
      const uint32_t n = min(*ls->cnt, ls->keep);
      __syncwarp();
      if (n == 0) break;
      row = ls->row[n - 1];
      xr = ls->x[n - 1];
      cw = CW_ROW;
      __syncwarp();
      if (lane == 0) *ls->cnt = n - 1;
      __syncwarp();
    }
    nedg += nedges;
    flush_touches(S, ls);  // before QC_DONE: quiescence implies every touch
    if (lane == 0 && S.ilog) {
      const unsigned long long at = atomicAdd(S.ilog, 1ull);
      if (at < S.ilog_cap) {
        unsigned long long *r = S.ilog + 4 + at * 4;
        r[0] = it_t0;
        r[1] = gtime();
        r[2] = S.tlstep;
        r[3] = nedges;
      }
    }
    if (lane == 0) add_release(S.qc + QC_DONE, 1ull);  // after this item's pushes
  }
}

// dense pass for the big CCs covered this step: v is a member of slot j's
// covered CC iff its slot holds that root, or v is the root.  8 slots per
// lane kept in registers; DR rows in flight per warp.
constexpr int DR = 4;
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
    for (size_t v0 = warp0 * DR; v0 < S.nr; v0 += nwarps * DR) {
      uint32_t x[DR][8];
      // the rows' vertex ids, loaded with the slots (lane r: row v0 + r), so
      // the per-row gain update does not wait on a dependent load
      const uint32_t vids = (lane < DR && v0 + lane < S.nr) ? __ldg(S.rmap + v0 + lane) : NONE;
      if (S.onew) {  // one window (the default): the plain vertex-major address
#pragma unroll
        for (int r = 0; r < DR; r++)
#pragma unroll
          for (int i = 0; i < 8; i++)
            x[r][i] = (cr[i] != NONE && v0 + r < S.nr)
                          ? ep_rd(__ldcs(S.L + (v0 + r) * S.B + j0 + lane + 32 * i), S.ep)
                          : NONE;
      } else {
#pragma unroll
        for (int r = 0; r < DR; r++)
#pragma unroll
          for (int i = 0; i < 8; i++)
            x[r][i] = (cr[i] != NONE && v0 + r < S.nr)
                          ? ep_rd(__ldcs(S.L + pc_addr(S.smap, S.nr, (uint32_t)(v0 + r), j0 + lane + 32 * i)), S.ep)
                          : NONE;
      }
#pragma unroll
      for (int r = 0; r < DR; r++) {
        const uint32_t v = (uint32_t)(v0 + r);
        long long d = 0;
#pragma unroll
        for (int i = 0; i < 8; i++)
          if (cr[i] != NONE && (x[r][i] == cr[i] || v == cr[i])) d += cd[i];
        const uint32_t vid = __shfl_sync(0xffffffffu, vids, r);
        if (!__any_sync(0xffffffffu, d != 0)) continue;
        for (int q = 16; q; q >>= 1) d += __shfl_xor_sync(0xffffffffu, d, q);
        if (lane == 0 && d) {
          if (vid != s) {
            atomicAdd((unsigned long long *)&S.target[vid], (unsigned long long)(-d));
            S.dlst.add(vid, -d);
          }
        }
      }
    }
  }
}

// phase D shortcut: when the step's dense set is exactly the giant hot (hub's)
// CCs, all covered now, the build's per-vertex hot sums are the member
// updates — one vector pass instead of a pass over the store (c2's first
// step).  Block-collective (uniform result); false: run the dense pass.
__device__ __noinline__ bool dense_hot(const uint32_t *cov_root, const uint32_t *hot_size,
                                       const uint32_t *hot_root, uint32_t big_t, uint32_t B,
                                       const int64_t *hotsum, long long *target, uint32_t nv,
                                       DeltaList dlst, uint32_t s, size_t tid, size_t nth) {
  int ok = 1;
  for (uint32_t j = threadIdx.x; j < B; j += blockDim.x) {
    const uint32_t cr = __ldcg(cov_root + j);
    const bool big = hot_size[j] > big_t;
    if (big != (cr != NONE) || (big && cr != hot_root[j])) ok = 0;
  }
  if (!__syncthreads_and(ok)) return false;
  for (size_t v = tid; v < nv; v += nth) {
    const long long h = hotsum[v];
    if (h && v != s) {
      atomicAdd((unsigned long long *)&target[v], (unsigned long long)(-h));
      dlst.add((uint32_t)v, -h);
    }
  }
  return true;
}

__device__ void load_tables(const Sel &S, uint32_t *shr, uint16_t *tab) {
  for (uint32_t i = threadIdx.x; i < S.B; i += blockDim.x) shr[i] = S.g_shr[i];
  for (uint32_t i = threadIdx.x; i <= (1u << PACIM_TB); i += blockDim.x) tab[i] = S.g_tab[i];
  __syncthreads();
}

struct SelOut {
  uint32_t k;
  uint32_t given;          // NONE: argmax over the gains; else the seed of a single
                           // multi-rank step (no argmax, target = delta vector)
  uint32_t *seeds;
  long long *gain_num;     // k, zeroed
  long long *arg_gain;     // k
};

// refresh the chunk maxima whose argmax lost gain in step parity par (all
// chunks if `all`); block-strided over chunks
__device__ void refresh_chunks(const Sel &S, uint32_t par, bool all, Best *sh) {
  const uint32_t nd = all ? S.nchunks : __ldcg(S.dcnt + par);
  for (uint32_t t = blockIdx.x; t < nd; t += gridDim.x) {
    const uint32_t c = all ? t : __ldcg(S.dlist + (size_t)par * S.nchunks + t);
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
}

// clear the visited bits and touched flags of the rows in touched list par
__device__ void clear_touched(const Sel &S, uint32_t par, size_t tid, size_t nth) {
  const uint32_t nt = __ldcg(S.tcnt + par);
  for (size_t t = tid; t < (size_t)nt * S.BW; t += nth) {
    const uint32_t r = __ldcg(S.touched + (size_t)par * S.nr + t / S.BW);
    S.vis[(size_t)r * S.BW + (t % S.BW)] = 0;
    if (t % S.BW == 0) S.tflag[r] = 0;
  }
}

// Step i (parity par): A argmax -> B MarkSeed + small CCs -> C shared
// traversal (until quiescence) -> D dense pass (big CCs) -> E refresh of the
// chunk maxima and clean-up, then ONE grid barrier.  At quiescence every
// update of B and C is complete (release/acquire on the producer and done
// counters), so E needs no barrier of its own; counters of parity par ^ 1
// (read during step i - 1) are re-armed in E of step i.
__global__ void __launch_bounds__(SEL_THREADS, 1) k_select(Sel S0, SelOut O, uint32_t par0) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint32_t dsm[];
  Sel S = S0;
  uint32_t *shr = dsm;
  uint16_t *tab = reinterpret_cast<uint16_t *>(dsm + S.B);
  // per-warp queue / visited set / tail of warp_bfs and the popped row's mask
  uint32_t *wbase = dsm + (table_words(S.B)) + (size_t)(threadIdx.x >> 5) * WARP_WORDS;
  uint32_t *wq = wbase, *whs = wbase + QCAP, *wtail = wbase + QCAP + HCAP;
  uint32_t *wm = wbase + QCAP + HCAP + 1;
  uint8_t *wl = reinterpret_cast<uint8_t *>(wm + MAX_BW);
  LStack lst;
  lst.row = wm + MAX_BW + MAX_BW / 4;
  lst.x = lst.row + LCAP;
  lst.cnt = lst.x + LCAP;
  lst.keep = S.lkeep;
  lst.trow = lst.cnt + 1;
  lst.tn = lst.trow + 32;
  if ((threadIdx.x & 31) == 0) *lst.tn = 0;
  __syncwarp();
  uint32_t *sdl = dsm + table_words(S.B) + SEL_WARPS * WARP_WORDS;  // block's copy of dl[B]
  __shared__ Best sh[33];
  load_tables(S, shr, tab);
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  const size_t gwarp = tid >> 5, nwarps = nth >> 5;
  const int lane = threadIdx.x & 31;
  // ---- prologue: every chunk maximum; arm the first step
  if (S.track) refresh_chunks(S, 0, true, sh);
  if (tid == 0) {
    S.qc[QC_PROD + 16 * (par0 & 1)] = nwarps;  // every warp produces in B
    S.dcnt[par0 & 1] = 0;
    S.tcnt[par0 & 1] = 0;
    S.dense[par0 & 1] = 0;
  }
  grid.sync();
  unsigned long long tstart = ld_acq(S.qc + QC_TAIL);  // stable: no traversal running
  for (uint32_t step = 0; step < O.k; step++) {
    if (__ldcg(S.diag + DG_ABORT)) break;  // uniform: read after a barrier
    S.par = (par0 + step) & 1;
    S.tlstep = step;
    const uint32_t nxt = S.par ^ 1;
    stamp(S, step, 0);
    // ---- A: every block reduces the chunk maxima -> s
    uint32_t s;
    long long sg = 0;
    if (O.given == NONE) {
      Best c{LLONG_MIN, 0xFFFFFFFFu};
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
    const uint32_t srow = S.cid[s];
    stamp(S, step, 1);
    if (tid == 0) {
      // reservations past the end of the previous traversal are void (every
      // consumer reserves only after all of B, including this warp's, is done)
      S.qc[QC_HEAD] = tstart;
      O.seeds[step] = s;
      O.arg_gain[step] = sg;
      if (O.given == NONE) {
        S.target[s] = -1;  // s leaves the candidate set (R6)
        mark_dirty(S, s >> S.csh);
      }
    }
    // ---- B: MarkSeed, one warp per slot; small newly covered CCs are
    //          enumerated right here by the warp (warp_bfs); the others are
    //          handed to the shared traversal through the seed row's mask
    {
      unsigned long long dsum = 0, nwarp = 0, ndef = 0;
      for (size_t j = gwarp; j < S.B; j += nwarps) {
        uint32_t d = 0;
        if (S.trav_only) {  // compressed store: MarkSeed done by the Get-center probe
          if (lane == 0 && __ldcg(S.dl + j)) {
            atomicOr(S.vis + (size_t)srow * S.BW + (j >> 5), 1u << (j & 31));
            touch(S, srow);
          }
        } else if (lane == 0) {
          d = cover_slot(S, srow, (uint32_t)j);
        }
        d = __shfl_sync(0xffffffffu, d, 0);
        __syncwarp();
        dsum += d;
        const uint32_t small = __shfl_sync(0xffffffffu, lane == 0 ? __ldcg(S.dl + j) : 0u, 0);
        if (small) {
          bool done = false;
          if (S.warp_ok && small <= S.warp_max)
            done = warp_bfs(S, s, (uint32_t)j, small, wq, whs, wtail, shr);
          if (done) {
            nwarp++;
          } else {
            ndef++;
            if (lane == 0) reach(S, srow, s, (uint32_t)j >> 5, 1u << (j & 31), nullptr);
          }
          __syncwarp();
        }
      }
      if (lane == 0) {
        if (dsum) atomicAdd((unsigned long long *)&O.gain_num[step], dsum);
        if (S.diag && (nwarp | ndef)) {
          atomicAdd(S.diag + DG_WARP, nwarp);
          atomicAdd(S.diag + DG_DEFER, ndef);
        }
        add_release(S.qc + QC_PROD + 16 * S.par, ~0ull);  // -1, after this warp's updates
      }
    }
    stamp(S, step, 2);
    // ---- C: the shared traversal, until quiescence
    const unsigned long long tend =
        queue_phase(S, s, wm, wl, shr, tab, sdl, S.qc + QC_PROD + 16 * S.par, &lst);
    stamp(S, step, 4);
    // ---- D: dense pass for big CCs (the flag is final: every B is done)
    const bool dense = __ldcg(S.dense + S.par) != 0;
    if (dense) {
      // the dense set exactly the giant hot (hub's) CCs, all covered now —
      // the build's per-vertex hot sums are the member updates (one vector
      // pass instead of a pass over the store; c2's first step)
      if (S.hotsum && dense_hot(S.cov_root, S.hot_size, S.hot_root, S.big_t, S.B, S.hotsum,
                                S.target, S.nv, S.dlst, s, tid, nth)) {
        if (tid == 0 && S.diag) atomicAdd(S.diag + DG_HOT, 1ull);
      } else {
        apply_dense(S, s, gwarp, nwarps);
      }
      if (tid == 0 && S.diag) atomicAdd(S.diag + DG_DENSE, 1ull);
      grid.sync();
    }
    stamp(S, step, 5);
    // ---- E: chunk maxima of this step, clean-up, re-arm parity nxt
    if (S.track) refresh_chunks(S, S.par, dense, sh);
    clear_touched(S, S.par, tid, nth);
    if (tid == 0) {
      S.qc[QC_PROD + 16 * nxt] = nwarps;
      S.dcnt[nxt] = 0;
      S.tcnt[nxt] = 0;
      S.dense[nxt] = 0;
      if (S.diag) atomicAdd(S.diag + DG_STEPS, 1ull);
    }
    stamp(S, step, 6);
    grid.sync();
    stamp(S, step, 7);
    tstart = tend;
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
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  // 8 independent streaming loads in flight per thread (one at a time left the
  // scan at half of HBM bandwidth: 0.17 ms for c4's 67M gains)
  for (; v + 7 * stride < n; v += 8 * stride) {
    long long g[8];
#pragma unroll
    for (int u = 0; u < 8; u++) g[u] = __ldcs(gain + v + u * stride);
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (better(g[u], (uint32_t)(v + u * stride), b.g, b.v)) {
        b.g = g[u];
        b.v = (uint32_t)(v + u * stride);
      }
  }
  for (; v < n; v += stride) {
    const long long g = __ldcs(gain + v);
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

// gain[v[i]] += d[i] (duplicates add up), then gain[s] = -1 (R6)
__global__ void k_apply_deltas(long long *gain, const uint32_t *v, const long long *d,
                               unsigned long long count) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    if (d[i]) atomicAdd((unsigned long long *)&gain[v[i]], (unsigned long long)d[i]);
}
__global__ void k_apply_dense(long long *gain, long long *delta, uint32_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const long long x = delta[i];
    if (x) {
      gain[i] += x;
      delta[i] = 0;
    }
  }
}
__global__ void k_clear_deltas(long long *delta, const uint32_t *v, unsigned long long count) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    delta[v[i]] = 0;
}
__global__ void k_set_gain(long long *gain, uint32_t s, long long x) { gain[s] = x; }

// ---------------------------------------------------------- NEXT f2
// Lazy (CELF-style) selection (prefix doubling P:2381-2401):
// fresh marginal gain of candidate cand[t] at the current S, one warp per
// candidate: sum over the slots of |C_j(v)| unless C_j(v) is covered (R17).
__global__ void k_lazy_eval(Sel S, const uint32_t *cand, uint32_t b0, uint32_t b1,
                            long long *delta) {
  const int lane = threadIdx.x & 31;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t t = b0 + warp; t < b1; t += nw) {
    const uint32_t v = cand[t];
    if (__ldcg(delta + v) < 0) continue;  // a seed (-1, R6): never a candidate again
    const uint32_t row = S.cid[v];
    long long g = 0;
    if (row == NONE) {
      g = S.B;  // isolated: a singleton in every sketch
    } else {
      for (uint32_t j = lane; j < S.B; j += 32) {
        const uint32_t sv = ep_rd(__ldcg(S.L + pc_addr(S.smap, S.nr, row, j)), S.ep);
        uint32_t rv;
        if (sv == (PACIM_HIGH | 1u)) {
          g += 1;  // {v}: never covered while v is not a seed
          continue;
        }
        rv = (sv & PACIM_HIGH) ? sv : ep_rd(__ldcg(S.L + pc_addr(S.smap, S.nr, sv, j)), S.ep);
        if (!(rv & COV)) g += rv & SIZE;
      }
      for (int d = 16; d; d >>= 1) g += __shfl_xor_sync(0xffffffffu, g, d);
    }
    if (lane == 0) delta[v] = g;
  }
}

// MarkSeed(s) for every slot (no member updates in the lazy selector)
__global__ void k_lazy_mark(Sel S, uint32_t s) {
  const uint32_t srow = S.cid[s];
  if (srow == NONE) return;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < S.B; j += gridDim.x * blockDim.x) {
    const uint32_t sl =
        ep_rd(S.L[S.onew ? (size_t)srow * S.B + j : pc_addr(S.smap, S.nr, srow, j)], S.ep);
    if (sl == (PACIM_HIGH | 1u)) continue;  // singleton
    const uint32_t root = (sl & PACIM_HIGH) ? srow : sl;
    const size_t ra = S.onew ? (size_t)root * S.B + j : pc_addr(S.smap, S.nr, root, j);
    const uint32_t x = atomicOr(S.L + ra, COV);
    if (!(x & COV)) {
      const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
      if (at < S.cov_cap) S.cov_list[at] = ra;
    }
  }
}

// sort keys of the candidate order (stale gain desc, id asc via a stable
// sort of ids in ascending order); seeds (gain -1) last
__global__ void k_lazy_keys(const long long *delta, uint32_t n, uint64_t *key, uint32_t *id) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    const long long d = delta[v];
    key[v] = d < 0 ? ~0ull : (~0ull >> 1) - (uint64_t)d;
    id[v] = (uint32_t)v;
  }
}

// best (fresh gain desc, id asc) of cand[0, b) -> out (block reduction + atomics-free
// two-level: one block per 4096 candidates, then the host combines)
__global__ void __launch_bounds__(SEL_THREADS) k_lazy_best(const long long *delta,
                                                           const uint32_t *cand, uint32_t b,
                                                           Best *part) {
  __shared__ Best sh[33];
  Best x{LLONG_MIN, 0xFFFFFFFFu};
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < b; t += gridDim.x * blockDim.x) {
    const uint32_t v = cand[t];
    const long long g = delta[v];
    if (better(g, v, x.g, x.v)) {
      x.g = g;
      x.v = v;
    }
  }
  x = block_best(x, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = x;
}

// Win-Tree selector (NEXT f2) on the dense store: the same
// level-synchronous FindMax in one block as store_cs.cu's k_cs_wintree, with
// the fresh marginal gain read from the vertex-major store (k_lazy_eval's
// rule) and MarkSeed by the covered bit of the root slots.
constexpr int WT_THREADS = 1024;

__device__ __forceinline__ uint32_t wt_win(const long long *key, uint32_t a, uint32_t b) {
  if (a == NONE) return b;
  if (b == NONE) return a;
  const long long ka = key[a], kb = key[b];
  return (ka > kb || (ka == kb && a < b)) ? a : b;
}

__device__ long long dense_eval(const Sel &S, uint32_t v) {
  const int lane = threadIdx.x & 31;
  const uint32_t row = S.cid[v];
  if (row == NONE) return S.B;  // isolated: a singleton in every sketch
  long long g = 0;
  for (uint32_t j = lane; j < S.B; j += 32) {
    const uint32_t sv = ep_rd(__ldcg(S.L + pc_addr(S.smap, S.nr, row, j)), S.ep);
    if (sv == (PACIM_HIGH | 1u)) {
      g += 1;  // {v}: never covered while v is not a seed
      continue;
    }
    const uint32_t rv =
        (sv & PACIM_HIGH) ? sv : ep_rd(__ldcg(S.L + pc_addr(S.smap, S.nr, sv, j)), S.ep);
    if (!(rv & COV)) g += rv & SIZE;
  }
  for (int d = 16; d; d >>= 1) g += __shfl_xor_sync(0xffffffffu, g, d);
  return g;
}

struct WTd {
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
__global__ void __launch_bounds__(WT_THREADS, 1) k_wintree_dense(Sel S, WTd W, uint32_t k) {
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
        const long long g = dense_eval(S, v);
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
    const uint32_t srow = S.cid[s];
    if (srow != NONE)
      for (uint32_t j = threadIdx.x; j < S.B; j += blockDim.x) {
        const uint32_t sl = ep_rd(S.L[pc_addr(S.smap, S.nr, srow, j)], S.ep);
        if (sl == (PACIM_HIGH | 1u)) continue;
        const uint32_t root = (sl & PACIM_HIGH) ? srow : sl;
        const size_t ra = pc_addr(S.smap, S.nr, root, j);
        if (!(atomicOr(S.L + ra, COV) & COV)) {
          const unsigned long long at = atomicAdd(S.cov_cnt, 1ull);
          if (at < S.cov_cap) S.cov_list[at] = ra;
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

__global__ void k_wtd_leaves(uint32_t *T, uint32_t N, uint32_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    T[N + i] = i < n ? (uint32_t)i : NONE;
}

__global__ void k_wtd_level(uint32_t *T, const long long *key, uint32_t lo, uint32_t hi) {
  for (size_t t = lo + (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < hi;
       t += (size_t)gridDim.x * blockDim.x)
    T[t] = wt_win(key, T[2 * t], T[2 * t + 1]);
}

// empty ring: slot i expects ticket i
__global__ void k_ring_init(Item *ring, unsigned long long Q) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < Q;
       i += (size_t)gridDim.x * blockDim.x)
    ring[i] = Item{(uint32_t)i, NONE, 0, 0};
}

}  // namespace

// ------------------------------------------------------------------ host
static uint64_t env_u64(const char *name, uint64_t dflt) {
  const char *e = getenv(name);
  return e ? (uint64_t)std::max(1LL, atoll(e)) : dflt;
}

// Device state shared by the single-rank selection and the multi-rank steps.
// work-queue ring items for rows: a power of two >= 2 (rows + 2^18), at most 2^28
static uint64_t ring_items(uint32_t nr) {
  uint64_t qcap = 1024;
  while (qcap < 2ull * ((uint64_t)nr + (1ull << 18)) && qcap < (1ull << 28)) qcap <<= 1;
  return qcap;
}

// device bytes of the selection's traversal state (make_sel's layout)
size_t pc_select_state_bytes(uint32_t nr, uint32_t B) {
  const size_t BW = (B + 31) / 32;
  return 4 * (2 * (size_t)QC_WORDS + 2 * DG_WORDS + 4 + 2 * (size_t)nr * BW + 4 * (size_t)nr +
              4 * ring_items(nr) + 4);
}

static Sel make_sel(pacim_ctx *ctx, long long *target) {
  const uint32_t B = ctx->R_local, n = ctx->n, nr = ctx->nr;
  PC_REQUIRE((B + 31) / 32 <= MAX_BW, PACIM_ENOTIMPL,
             "selection supports at most 1024 local sketches per context");
  Sel S;
  S.off = ctx->off.as<uint64_t>();
  S.nbr = ctx->nbr.as<uint32_t>();
  S.K = ctx->K;
  S.t32 = ctx->t32;
  S.tcsr = ctx->tcsr.as<uint32_t>();  // valid after pc_ensure_tcsr (the traversals' callers)
  S.wic = ctx->pmodel != PACIM_P_CONST;  // per-edge thresholds in tcsr
  S.toff = ctx->toff();
  S.g_shr = ctx->d_shr.as<uint32_t>();
  S.hr64 = ctx->d_hr64.as<uint64_t>();
  S.decor = ctx->hash_rule;
  S.g_tab = ctx->d_tab.as<uint16_t>();
  S.L = ctx->L.as<uint32_t>();
  S.ep = ctx->ep;
  S.smap = ctx->d_smap.as<uint32_t>();
  S.onew = ctx->win_first.size() <= 2;
  S.nr = nr;
  S.B = B;
  S.BW = (B + 31) / 32;
  S.nv = n;
  S.cid = ctx->cid.as<uint32_t>();
  S.rmap = ctx->rmap.as<uint32_t>();
  S.target = target;
  // dense pass only for CCs whose traversal would cost more than streaming
  // the store (tests force it down with PACIM_BIG_T)
  S.big_t = (uint32_t)env_u64("PACIM_BIG_T", std::max<uint64_t>(65536, nr / 8));
  S.warp_ok = getenv("PACIM_NO_WARP_BFS") == nullptr;
  S.warp_max = (uint32_t)std::min<uint64_t>(
      QCAP, getenv("PACIM_WARP_MAX") ? atoll(getenv("PACIM_WARP_MAX")) : QCAP);
  // the hot sums of this build, if kept for this dense threshold (one window)
  S.hotsum = (ctx->hot_any && ctx->hot_big_t == S.big_t && S.onew) ? ctx->hotsum.as<int64_t>()
                                                                   : nullptr;
  S.hot_root = ctx->d_hot.as<uint32_t>();
  S.hot_size = ctx->d_hot_size.as<uint32_t>();
  S.ch = (uint32_t)env_u64("PACIM_CHUNK", CH_DEFAULT);
  S.lkeep = (uint32_t)std::min<uint64_t>(16, getenv("PACIM_LKEEP") ? atoll(getenv("PACIM_LKEEP")) : 2);
  S.hidx = ctx->hidx.as<uint32_t>();
  S.hla_off = ctx->hla_ok ? ctx->hla_off.as<unsigned long long>() : nullptr;
  S.hla_row = ctx->hla_row.as<uint32_t>();
  S.max_sleep = (uint32_t)env_u64("PACIM_MAX_SLEEP", 4096);
  // argmax cache geometry: <= MAX_CHUNKS chunks of 2^csh vertices
  uint32_t csh = 10;
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
  // argmax cache: cmax[nchunks], cdirty[nchunks], dlist[2][nchunks], dcnt[2]
  pc_ensure(ctx, ctx->sel_partial, (size_t)S.nchunks * (sizeof(Best) + 12) + 64);
  S.cmax = ctx->sel_partial.as<Best>();
  S.cdirty = reinterpret_cast<uint32_t *>(S.cmax + S.nchunks);
  S.dlist = S.cdirty + S.nchunks;
  S.dcnt = S.dlist + 2 * (size_t)S.nchunks;
  // traversal state (words): qc[QC_WORDS] u64, diag[DG_WORDS] u64, tcnt[4],
  // vis, pend (rows x BW each), inq, tflag, touched[2] (rows each), ring (Q
  // items of 4 words).  Outstanding row items <= rows (one per row at a
  // time); chunk items are queued only while fewer than Q/2 items are
  // outstanding, so Q >= 2 (rows + 2^18) never blocks a producer for good.
  // capped at 2^28 items (4 GB): outstanding rows are the rows reached but
  // not yet expanded, far below `rows` in practice (c5: 268M rows); a full
  // ring would stall producers until the watchdog reports it (ECHECK)
  const uint64_t qcap = ring_items(nr);
  const size_t bw = (size_t)nr * S.BW;
  const size_t head = 2 * QC_WORDS + 2 * DG_WORDS + 4;
  const size_t words = head + 2 * bw + 4 * (size_t)nr + 4 * qcap + 4;
  if (ctx->bfs.bytes < words * 4 || ctx->bfs_nr != nr || ctx->bfs_bw != S.BW) {
    // new layout: every mask, flag and counter starts at zero, the ring empty
    pc_ensure(ctx, ctx->bfs, words * 4);
    PC_CUDA(cudaMemsetAsync(ctx->bfs.p, 0, words * 4, ctx->stream));
    ctx->bfs_nr = nr;
    ctx->bfs_bw = S.BW;
    ctx->bfs_ring_reset = true;
    ctx->sel_par = 0;
  }
  uint32_t *q = ctx->bfs.as<uint32_t>();
  S.qc = reinterpret_cast<unsigned long long *>(q);
  S.diag = S.qc + QC_WORDS;
  S.tcnt = q + 2 * QC_WORDS + 2 * DG_WORDS;
  S.vis = q + head;
  S.pend = S.vis + bw;
  S.inq = S.pend + bw;
  S.tflag = S.inq + nr;
  S.touched = S.tflag + nr;
  S.ring = reinterpret_cast<Item *>(S.touched + 2 * (size_t)nr + ((4 - (head + 2 * bw) % 4) % 4));
  S.qmask = qcap - 1;
  S.qguard = qcap / 2;
  if (ctx->bfs_ring_reset) {
    k_ring_init<<<pc_grid(ctx, qcap, 256), 256, 0, ctx->stream>>>(S.ring, qcap);
    PC_CHECK_LAUNCH();
    ctx->bfs_ring_reset = false;
  }
  S.par = 0;
  S.track = 0;
  S.trav_only = 0;
  S.tl = nullptr;
  S.tlstep = 0;
  S.ilog = nullptr;
  S.ilog_cap = 0;
  S.dlst = ctx->dlist;
  return S;
}

static size_t sel_smem(uint32_t B) {
  return (size_t)table_words(B) * 4 + (size_t)SEL_WARPS * WARP_WORDS * 4 + (size_t)B * 4;
}

static unsigned sel_grid(pacim_ctx *ctx, size_t smem) {
  PC_REQUIRE(smem <= 200 * 1024, PACIM_ENOTIMPL, "too many sketch slots for k_select");
  PC_CUDA(cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  PC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_select, SEL_THREADS, smem));
  PC_REQUIRE(occ >= 1, PACIM_ECUDA, "k_select cannot be resident");
  const int bps = (int)env_u64("PACIM_SEL_BPS", 1);  // resident blocks per SM
  return (unsigned)ctx->sm_count * (unsigned)std::min(occ, bps);
}

// clear covered bits of the previous selection and the traversal bookkeeping
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
  // diagnostics.  Queue tickets keep counting (the ring's sequence numbers
  // follow them); visited bits, touched flags, pending bits and queue flags
  // are all clear after every completed step.
  PC_CUDA(cudaMemsetAsync(S.diag, 0, DG_WORDS * 8, ctx->stream));
  ctx->sel_list_valid = true;
}

void pc_select_reset(pacim_ctx *ctx) {
  if (ctx->cs) return pc_cs_select_reset(ctx);
  Sel S = make_sel(ctx, nullptr);
  uncover(ctx, S);
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

static void read_diag(pacim_ctx *ctx, const Sel &S) {
  unsigned long long d[DG_WORDS];
  PC_CUDA(cudaMemcpyAsync(d, S.diag, sizeof(d), cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->stats.select_member_updates = 0;
  ctx->stats.select_bfs_visits = d[DG_ROWS] + d[DG_CHUNKS];
  ctx->stats.select_dense_steps = d[DG_DENSE];
  ctx->stats.select_warp_slots = d[DG_WARP];
  ctx->stats.select_deferred_slots = d[DG_DEFER];
  ctx->stats.select_row_items = d[DG_ROWS];
  ctx->stats.select_chunk_items = d[DG_CHUNKS];
  ctx->stats.select_inline_rows = d[DG_INLINE];
  ctx->stats.select_edges = d[DG_EDGES];
  ctx->stats.select_hotsum_steps = d[DG_HOT];
  PC_REQUIRE(!d[DG_ABORT], PACIM_ECHECK, "select: traversal watchdog expired (internal error)");
}

void pc_select(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
               int64_t *sigma_num) {
  if (ctx->cs) return pc_cs_select(ctx, k, seeds, gain_num, sigma_num);
  pc_ensure_tcsr(ctx);  // the cover traversal reads per-entry thresholds
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
  O.given = NONE;
  O.seeds = ctx->sel_seeds.as<uint32_t>();
  O.gain_num = ctx->sel_gain.as<long long>();
  O.arg_gain = O.gain_num + k;
  const size_t smem = sel_smem(S.B);
  const unsigned grid = sel_grid(ctx, smem);
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
  uint32_t par0 = ctx->sel_par;
  TmpBuf tlb(ctx);
  const bool timeline = getenv("PACIM_TIMELINE") != nullptr;
  if (timeline) {
    pc_ensure(ctx, tlb, (size_t)k * 64);
    S.tl = tlb.as<unsigned long long>();
  }
  TmpBuf ilb(ctx);
  const char *ilog_path = getenv("PACIM_ITEMLOG");
  if (ilog_path) {
    S.ilog_cap = 4u << 20;
    pc_ensure(ctx, ilb, (S.ilog_cap * 4 + 4) * 8);
    PC_CUDA(cudaMemsetAsync(ilb.p, 0, 32, ctx->stream));
    S.ilog = ilb.as<unsigned long long>();
  }
  void *args[] = {&S, &O, &par0};
  PC_CUDA(cudaLaunchCooperativeKernel((void *)k_select, grid, SEL_THREADS, args, smem, ctx->stream));
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  if (ilog_path) {  // raw item log -> file (u64 count, then 4 x u64 per item)
    unsigned long long cnt = 0;
    PC_CUDA(cudaMemcpyAsync(&cnt, S.ilog, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    cnt = std::min(cnt, S.ilog_cap);
    std::vector<unsigned long long> h(cnt * 4 + 4);
    PC_CUDA(cudaMemcpyAsync(h.data(), S.ilog, (cnt * 4 + 4) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    h[0] = cnt;
    if (FILE *f = fopen(ilog_path, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  if (timeline) {  // mean ns per phase over the steps, on stderr
    std::vector<unsigned long long> h((size_t)k * 8);
    PC_CUDA(cudaMemcpyAsync(h.data(), S.tl, (size_t)k * 64, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    double acc[8] = {0};
    for (uint32_t i = 0; i < k; i++)
      for (int p = 1; p < 8; p++) acc[p] += (double)(h[i * 8 + p] - h[i * 8 + p - 1]);
    fprintf(stderr, "timeline us/step: A %.2f B %.2f waitB %.2f queue %.2f dense %.2f E %.2f sync %.2f\n",
            acc[1] / k / 1e3, acc[2] / k / 1e3, acc[3] / k / 1e3, acc[4] / k / 1e3, acc[5] / k / 1e3,
            acc[6] / k / 1e3, acc[7] / k / 1e3);
  }
  std::vector<long long> hg(2 * (size_t)k);
  PC_CUDA(cudaMemcpyAsync(seeds, O.seeds, (size_t)k * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(hg.data(), O.gain_num, (2 * (size_t)k) * 8, cudaMemcpyDeviceToHost,
                          ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms = ms;
  ctx->stats.kernel_launches_select = 2;
  read_diag(ctx, S);
  ctx->sel_par = (par0 + k) & 1;
  ctx->stats.select_evaluations = 0;  // the lazy selectors' counters
  ctx->stats.select_eval_rounds = 0;
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

// One multi-rank step: MarkSeed of the given seed s on this ctx's sketches and
// the member deltas (-delta per member) accumulated into d_delta.
void pc_cover_local(pacim_ctx *ctx, uint32_t s, int64_t *d_delta, int64_t *local_gain) {
  pc_ensure_tcsr(ctx);  // the cover traversal reads per-entry thresholds
  if (ctx->cs) return pc_cs_cover_local(ctx, s, d_delta, local_gain);
  PC_REQUIRE(ctx->sel_list_valid, PACIM_ESTATE, "pacim_select_reset first");
  Sel S = make_sel(ctx, reinterpret_cast<long long *>(d_delta));
  pc_ensure(ctx, ctx->sel_gain, 64);
  pc_ensure(ctx, ctx->sel_seeds, 16);
  SelOut O;
  O.k = 1;
  O.given = s;
  O.seeds = ctx->sel_seeds.as<uint32_t>();
  O.gain_num = ctx->sel_gain.as<long long>();
  O.arg_gain = O.gain_num + 1;
  PC_CUDA(cudaMemsetAsync(O.gain_num, 0, 16, ctx->stream));
  const size_t smem = sel_smem(S.B);
  const unsigned grid = sel_grid(ctx, smem);
  uint32_t par0 = ctx->sel_par;
  void *args[] = {&S, &O, &par0};
  PC_CUDA(cudaLaunchCooperativeKernel((void *)k_select, grid, SEL_THREADS, args, smem, ctx->stream));
  ctx->sel_par ^= 1;
  long long h = 0;
  unsigned long long abort_flag = 0;
  PC_CUDA(cudaMemcpyAsync(&h, O.gain_num, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaMemcpyAsync(&abort_flag, S.diag + DG_ABORT, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  PC_REQUIRE(!abort_flag, PACIM_ECHECK, "cover: traversal watchdog expired (internal error)");
  *local_gain = (int64_t)h;
}

// the argmax (gain desc, id asc) left on the device: {i64 gain at +0, u32 id at +8}
const void *pc_argmax_async(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n) {
  unsigned grid = pc_grid(ctx, n, SEL_THREADS, 4);
  DevBuf &part = ctx->argmax_part;  // persistent: no allocation per step
  pc_ensure(ctx, part, (size_t)(grid + 1) * sizeof(Best));
  k_argmax_part<<<grid, SEL_THREADS, 0, ctx->stream>>>(reinterpret_cast<const long long *>(d_gain),
                                                       n, part.as<Best>());
  PC_CHECK_LAUNCH();
  k_argmax_final<<<1, SEL_THREADS, 0, ctx->stream>>>(part.as<Best>(), grid,
                                                     part.as<Best>() + grid);
  PC_CHECK_LAUNCH();
  static_assert(sizeof(Best) == 16 && offsetof(Best, v) == 8, "Best layout");
  return part.as<Best>() + grid;
}

void pc_argmax(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n, uint32_t *s, int64_t *g) {
  const Best *d = static_cast<const Best *>(pc_argmax_async(ctx, d_gain, n));
  Best h;
  PC_CUDA(cudaMemcpyAsync(&h, d, sizeof(Best), cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  *s = h.v;
  *g = h.g;
}

void pc_apply_deltas(pacim_ctx *ctx, int64_t *d_gain, const uint32_t *v, const int64_t *d,
                     uint64_t count, uint32_t s) {
  if (count) {
    k_apply_deltas<<<pc_grid(ctx, count, 256), 256, 0, ctx->stream>>>(
        reinterpret_cast<long long *>(d_gain), v, reinterpret_cast<const long long *>(d), count);
    PC_CHECK_LAUNCH();
  }
  if (s != NONE) {
    k_set_gain<<<1, 1, 0, ctx->stream>>>(reinterpret_cast<long long *>(d_gain), s, -1);
    PC_CHECK_LAUNCH();
  }
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

void pc_apply_dense(pacim_ctx *ctx, int64_t *d_gain, int64_t *d_delta, uint32_t n, uint32_t s) {
  k_apply_dense<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(
      reinterpret_cast<long long *>(d_gain), reinterpret_cast<long long *>(d_delta), n);
  PC_CHECK_LAUNCH();
  if (s != NONE) {
    k_set_gain<<<1, 1, 0, ctx->stream>>>(reinterpret_cast<long long *>(d_gain), s, -1);
    PC_CHECK_LAUNCH();
  }
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

void pc_clear_deltas(pacim_ctx *ctx, int64_t *d_delta, const uint32_t *v, uint64_t count) {
  if (count) {
    k_clear_deltas<<<pc_grid(ctx, count, 256), 256, 0, ctx->stream>>>(
        reinterpret_cast<long long *>(d_delta), v, count);
    PC_CHECK_LAUNCH();
  }
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Store-less member traversal for the compressed store's big CCs (H10 with
// H6c): slot j's members of C_j(s) lose delta[j] (HOST, R_local entries).
void pc_traverse_slots(pacim_ctx *ctx, uint32_t s, int64_t *target, const uint32_t *delta) {
  pc_ensure_tcsr(ctx);  // the cover traversal reads per-entry thresholds
  Sel S = make_sel(ctx, reinterpret_cast<long long *>(target));
  S.trav_only = 1;
  S.warp_ok = 0;  // these CCs are larger than the probe's queue
  PC_CUDA(cudaMemcpyAsync(S.dl, delta, (size_t)S.B * 4, cudaMemcpyHostToDevice, ctx->stream));
  pc_ensure(ctx, ctx->sel_gain, 64);
  pc_ensure(ctx, ctx->sel_seeds, 16);
  SelOut O;
  O.k = 1;
  O.given = s;
  O.seeds = ctx->sel_seeds.as<uint32_t>();
  O.gain_num = ctx->sel_gain.as<long long>();
  O.arg_gain = O.gain_num + 1;
  const size_t smem = sel_smem(S.B);
  const unsigned grid = sel_grid(ctx, smem);
  uint32_t par0 = ctx->sel_par;
  void *args[] = {&S, &O, &par0};
  PC_CUDA(cudaLaunchCooperativeKernel((void *)k_select, grid, SEL_THREADS, args, smem, ctx->stream));
  ctx->sel_par ^= 1;
  unsigned long long abort_flag = 0;
  PC_CUDA(cudaMemcpyAsync(&abort_flag, S.diag + DG_ABORT, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  PC_REQUIRE(!abort_flag, PACIM_ECHECK, "compressed cover: traversal watchdog expired");
}

// NEXT f2: the lazy selector.  Per step: candidates ordered by (stale gain
// desc, id asc); fresh gains evaluated for prefixes of 1, 2, 4, ... until the
// best fresh (g*, v*) precedes the next unevaluated candidate in that order
// (stale >= fresh by submodularity, so nothing unevaluated can beat it, ties
// included) — the same sequence as GeneralGreedy (R17).  Evaluations are
// counted (the paper's metric).
void pc_select_lazy(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                    int64_t *sigma_num) {
  const uint32_t n = ctx->n;
  const bool cs = ctx->cs;
  if (k > ctx->sel_k_cap) {
    if (ctx->sel_list_valid) {
      if (cs) {
        pc_cs_select_reset(ctx);
      } else {
        Sel old = make_sel(ctx, nullptr);
        uncover(ctx, old);
      }
    }
    ctx->sel_k_cap = k;
    ctx->sel_list_valid = false;
  }
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  Sel S{};
  if (!cs) pc_ensure_tcsr(ctx);  // the cover traversal reads the lists and thresholds
  if (!cs) S = make_sel(ctx, ctx->gain.as<long long>());
  cudaEvent_t e0, e1;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  if (cs)
    pc_cs_select_reset(ctx);
  else
    uncover(ctx, S);
  long long *delta = ctx->gain.as<long long>();
  PC_CUDA(cudaMemcpyAsync(delta, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  // sort buffers: keys x2, ids x2, partial maxima
  TmpBuf sb(ctx);
  const unsigned pg = std::max<unsigned>(1, std::min<unsigned>((n + 4095) / 4096, 4096));
  const size_t off_part = ((size_t)n * 24 + 15) & ~(size_t)15;  // 16-B aligned
  pc_ensure(ctx, sb, off_part + (size_t)pg * sizeof(Best) + 64);
  uint64_t *k0 = sb.as<uint64_t>(), *k1 = k0 + n;
  uint32_t *i0 = reinterpret_cast<uint32_t *>(k1 + n), *i1 = i0 + n;
  Best *part = reinterpret_cast<Best *>(sb.as<char>() + off_part);
  size_t tmp = 0;
  {
    cub::DoubleBuffer<uint64_t> dk(k0, k1);
    cub::DoubleBuffer<uint32_t> dv(i0, i1);
    PC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, (int64_t)n, 0, 64, ctx->stream));
  }
  TmpBuf ct(ctx);
  pc_ensure(ctx, ct, tmp + 16);
  std::vector<Best> hp(pg);
  unsigned long long evals = 0, rounds = 0;
  long long run = 0;
  for (uint32_t step = 0; step < k; step++) {
    k_lazy_keys<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(delta, n, k0, i0);
    PC_CHECK_LAUNCH();
    cub::DoubleBuffer<uint64_t> dk(k0, k1);
    cub::DoubleBuffer<uint32_t> dv(i0, i1);
    PC_CUDA(cub::DeviceRadixSort::SortPairs(ct.p, tmp, dk, dv, (int64_t)n, 0, 64, ctx->stream));
    const uint32_t *cand = dv.Current();
    uint32_t done = 0, b = 1;
    Best best{LLONG_MIN, NONE};
    for (;;) {
      if (cs) {
        pc_cs_lazy_eval(ctx, cand, done, b, delta);
      } else {
        k_lazy_eval<<<pc_grid(ctx, (size_t)(b - done) * 32, 256, 8), 256, 0, ctx->stream>>>(
            S, cand, done, b, delta);
        PC_CHECK_LAUNCH();
      }
      evals += b - done;
      rounds++;
      const unsigned g = std::min<unsigned>(pg, (b + SEL_THREADS - 1) / SEL_THREADS);
      k_lazy_best<<<g, SEL_THREADS, 0, ctx->stream>>>(delta, cand, b, part);
      PC_CHECK_LAUNCH();
      uint32_t nxt = NONE;
      long long nd = LLONG_MIN;
      if (b < n) PC_CUDA(cudaMemcpyAsync(&nxt, cand + b, 4, cudaMemcpyDeviceToHost, ctx->stream));
      PC_CUDA(cudaMemcpyAsync(hp.data(), part, g * sizeof(Best), cudaMemcpyDeviceToHost, ctx->stream));
      PC_CUDA(cudaStreamSynchronize(ctx->stream));
      best = Best{LLONG_MIN, NONE};
      for (unsigned i = 0; i < g; i++)
        if (hp[i].g > best.g || (hp[i].g == best.g && hp[i].v < best.v)) best = hp[i];
      if (b >= n) break;
      PC_CUDA(cudaMemcpyAsync(&nd, delta + nxt, 8, cudaMemcpyDeviceToHost, ctx->stream));
      PC_CUDA(cudaStreamSynchronize(ctx->stream));
      if (best.g > nd || (best.g == nd && best.v < nxt)) break;  // nothing unevaluated can win
      done = b;
      b = (uint32_t)std::min<uint64_t>(2ull * b, n);
    }
    seeds[step] = best.v;
    gain_num[step] = best.g;
    run += best.g;
    sigma_num[step] = run;
    if (cs) {
      pc_cs_lazy_mark(ctx, best.v);
    } else {
      k_lazy_mark<<<(S.B + 255) / 256, 256, 0, ctx->stream>>>(S, best.v);
      PC_CHECK_LAUNCH();
    }
    const long long m1 = -1;  // s leaves the candidate set (R6)
    PC_CUDA(cudaMemcpyAsync(delta + best.v, &m1, 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms = ms;
  ctx->stats.select_evaluations = evals;
  ctx->stats.select_eval_rounds = rounds;
  ctx->stats.kernel_launches_select = (uint32_t)(k * 3 + rounds * 2);
}

// NEXT f2: the Win-Tree selector on the dense store (selector 2)
void pc_select_wintree_dense(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                             int64_t *sigma_num) {
  const uint32_t n = ctx->n;
  uint32_t N = 1, depth = 0;
  while (N < n) {
    N <<= 1;
    depth++;
  }
  if (k > ctx->sel_k_cap) {
    if (ctx->sel_list_valid) {
      Sel old = make_sel(ctx, nullptr);
      uncover(ctx, old);
    }
    ctx->sel_k_cap = k;
    ctx->sel_list_valid = false;
  }
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  Sel S = make_sel(ctx, ctx->gain.as<long long>());
  // persistent scratch (capacity reused): T[2N], H0[2N], H1[2N], Ev[N], Et[N], X[N], outputs
  DevBuf &wb = ctx->wt_buf;
  pc_ensure(ctx, wb, (size_t)9 * N * 4 + (size_t)k * 12 + 64);
  WTd W;
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
  uncover(ctx, S);
  PC_CUDA(cudaMemcpyAsync(W.key, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  k_wtd_leaves<<<pc_grid(ctx, N, 256), 256, 0, ctx->stream>>>(W.T, N, n);
  for (uint32_t lo = N >> 1; lo >= 1; lo >>= 1)
    k_wtd_level<<<pc_grid(ctx, lo, 256), 256, 0, ctx->stream>>>(W.T, W.key, lo, 2 * lo);
  PC_CHECK_LAUNCH();
  k_wintree_dense<<<1, WT_THREADS, 0, ctx->stream>>>(S, W, k);
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
  ctx->stats.select_eval_rounds = ev[1];
  ctx->stats.kernel_launches_select = depth + 2;
  long long run = 0;
  for (uint32_t i = 0; i < k; i++) {
    gain_num[i] = hg[i];
    run += hg[i];
    sigma_num[i] = run;
  }
}
