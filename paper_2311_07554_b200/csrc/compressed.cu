// compressed.cu — the paper's compressed sketches (Alg. 3; §3
// P:1104-1253): H6c (center store) and H11 (warp-cooperative Get-center).
//
// Build: the R_g sketches are processed in batches of Bb slots.  Each batch
// runs the same union-find pass as the uncompressed store into a temporary
// parent array, adds its CC sizes to gain0 (H7), and keeps only, for each
// center c_i (R9: hi32(mix64(v ^ K_c)) < A32, index = rank in vertex order),
//   label[i][j] = min{ j' : c_j' in the same CC as c_i }
//   size[i][j]  = CC size if label[i][j] = i, else 0
// Total space O((1 + alpha R) n) (Thm 3.1).
//
// Select: per greedy step and slot, GetCenter(s) is a BFS from
// the seed s over the live edges of G'_r run by one warp with a local queue
// and visited set in shared memory ("Get-center allocates a local
// queue").  The first center met gives <size[label], label>; a CC without a
// center gives <0,-1> if a seed was visited, else <n', -1>.  MarkSeed
// zeroes size[label].  The members of a newly covered CC lose
// delta from their gain (incremental update, R17): small CCs are
// enumerated by the same warp BFS; CCs larger than the queue are handled by
// re-running the sketch pass for their batch and one dense pass (the only
// place the full labels are rebuilt).
#include <algorithm>
#include <cstdlib>

#include "pacim_internal.cuh"

namespace {

// A center's CC size in the store, with bit 31 set once MarkSeed covered the
// CC in the current selection (one word per (center, slot): the paper's
// label + size pair, no separate working copy); cleared by the select reset.
constexpr uint32_t CSZ_COV = 0x80000000u;
__device__ __forceinline__ uint32_t csz_live(uint32_t x) { return (x & CSZ_COV) ? 0u : x; }

__global__ void k_csz_uncover(uint32_t *csz, size_t N) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    if (csz[i] & CSZ_COV) csz[i] &= ~CSZ_COV;
}


constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr int PROBE_WARPS = 4;     // warps per block in k_probe
constexpr uint32_t HOT_BIG_T = 65536;  // covered CCs above this go to the rebuild (or hotsum)
constexpr uint32_t QCAP = 512;     // Get-center local queue capacity
constexpr uint32_t HCAP = 1024;    // its visited hash set (power of two)

// probe outcomes
constexpr uint32_t ST_DONE = 0;       // delta known and applied (or zero)
constexpr uint32_t ST_BIG_KNOWN = 1;  // uncovered CC with a center, too big to enumerate
constexpr uint32_t ST_BIG_UNKNOWN = 2;// no center within QCAP visits: needs the dense analysis

// ------------------------------------------------------------- centers
__global__ void k_center_flag(uint32_t n, uint64_t Kc, uint64_t a32, uint64_t *flag) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x)
    flag[v] = (a32 >= (1ull << 32) || (pc_mix64((uint64_t)v ^ Kc) >> 32) < a32) ? 1 : 0;
}

__global__ void k_center_index(const uint64_t *flag, const uint64_t *pos, uint32_t n,
                               uint32_t *center_of, uint32_t *centers) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    if (flag[v]) {
      center_of[v] = (uint32_t)pos[v];
      centers[pos[v]] = (uint32_t)v;
    } else {
      center_of[v] = NONE;
    }
  }
}

// ------------------------------------------------------- batch outputs
// gain0[v] += sum over the batch's slots of (|C_j(v)| - 1) (gain0 starts at B)
// ... and hotsum[v] += the sizes of the hub's CCs of more than big_t vertices
// that contain v (hot[jj]: the hub's root row in batch slot jj; their sizes
// to hot_size[j0 + jj]): the member update of the hub's giant CCs when the
// hub itself is chosen, without a rebuild (pc_cover_compressed)
__global__ void k_gain_sizes(const uint32_t *Lb, uint32_t nr, uint32_t Bb, const uint32_t *rmap,
                             int64_t *gain0, unsigned long long *ncc_ctr, const uint32_t *hot,
                             uint32_t j0, uint32_t big_t, uint32_t *hot_size, int64_t *hotsum) {
  unsigned long long ncc = 0;  // roots of size >= 2: the non-singleton CCs
  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  if (warp == 0)
    for (uint32_t j = lane; j < Bb; j += 32)
      hot_size[j0 + j] = hot[j] < nr ? (Lb[(size_t)hot[j] * Bb + j] & PACIM_LOW) : 0u;
  for (size_t v = warp; v < nr; v += nw) {
    long long g = 0, hs = 0;
    for (uint32_t j = lane; j < Bb; j += 32) {
      uint32_t s = Lb[v * Bb + j];
      if (s == (PACIM_HIGH | 1u)) continue;  // singleton: size 1, already counted
      ncc += (s & PACIM_HIGH) != 0;
      uint32_t sz = (s & PACIM_HIGH) ? (s & PACIM_LOW) : (Lb[(size_t)s * Bb + j] & PACIM_LOW);
      g += (long long)sz - 1;
      const uint32_t root = (s & PACIM_HIGH) ? (uint32_t)v : s;
      if (root == hot[j] && sz > big_t) hs += sz;
    }
    for (int d = 16; d; d >>= 1) {
      g += __shfl_xor_sync(0xffffffffu, g, d);
      hs += __shfl_xor_sync(0xffffffffu, hs, d);
    }
    if (lane == 0 && g) gain0[rmap[v]] += g;
    if (lane == 0 && hs) hotsum[rmap[v]] += hs;
  }
  for (int d = 16; d; d >>= 1) ncc += __shfl_xor_sync(0xffffffffu, ncc, d);
  if (lane == 0 && ncc) atomicAdd(ncc_ctr, ncc);
}

// k_gain_sizes for narrow batches (Bb <= 32 S slots): S slots per lane and
// 16 / S rows per warp iteration, every row's slot words and then every
// non-root's root word in flight together, the per-row sums through shared
// memory (lane r adds row r's 32 partials).  The warp-per-row kernel kept one
// dependent pair of loads in flight per lane and spent 20 shuffles per row
// (c5: ~37-slot batches, 27 ms of gain pass per batch)
template <int S>
__global__ void __launch_bounds__(256) k_gain_sizes_n(const uint32_t *Lb, uint32_t nr, uint32_t Bb,
                                                      const uint32_t *rmap, int64_t *gain0,
                                                      unsigned long long *ncc_ctr,
                                                      const uint32_t *hot, uint32_t j0,
                                                      uint32_t big_t, uint32_t *hot_size,
                                                      int64_t *hotsum) {
  constexpr int GR = 16 / S;
  __shared__ uint32_t redg[8][GR][33], redh[8][GR][33];
  unsigned long long ncc = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  if (warp == 0)
    for (uint32_t j = lane; j < Bb; j += 32)
      hot_size[j0 + j] = hot[j] < nr ? (Lb[(size_t)hot[j] * Bb + j] & PACIM_LOW) : 0u;
  uint32_t hj[S];
#pragma unroll
  for (int i = 0; i < S; i++) hj[i] = (lane + 32 * i < Bb) ? hot[lane + 32 * i] : NONE;
  for (size_t v0 = warp * GR; v0 < nr; v0 += nw * GR) {
    uint32_t sv[GR][S], rt[GR][S];
#pragma unroll
    for (int r = 0; r < GR; r++)
#pragma unroll
      for (int i = 0; i < S; i++) {
        const uint32_t j = lane + 32 * i;
        sv[r][i] = (j < Bb && v0 + r < nr) ? Lb[(v0 + r) * Bb + j] : (PACIM_HIGH | 1u);
      }
#pragma unroll
    for (int r = 0; r < GR; r++)
#pragma unroll
      for (int i = 0; i < S; i++) {
        const uint32_t s = sv[r][i];
        rt[r][i] = (s & PACIM_HIGH) ? s : Lb[(size_t)s * Bb + lane + 32 * i];  // the root's word
      }
#pragma unroll
    for (int r = 0; r < GR; r++) {
      uint32_t g = 0, h = 0;  // < 2^32: at most two sizes below 2^31 (S <= 2)
#pragma unroll
      for (int i = 0; i < S; i++) {
        const uint32_t s = sv[r][i];
        if (s == (PACIM_HIGH | 1u)) continue;  // singleton: size 1, already counted
        ncc += (s & PACIM_HIGH) != 0;
        const uint32_t sz = rt[r][i] & PACIM_LOW;
        g += sz - 1;
        const uint32_t root = (s & PACIM_HIGH) ? (uint32_t)(v0 + r) : s;
        if (root == hj[i] && sz > big_t) h += sz;
      }
      redg[wid][r][lane] = g;
      redh[wid][r][lane] = h;
    }
    __syncwarp();
    if (lane < GR && v0 + lane < nr) {
      long long g = 0, h = 0;
#pragma unroll 8
      for (int l = 0; l < 32; l++) {
        g += redg[wid][lane][l];
        h += redh[wid][lane][l];
      }
      if (g) gain0[rmap[v0 + lane]] += g;
      if (h) hotsum[rmap[v0 + lane]] += h;
    }
    __syncwarp();
  }
  for (int d = 16; d; d >>= 1) ncc += __shfl_xor_sync(0xffffffffu, ncc, d);
  if (lane == 0 && ncc) atomicAdd(ncc_ctr, ncc);
}

// center i, batch slot jj: its CC's root row (NONE: singleton) and CC size
__global__ void k_center_a(const uint32_t *Lb, uint32_t Bb, uint32_t rho, const uint32_t *centers,
                           const uint32_t *cid, uint32_t *croot, uint32_t *csz, uint32_t B,
                           uint32_t j0) {
  const size_t tot = (size_t)rho * Bb;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (size_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(t / Bb), jj = (uint32_t)(t % Bb);
    const uint32_t r = cid[centers[i]];
    uint32_t root = NONE, size = 1;
    if (r != NONE) {
      const uint32_t s = Lb[(size_t)r * Bb + jj];
      if (s == (PACIM_HIGH | 1u)) {
        // a singleton: no root (label = the center's own index)
      } else if (s & PACIM_HIGH) {
        root = r;
        size = s & PACIM_LOW;
      } else {
        root = s;
        size = Lb[(size_t)s * Bb + jj] & PACIM_LOW;
      }
    }
    croot[t] = root;
    csz[(size_t)i * B + j0 + jj] = size;
  }
}

// the root slot (HIGH|size > any center index) takes the minimum center index
__global__ void k_center_b(uint32_t *Lb, uint32_t Bb, uint32_t rho, const uint32_t *croot) {
  const size_t tot = (size_t)rho * Bb;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (size_t)gridDim.x * blockDim.x) {
    const uint32_t root = croot[t];
    if (root != NONE) atomicMin(Lb + (size_t)root * Bb + (t % Bb), (uint32_t)(t / Bb));
  }
}

__global__ void k_center_c(const uint32_t *Lb, uint32_t Bb, uint32_t rho, const uint32_t *croot,
                           uint32_t *clabel, uint32_t *csz, uint32_t B, uint32_t j0) {
  const size_t tot = (size_t)rho * Bb;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (size_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(t / Bb), jj = (uint32_t)(t % Bb);
    const uint32_t root = croot[t];
    const uint32_t label = root == NONE ? i : Lb[(size_t)root * Bb + jj];
    clabel[(size_t)i * B + j0 + jj] = label;
    if (label != i) csz[(size_t)i * B + j0 + jj] = 0;  // size kept at the label only
  }
}

__global__ void k_fill_i64c(int64_t *a, uint32_t n, int64_t x) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x)
    a[v] = x;
}

// --------------------------------------------------------- Get-center
struct ProbeParams {
  const uint64_t *off;
  const uint32_t *nbr;
  uint64_t K, t32;
  const uint32_t *tcsr;     // per-edge models (WIC R4, Uniform R19): T32 - toff per CSR entry
  uint32_t toff;
  int decor;                // R20: live <=> hi32(mix64(hash(r) ^ hash(e))) < T32
  // live hub adjacency (hla_off != nullptr): a hub's live neighbours in slot j
  // are the rows hla_row[hla_off[h * B + j] .. hla_off[h * B + j + 1])
  const uint32_t *cid, *hidx, *rmap;
  const unsigned long long *hla_off;
  const uint32_t *hla_row;
  uint64_t hub_deg;         // rows of degree > hub_deg are hubs
  const uint64_t *hr64;     // hash(r) per slot
  const uint32_t *shr;      // hi32(hash(r)) per slot
  uint32_t B;
  const uint32_t *center_of;
  const uint32_t *clabel;   // [rho][B]
  uint32_t *csw;            // [rho][B] sizes; bit 31 = covered in this selection
  const uint8_t *is_seed;
  long long *target;        // gain (or delta) vector, n entries
  DeltaList dlst;           // multi-rank sparse deltas (v == nullptr: off)
  uint32_t *st;             // per slot: outcome
  uint32_t *lab;            // per slot: label (BIG_KNOWN)
  uint32_t *dl;             // per slot: delta
  unsigned long long *sum;  // [0] sum of DONE deltas, [1] number of BIG slots, [2] visits
  const uint16_t *tab;      // candidate bucket table of the sorted slots
  const uint32_t *slive;    // [B][QCAP] live neighbours of the seed per slot (pre-expansion)
  const uint32_t *scnt;     // [B] their number (> QCAP - 1: overflow, expand s in the probe)
};

__device__ __forceinline__ uint64_t thr_of(const ProbeParams &P, uint64_t e) {
  return P.tcsr ? (uint64_t)P.tcsr[e] + P.toff : P.t32;
}

// edge (x, w) at CSR entry e live in the slot of hash hr (hrj: R20)
__device__ __forceinline__ bool live_edge(const ProbeParams &P, uint32_t x, uint32_t w,
                                          uint64_t e, uint32_t hr, uint64_t hrj) {
  const uint64_t a = x < w ? x : w, b = x < w ? w : x;
  const uint64_t he64 = pc_mix64(((a << 32) | b) ^ P.K);
  const uint32_t he = (uint32_t)(he64 >> 32);
  const uint64_t T = thr_of(P, e);
  if (P.decor) return T >= (1ull << 32) || (pc_mix64(hrj ^ he64) >> 32) < T;  // R20
  return (uint64_t)(hr ^ he) < T;  // R3
}

// The seed's live neighbours for every slot, its adjacency read and each
// edge hashed once by the whole grid (a hub seed would otherwise be scanned
// by every slot's probe warp).  Candidate slots from the bucket table (R2),
// live test R3 / R4.
__global__ void k_seed_live(ProbeParams P, uint32_t s, const uint32_t *s_dev, uint32_t *slive,
                            uint32_t *scnt) {
  if (s_dev) s = *s_dev;  // the argmax on the device
  const uint64_t e0 = P.off[s], e1 = P.off[s + 1];
  for (uint64_t e = e0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w = P.nbr[e];
    const uint64_t a = s < w ? s : w, b = s < w ? w : s;
    const uint64_t he64 = pc_mix64(((a << 32) | b) ^ P.K);
    const uint32_t he = (uint32_t)(he64 >> 32);
    const uint64_t T = thr_of(P, e);
    if (T == 0) continue;
    const uint32_t wb = __clz((uint32_t)(T - 1));
    uint32_t lo, hi;
    if (P.decor) {  // R20: every slot is a candidate
      lo = 0;
      hi = P.B;
    } else if (wb >= PACIM_TB) {
      const uint32_t p = he >> (32 - PACIM_TB);
      lo = P.tab[p];
      hi = P.tab[p + 1];
    } else if (wb == 0) {
      lo = 0;
      hi = P.B;
    } else {
      const uint32_t p = (he >> (32 - wb)) << (PACIM_TB - wb);
      lo = P.tab[p];
      hi = P.tab[p + (1u << (PACIM_TB - wb))];
    }
    for (uint32_t j = lo; j < hi; j++) {
      if (P.decor ? (T < (1ull << 32) && (pc_mix64(P.hr64[j] ^ he64) >> 32) >= T)
                  : (uint64_t)(P.shr[j] ^ he) >= T)
        continue;
      const uint32_t at = atomicAdd(scnt + j, 1u);
      if (at < QCAP - 1) slive[(size_t)j * QCAP + at] = w;
    }
  }
}

// one warp per slot: BFS from s with a shared-memory queue and visited set
__global__ void __launch_bounds__(PROBE_WARPS * 32) k_probe(ProbeParams P, uint32_t s,
                                                             const uint32_t *s_dev) {
  if (s_dev) s = *s_dev;  // the argmax on the device
  __shared__ uint32_t q[PROBE_WARPS][QCAP];
  __shared__ uint32_t hs[PROBE_WARPS][HCAP];
  __shared__ uint32_t tail[PROBE_WARPS], ovf[PROBE_WARPS], found[PROBE_WARPS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long mysum = 0, nbig = 0, visits = 0, cvis = 0, nfound = 0;
  for (uint32_t j = blockIdx.x * PROBE_WARPS + w; j < P.B; j += gridDim.x * PROBE_WARPS) {
    const uint32_t hr = P.shr[j];
    const uint64_t hrj = P.decor ? P.hr64[j] : 0;
    for (uint32_t i = lane; i < HCAP; i += 32) hs[w][i] = NONE;
    __syncwarp();
    if (lane == 0) {
      q[w][0] = s;
      hs[w][(s * 2654435761u) & (HCAP - 1)] = s;
      tail[w] = 1;
      ovf[w] = 0;
    }
    __syncwarp();
    uint32_t head = 0, label = NONE, delta = 0;
    bool seed_seen = false, enumerate = false;
    if (lane == 0) found[w] = NONE;
    {  // the start vertex itself (R12: center check first)
      const uint32_t ci = P.center_of[s];
      if (ci != NONE && lane == 0) found[w] = P.clabel[(size_t)ci * P.B + j];
    }
    __syncwarp();
    const uint32_t nsl = P.slive ? P.scnt[j] : QCAP;
    if (nsl < QCAP - 1) {
      // the seed was expanded by k_seed_live: its live neighbours are the
      // next queue entries (distinct: one CSR entry per neighbour), centers
      // among them recognised at discovery
      for (uint32_t i = lane; i < nsl; i += 32) {
        const uint32_t v = P.slive[(size_t)j * QCAP + i];
        q[w][1 + i] = v;
        uint32_t h = (v * 2654435761u) & (HCAP - 1);
        while (atomicCAS(&hs[w][h], NONE, v) != NONE) h = (h + 1) & (HCAP - 1);
        const uint32_t ci = P.center_of[v];
        if (ci != NONE) found[w] = P.clabel[(size_t)ci * P.B + j];
      }
      if (lane == 0) {
        tail[w] = 1 + nsl;
        if (P.is_seed[s]) seed_seen = true;
      }
      seed_seen = __shfl_sync(0xffffffffu, seed_seen, 0);
      head = 1;
      __syncwarp();
    }
    while (head < tail[w]) {
      // A center met anywhere in the CC gives the same <size, label> (all
      // centers of a CC share the label), so centers are recognised when
      // discovered, not only when dequeued: a hub seed finds one among its
      // live neighbours without filling the queue.
      if (!enumerate && found[w] != NONE) {
        label = found[w];
        cvis += head;  // Get-center visits until a center was met (Thm 3.1)
        nfound++;
        delta = csz_live(P.csw[(size_t)label * P.B + j]);
        if (delta == 0 || delta > QCAP) break;  // covered, or too big to enumerate here
        enumerate = true;  // uncovered CC of delta <= QCAP vertices: list its members
      }
      const uint32_t x = q[w][head++];
      if (!enumerate && P.is_seed[x]) seed_seen = true;
      // a hub's live neighbours come from the HLA segment of (hub, j) instead
      // of its whole adjacency (every entry live, no test)
      uint64_t a0 = P.off[x], a1 = P.off[x + 1];
      bool viah = false;
      if (P.hla_off && a1 - a0 > P.hub_deg) {
        const uint32_t h = P.hidx[P.cid[x]];
        if (h != NONE) {
          viah = true;
          a0 = P.hla_off[(size_t)h * P.B + j];
          a1 = P.hla_off[(size_t)h * P.B + j + 1];
        }
      }
      const uint64_t e1 = a1;
      for (uint64_t e0 = a0; e0 < e1; e0 += 32) {
        const uint64_t e = e0 + lane;
        // the set never holds more than QCAP + 31 < HCAP vertices: lanes stop
        // inserting once the queue is full, so probing always terminates
        if (e < e1 && tail[w] < QCAP) {
          const uint32_t v = viah ? P.rmap[P.hla_row[e]] : P.nbr[e];
          if (viah || live_edge(P, x, v, e, hr, hrj)) {
            uint32_t h = (v * 2654435761u) & (HCAP - 1);
            for (;;) {
              const uint32_t old = atomicCAS(&hs[w][h], NONE, v);
              if (old == NONE) {  // newly visited
                const uint32_t pos = atomicAdd(&tail[w], 1u);
                if (pos < QCAP) q[w][pos] = v; else ovf[w] = 1;
                const uint32_t ci = P.center_of[v];
                if (ci != NONE && !enumerate) found[w] = P.clabel[(size_t)ci * P.B + j];
                break;
              }
              if (old == v) break;
              h = (h + 1) & (HCAP - 1);
            }
          }
        } else if (e < e1) {
          ovf[w] = 1;  // queue full with adjacency left
        }
        __syncwarp();
        if (ovf[w] || (!enumerate && found[w] != NONE)) break;
      }
      __syncwarp();
      if (!enumerate && found[w] != NONE) {
        label = found[w];
        cvis += head;
        nfound++;
        delta = csz_live(P.csw[(size_t)label * P.B + j]);
        if (delta == 0 || delta > QCAP) break;
        // uncovered and small: restart the walk from the queue head to list
        // every member (the queue already holds the visited part of the CC;
        // the current vertex's remaining adjacency is rescanned below)
        enumerate = true;
        head--;  // re-expand x fully
        continue;
      }
      if (ovf[w]) break;
    }
    const uint32_t nvis = min(tail[w], QCAP);
    visits += head;
    uint32_t status = ST_DONE;
    if (label != NONE) {
      if (delta > QCAP) {
        status = ST_BIG_KNOWN;
      } else if (delta > 0) {
        // enumerated: q[0..delta) are exactly the CC's members
        for (uint32_t i = lane; i < nvis; i += 32) {
          const uint32_t u = q[w][i];
          if (u != s) {
            atomicAdd((unsigned long long *)&P.target[u], (unsigned long long)(-(long long)delta));
            P.dlst.add(u, -(long long)delta);
          }
        }
      }
      if (lane == 0 && delta > 0) P.csw[(size_t)label * P.B + j] |= CSZ_COV;  // MarkSeed
    } else if (ovf[w]) {
      status = ST_BIG_UNKNOWN;  // no center among the first QCAP vertices
    } else {
      // BFS exhausted the CC without a center
      delta = seed_seen ? 0 : nvis;
      if (delta)
        for (uint32_t i = lane; i < nvis; i += 32) {
          const uint32_t u = q[w][i];
          if (u != s) {
            atomicAdd((unsigned long long *)&P.target[u], (unsigned long long)(-(long long)delta));
            P.dlst.add(u, -(long long)delta);
          }
        }
    }
    if (lane == 0) {
      P.st[j] = status;
      P.lab[j] = label;
      P.dl[j] = delta;
      if (status == ST_DONE) mysum += delta; else nbig++;
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (mysum) atomicAdd(P.sum + 0, mysum);
    if (nbig) atomicAdd(P.sum + 1, nbig);
    if (visits) atomicAdd(P.sum + 2, visits);
    if (cvis) atomicAdd(P.sum + 3, cvis);
    if (nfound) atomicAdd(P.sum + 4, nfound);
  }
}

// ------------------------------------------- dense path for big components
// root row of row v in batch slot jj of the rebuilt parent array
__device__ __forceinline__ uint32_t root_of(const uint32_t *Lb, uint32_t Bb, uint32_t v,
                                            uint32_t jj) {
  const uint32_t s = Lb[(size_t)v * Bb + jj];
  return (s == v || (s & PACIM_HIGH)) ? v : s;
}

// per big slot: size of the seed's CC, any center's label in it, seed present
__global__ void k_big_analyze(const uint32_t *Lb, uint32_t nr, uint32_t Bb, uint32_t j0,
                             uint32_t B, const uint32_t *st, const uint32_t *sroot,
                             const uint32_t *rmap, const uint32_t *center_of,
                             const uint32_t *clabel, const uint8_t *is_seed,
                             unsigned long long *cnt, uint32_t *clab, uint32_t *seedf) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < (size_t)nr * Bb;
       t += (size_t)gridDim.x * blockDim.x) {
    const uint32_t v = (uint32_t)(t / Bb), jj = (uint32_t)(t % Bb);
    if (st[j0 + jj] != ST_BIG_UNKNOWN) continue;
    if (root_of(Lb, Bb, v, jj) != sroot[jj]) continue;
    atomicAdd(cnt + jj, 1ull);
    const uint32_t vid = rmap[v];
    const uint32_t ci = center_of[vid];
    if (ci != NONE) atomicMin(clab + jj, clabel[(size_t)ci * B + j0 + jj]);
    if (is_seed[vid]) seedf[jj] = 1;
  }
}

__global__ void k_big_decide(uint32_t Bb, uint32_t j0, uint32_t B, uint32_t *st, uint32_t *dl,
                             const uint32_t *lab, const unsigned long long *cnt,
                             const uint32_t *clab, const uint32_t *seedf, uint32_t *csw,
                             unsigned long long *sum) {
  for (uint32_t jj = blockIdx.x * blockDim.x + threadIdx.x; jj < Bb; jj += gridDim.x * blockDim.x) {
    const uint32_t j = j0 + jj;
    uint32_t d = 0;
    if (st[j] == ST_BIG_KNOWN) {
      d = dl[j];
      csw[(size_t)lab[j] * B + j] |= CSZ_COV;
    } else if (st[j] == ST_BIG_UNKNOWN) {
      if (clab[jj] != NONE) {
        d = csz_live(csw[(size_t)clab[jj] * B + j]);
        csw[(size_t)clab[jj] * B + j] |= CSZ_COV;
      } else {
        d = seedf[jj] ? 0 : (uint32_t)cnt[jj];
      }
    } else {
      continue;
    }
    dl[j] = d;
    atomicAdd(sum, (unsigned long long)d);
  }
}

__global__ void k_big_apply(const uint32_t *Lb, uint32_t nr, uint32_t Bb, uint32_t j0,
                            const uint32_t *st, const uint32_t *dl, const uint32_t *sroot,
                            const uint32_t *rmap, uint32_t s, long long *target,
                            DeltaList dlst) {
  // one warp per 4 rows; lanes over the batch's slots, the slots' status,
  // delta and root loaded once (Bb <= 32 per lane pass), rows in flight together
  constexpr int AR = 4;
  const int lane = threadIdx.x & 31;
  size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (uint32_t jb = 0; jb < Bb; jb += 32) {
    const uint32_t jj = jb + lane;
    const bool act = jj < Bb && st[j0 + jj] != ST_DONE && dl[j0 + jj] != 0;
    if (!__any_sync(0xffffffffu, act)) continue;
    const uint32_t d_j = act ? dl[j0 + jj] : 0, r_j = act ? sroot[jj] : NONE;
    for (size_t v0 = warp * AR; v0 < nr; v0 += nw * AR) {
      uint32_t sv[AR];
#pragma unroll
      for (int r = 0; r < AR; r++)
        sv[r] = (act && v0 + r < nr) ? __ldcs(Lb + (v0 + r) * Bb + jj) : NONE;
#pragma unroll
      for (int r = 0; r < AR; r++) {
        const uint32_t v = (uint32_t)(v0 + r);
        long long d = 0;
        if (sv[r] != NONE) {
          const uint32_t root = (sv[r] == v || (sv[r] & PACIM_HIGH)) ? v : sv[r];
          if (root == r_j) d = d_j;
        }
        if (!__any_sync(0xffffffffu, d != 0)) continue;
        for (int q = 16; q; q >>= 1) d += __shfl_xor_sync(0xffffffffu, d, q);
        if (lane == 0) {
          const uint32_t vid = rmap[v];
          if (vid != s) {
            atomicAdd((unsigned long long *)&target[vid], (unsigned long long)(-d));
            dlst.add(vid, -d);
          }
        }
      }
    }
  }
}

__global__ void k_seed_roots(const uint32_t *Lb, uint32_t Bb, uint32_t srow, uint32_t *sroot) {
  for (uint32_t jj = blockIdx.x * blockDim.x + threadIdx.x; jj < Bb; jj += gridDim.x * blockDim.x)
    sroot[jj] = root_of(Lb, Bb, srow, jj);
}

// target[v] -= hotsum[v] for v != s (the hub's giant CCs covered at once)
__global__ void k_apply_hotsum(long long *target, const int64_t *hotsum, uint32_t n, uint32_t s,
                               DeltaList dlst) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (size_t)gridDim.x * blockDim.x) {
    const long long h = hotsum[v];
    if (h && v != s) {
      atomicAdd((unsigned long long *)&target[v], (unsigned long long)(-h));
      dlst.add((uint32_t)v, -h);
    }
  }
}

__global__ void k_set_seed(long long *gain, uint8_t *is_seed, uint32_t s, int set_gain) {
  if (set_gain) gain[s] = -1;
  is_seed[s] = 1;
}

}  // namespace

// ------------------------------------------------------------------ host
static uint32_t choose_batch(pacim_ctx *ctx) {
  const uint32_t B = ctx->R_local;
  if (const char *e = getenv("PACIM_BATCH")) return std::max<uint32_t>(1, std::min<uint32_t>(B, atoi(e)));
  size_t fr = 0, tot = 0;
  pc_mem_info(ctx, &fr, &tot);
  fr += ctx->Ltmp.bytes + ctx->cwork.bytes;  // earlier batch buffers: reused or freed before growing
  // everything but what the selection will still allocate (its traversal
  // state, for CCs too big for a probe) and 2 GB of headroom; at least a third
  // (one batch of all 256 slots at c4 alpha = 1/8: build 132 -> 104 ms, one
  // edge pass instead of two)
  // the selection's traversal state is not reserved: if it is needed later,
  // the batch buffer is released first and re-created smaller on demand
  // (pc_release_batch / the rebuild in pc_cover_compressed)
  // Thm 3.1: the store is O((1 + alpha R) n) words; the batch
  // parent arrays are scratch on top of it, so their budget follows the store
  // (twice its bytes, at least 4 GB) instead of taking the free memory —
  // peak memory then tracks alpha.  PACIM_BATCH_MEM overrides (bytes).
  // headroom: 2 GB + the selection's per-vertex arrays (gain i64[n], is_seed
  // u8[n]) allocated after the build (c5 ran out by 268 MB once the lean
  // graph's upper offsets took 3 GB more)
  const size_t keep = ((size_t)2 << 30) + 9 * (size_t)ctx->n;
  const size_t avail = fr > keep ? fr - keep : fr / 2;
  const size_t store = 2 * (size_t)ctx->rho * B * 4;  // label + size per (center, slot)
  size_t budget = std::max<size_t>(2 * store, (size_t)4 << 30);
  if (const char *e = getenv("PACIM_BATCH_MEM")) budget = (size_t)std::max(1LL, atoll(e));
  budget = std::min(budget, avail);
  // per slot: a parent word per row (Ltmp) and a root word per center (cwork)
  size_t per = ((size_t)std::max<uint32_t>(ctx->nr, 1) + ctx->rho) * 4;
  size_t bb = budget / per;
  return (uint32_t)std::max<size_t>(1, std::min<size_t>(B, bb));
}

void pc_build_compressed(pacim_ctx *ctx) {
  const uint32_t n = ctx->n, nr = ctx->nr, B = ctx->R_local;
  PC_REQUIRE(B >= 1 && B <= 65535, PACIM_EINVAL, "local sketch count must be in [1, 65535]");
  pc_slot_table(ctx);
  ctx->hot_any = false;
  // the uncompressed store and its selection state of an earlier build are
  // released first (the point of the compressed mode is not to hold them)
  // and so is the HLA of an earlier build; its batch parent arrays are kept
  // for reuse (choose_batch counts them as free)
  pc_cs_free(ctx);  // a compact store of an earlier build
  // the selection's Get-center probes read the symmetric lists and the
  // per-entry thresholds: derived before the batch takes the free memory
  // (derived lazily after it, c4 at alpha = 1/2 ran out of memory)
  pc_ensure_tcsr(ctx);
  ctx->ep = Ep{};   // batch stores are reset in line (no slot epochs)
  ctx->skip_init = false;
  for (DevBuf *d : {&ctx->L, &ctx->bfs, &ctx->pkeys, &ctx->hla_off, &ctx->hla_row, &ctx->hla_raw})
    pc_free(ctx, *d);
  ctx->hla_ok = false;
  ctx->bfs_nr = 0;
  ctx->sel_list_valid = false;
  pc_ensure(ctx, ctx->counters, 64 * sizeof(uint64_t));
  unsigned long long *ctr = ctx->counters.as<unsigned long long>();
  PC_CUDA(cudaMemsetAsync(ctr, 0, 64 * sizeof(uint64_t), ctx->stream));
  cudaEvent_t e0, e1, e2;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventCreate(&e2));
  ctx->launches = 0;
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  // ---- centers (R9)
  const uint64_t Kc = pc_mix64(ctx->hash_seed ^ 0x9E3779B97F4A7C15ull);
  pc_ensure(ctx, ctx->scratch, 2 * ((size_t)n + 1) * 8);
  uint64_t *flag = ctx->scratch.as<uint64_t>(), *pos = flag + n + 1;
  k_center_flag<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(n, Kc, ctx->a32, flag);
  PC_CHECK_LAUNCH();
  PC_CUDA(cudaMemsetAsync(flag + n, 0, 8, ctx->stream));
  pc_exclusive_scan_u64(ctx, flag, pos, (size_t)n + 1);
  uint64_t rho = 0;
  PC_CUDA(cudaMemcpyAsync(&rho, pos + n, 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->rho = (uint32_t)rho;
  pc_ensure(ctx, ctx->center_of, (size_t)n * 4);
  pc_ensure(ctx, ctx->centers, std::max<size_t>(rho, 1) * 4);
  k_center_index<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(
      flag, pos, n, ctx->center_of.as<uint32_t>(), ctx->centers.as<uint32_t>());
  PC_CHECK_LAUNCH();
  const size_t cs = std::max<size_t>((size_t)rho * B, 1) * 4;
  pc_free(ctx, ctx->csz_work);  // no working copy (covered bit in csz)
  for (DevBuf *d : {&ctx->clabel, &ctx->csz})
    if (d->bytes > 2 * cs) pc_free(ctx, *d);  // an earlier, larger alpha's store
  pc_ensure(ctx, ctx->clabel, cs);
  pc_ensure(ctx, ctx->csz, cs);
  pc_ensure(ctx, ctx->gain0, (size_t)n * 8);
  k_fill_i64c<<<pc_grid(ctx, n, 256), 256, 0, ctx->stream>>>(ctx->gain0.as<int64_t>(), n,
                                                            (int64_t)B);
  PC_CHECK_LAUNCH();
  // covered CCs above cbig_t go to the batch rebuild (or the hub's hotsum);
  // PACIM_CBIG_T lowers it for tests (read once per build: select uses the same)
  ctx->cbig_t = getenv("PACIM_CBIG_T") ? (uint32_t)std::max(1LL, atoll(getenv("PACIM_CBIG_T")))
                                       : HOT_BIG_T;
  pc_ensure(ctx, ctx->hotsum, (size_t)n * 8);
  pc_ensure(ctx, ctx->d_hot_size, (size_t)B * 4);
  PC_CUDA(cudaMemsetAsync(ctx->hotsum.p, 0, (size_t)n * 8, ctx->stream));
  // live hub adjacency for the Get-center probes (a hub met by a probe is
  // expanded from its live list, not its whole adjacency), recorded when its
  // expected size is at most m / 4 entries (c4 WIC: 94M entries, the select
  // 1.5 s -> 70 ms; c2 p = 0.01: 223M entries, +10 ms build for no select
  // gain).  PACIM_HLA=1: always, PACIM_NO_HLA: never.
  Hla hla{};
  const double hla_lim = getenv("PACIM_HLA") || getenv("PACIM_FORCE_HLA") ? 1e30 : 0.25;
  const bool rec_hla = getenv("PACIM_NO_HLA") == nullptr && pc_hla_begin(ctx, &hla, hla_lim);
  if (!rec_hla) ctx->hla_ok = false;
  // ---- batches of Bb slots
  ctx->Bb = choose_batch(ctx);
  const uint32_t Bb = ctx->Bb;
  pc_ensure(ctx, ctx->Ltmp, std::max<size_t>((size_t)nr * Bb, 1) * 4);
  pc_ensure(ctx, ctx->cwork, std::max<size_t>((size_t)rho * Bb, 1) * 4 + 64);
  uint32_t *Lb = ctx->Ltmp.as<uint32_t>();
  uint32_t *croot = ctx->cwork.as<uint32_t>();
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  // per batch: start, after init / edges / compress, after the gain pass
  const uint32_t nbat = (B + Bb - 1) / Bb;
  std::vector<cudaEvent_t> bev(5 * (size_t)nbat);
  for (auto &e : bev) PC_CUDA(cudaEventCreate(&e));
  for (uint32_t j0 = 0; j0 < B; j0 += Bb) {
    const uint32_t bb = std::min(Bb, B - j0);
    cudaEvent_t *ev = bev.data() + 5 * (size_t)(j0 / Bb);
    PC_CUDA(cudaEventRecord(ev[0], ctx->stream));
    pc_sketch_pass(ctx, Lb, j0, bb, ctr, ev + 1, rec_hla ? &hla : nullptr);
    if (bb <= 64 && !(getenv("PACIM_GAIN_NARROW") && !atoi(getenv("PACIM_GAIN_NARROW")))) {
      auto kg = bb <= 32 ? k_gain_sizes_n<1> : k_gain_sizes_n<2>;
      kg<<<pc_grid(ctx, (size_t)nr * (bb <= 32 ? 2 : 4), 256, 8), 256, 0, ctx->stream>>>(
          Lb, nr, bb, ctx->rmap.as<uint32_t>(), ctx->gain0.as<int64_t>(), ctr,
          ctx->d_hot.as<uint32_t>(), j0, ctx->cbig_t, ctx->d_hot_size.as<uint32_t>(),
          ctx->hotsum.as<int64_t>());
    } else {
      k_gain_sizes<<<pc_grid(ctx, (size_t)nr * 32, 256, 16), 256, 0, ctx->stream>>>(
          Lb, nr, bb, ctx->rmap.as<uint32_t>(), ctx->gain0.as<int64_t>(), ctr,
          ctx->d_hot.as<uint32_t>(), j0, ctx->cbig_t, ctx->d_hot_size.as<uint32_t>(),
          ctx->hotsum.as<int64_t>());
    }
    PC_CHECK_LAUNCH();
    PC_CUDA(cudaEventRecord(ev[4], ctx->stream));
    const size_t tot = (size_t)rho * bb;
    if (tot) {
      k_center_a<<<pc_grid(ctx, tot, 256), 256, 0, ctx->stream>>>(
          Lb, bb, (uint32_t)rho, ctx->centers.as<uint32_t>(), ctx->cid.as<uint32_t>(), croot,
          ctx->csz.as<uint32_t>(), B, j0);
      PC_CHECK_LAUNCH();
      k_center_b<<<pc_grid(ctx, tot, 256), 256, 0, ctx->stream>>>(Lb, bb, (uint32_t)rho, croot);
      PC_CHECK_LAUNCH();
      k_center_c<<<pc_grid(ctx, tot, 256), 256, 0, ctx->stream>>>(
          Lb, bb, (uint32_t)rho, croot, ctx->clabel.as<uint32_t>(), ctx->csz.as<uint32_t>(), B,
          j0);
      PC_CHECK_LAUNCH();
      ctx->launches += 3;
    }
    ctx->launches += 1;
  }
  if (rec_hla) pc_hla_finish(ctx, &hla);
  ctx->hot_size.resize(B);
  PC_CUDA(cudaMemcpyAsync(ctx->hot_size.data(), ctx->d_hot_size.p, (size_t)B * 4,
                          cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaEventRecord(e2, ctx->stream));
  unsigned long long h[6];
  PC_CUDA(cudaMemcpyAsync(h, ctr, 6 * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms_all = 0, ms_pre = 0;
  cudaEventElapsedTime(&ms_all, e0, e2);
  cudaEventElapsedTime(&ms_pre, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  ctx->ncomp = h[0];
  ctx->nnonsingle = h[0] + h[1];
  ctx->nmember = 0;
  ctx->stats.live_pairs = h[4];
  ctx->stats.t_build_ms = ms_all;
  ctx->stats.t_centers_ms = ms_pre;
  // kernel times summed over the batches (bench: per-kernel roofline)
  double ti = 0, te = 0, tc = 0, tg = 0;
  for (uint32_t bi = 0; bi < nbat; bi++) {
    cudaEvent_t *ev = bev.data() + 5 * (size_t)bi;
    float a = 0, b2 = 0, c = 0, d = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b2, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    cudaEventElapsedTime(&d, ev[3], ev[4]);
    ti += a;
    te += b2;
    tc += c;
    tg += d;
  }
  for (auto &e : bev) cudaEventDestroy(e);
  ctx->stats.t_init_ms = ti;
  ctx->stats.t_edges_ms = te;
  ctx->stats.t_compress_ms = tc;
  ctx->stats.t_compact_ms = 0;
  ctx->stats.t_gain_ms = tg;
  ctx->stats.kernel_launches_build = ctx->launches;
}

void pc_select_reset_compressed(pacim_ctx *ctx) {
  const size_t cw = (size_t)ctx->rho * ctx->R_local;
  if (cw)
    k_csz_uncover<<<pc_grid(ctx, cw, 256), 256, 0, ctx->stream>>>(ctx->csz.as<uint32_t>(), cw);
  PC_CHECK_LAUNCH();
  pc_ensure(ctx, ctx->is_seed, ctx->n);
  PC_CUDA(cudaMemsetAsync(ctx->is_seed.p, 0, ctx->n, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
}

// MarkSeed(s) on this ctx's compressed sketches; member gains in target
// decrease by delta_r.  Returns sum_r delta_r.  Marks s as a seed.
void pc_cover_compressed(pacim_ctx *ctx, uint32_t s, int64_t *target, int64_t *local_gain,
                         const void *dsel, uint32_t *s_out, int64_t *g_out) {
  const uint32_t *s_dev =
      dsel ? reinterpret_cast<const uint32_t *>(static_cast<const char *>(dsel) + 8) : nullptr;
  const uint32_t B = ctx->R_local, nr = ctx->nr;
  if (getenv("PACIM_FORCE_RELEASE")) {  // tests: every rebuild re-creates the batch buffer
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    pc_free(ctx, ctx->Ltmp);
    pc_free(ctx, ctx->cwork);
  }
  pc_ensure(ctx, ctx->cprobe, (size_t)B * 16 + 64);
  uint32_t *st = ctx->cprobe.as<uint32_t>(), *lab = st + B, *dl = lab + B;
  unsigned long long *sum = reinterpret_cast<unsigned long long *>(dl + B + (B & 1));
  PC_CUDA(cudaMemsetAsync(sum, 0, 5 * 8, ctx->stream));
  ProbeParams P;
  pc_ensure_tcsr(ctx);  // (and the symmetric lists of an upper-loaded graph)
  P.off = ctx->off.as<uint64_t>();
  P.nbr = ctx->nbr.as<uint32_t>();
  P.K = ctx->K;
  P.t32 = ctx->t32;
  pc_ensure_tcsr(ctx);
  P.tcsr = ctx->pmodel != PACIM_P_CONST ? ctx->tcsr.as<uint32_t>() : nullptr;
  P.toff = ctx->toff();
  P.decor = ctx->hash_rule;
  P.cid = ctx->cid.as<uint32_t>();
  P.hidx = ctx->hidx.as<uint32_t>();
  P.rmap = ctx->rmap.as<uint32_t>();
  P.hla_off = ctx->hla_ok ? ctx->hla_off.as<unsigned long long>() : nullptr;
  P.hla_row = ctx->hla_ok ? ctx->hla_row.as<uint32_t>() : nullptr;
  P.hub_deg = ctx->hub_deg;
  P.hr64 = ctx->d_hr64.as<uint64_t>();
  P.shr = ctx->d_shr.as<uint32_t>();
  P.B = B;
  P.center_of = ctx->center_of.as<uint32_t>();
  P.clabel = ctx->clabel.as<uint32_t>();
  P.csw = ctx->csz.as<uint32_t>();
  P.is_seed = ctx->is_seed.as<uint8_t>();
  P.target = reinterpret_cast<long long *>(target);
  P.dlst = ctx->dlist;
  P.tab = ctx->d_tab.as<uint16_t>();
  {  // seed pre-expansion (one grid pass over its adjacency for all slots)
    pc_ensure(ctx, ctx->cseed, ((size_t)B * QCAP + B) * 4);
    uint32_t *slive = ctx->cseed.as<uint32_t>(), *scnt = slive + (size_t)B * QCAP;
    PC_CUDA(cudaMemsetAsync(scnt, 0, (size_t)B * 4, ctx->stream));
    P.slive = nullptr;
    P.scnt = nullptr;
    k_seed_live<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(P, s, s_dev, slive, scnt);
    PC_CHECK_LAUNCH();
    P.slive = slive;
    P.scnt = scnt;
    ctx->launches++;
  }
  P.st = st;
  P.lab = lab;
  P.dl = dl;
  P.sum = sum;
  k_probe<<<std::min<unsigned>((B + PROBE_WARPS - 1) / PROBE_WARPS, ctx->sm_count * 8),
            PROBE_WARPS * 32, 0, ctx->stream>>>(P, s, s_dev);
  PC_CHECK_LAUNCH();
  ctx->launches++;
  unsigned long long hs[5];
  PC_CUDA(cudaMemcpyAsync(hs, sum, 40, cudaMemcpyDeviceToHost, ctx->stream));
  struct {
    long long g;
    uint32_t v, pad;
  } hb{0, 0, 0};
  if (dsel) PC_CUDA(cudaMemcpyAsync(&hb, dsel, 16, cudaMemcpyDeviceToHost, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (dsel) {  // the seed and its gain, with the probe's sums in one read-back
    s = hb.v;
    if (s_out) *s_out = hb.v;
    if (g_out) *g_out = hb.g;
  }
  ctx->stats.select_bfs_visits += hs[2];
  ctx->stats.select_center_visits += hs[3];
  ctx->stats.select_center_found += hs[4];
  unsigned long long total = hs[0], known = 0;
  if (hs[1]) {
    std::vector<uint32_t> hst(B), hdl(B);
    PC_CUDA(cudaMemcpyAsync(hst.data(), st, (size_t)B * 4, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaMemcpyAsync(hdl.data(), dl, (size_t)B * 4, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    // big CCs with a center (MarkSeed done by the probe, delta = its size):
    // members enumerated by the store-less cover traversal of select.cu
    bool unknown = false;
    std::vector<uint32_t> tdl(B, 0);
    // giant CCs stay with the batch rebuild + dense pass (a queue traversal of
    // a giant is slower)
    // measured: a queue traversal of c5's giant CCs took 3.4 s, the batch
    // rebuild + dense pass a few hundred ms
    const uint64_t big_t = ctx->cbig_t;
    bool changed = false;
    if (s == ctx->hub && ctx->hot_size.size() == B) {
      // the hub chosen while its giant CCs (> big_t) are all still uncovered:
      // their member updates are the build's hotsum, no rebuild
      bool ok = true, any = false;
      for (uint32_t j = 0; j < B && ok; j++)
        if (ctx->hot_size[j] > big_t) {
          any = true;
          ok = hst[j] == ST_BIG_KNOWN && hdl[j] == ctx->hot_size[j];
        } else if (hst[j] == ST_BIG_KNOWN && hdl[j] > big_t) {
          ok = false;  // (cannot happen: the hub's CC is the hot CC)
        }
      if (ok && any) {
        k_apply_hotsum<<<pc_grid(ctx, ctx->n, 256), 256, 0, ctx->stream>>>(
            reinterpret_cast<long long *>(target), ctx->hotsum.as<int64_t>(), ctx->n, s,
            ctx->dlist);
        PC_CHECK_LAUNCH();
        ctx->launches++;
        for (uint32_t j = 0; j < B; j++)
          if (ctx->hot_size[j] > big_t) {
            known += hdl[j];
            hst[j] = ST_DONE;
          }
        changed = true;
        ctx->stats.select_hotsum_steps++;
      }
    }
    uint64_t tknown = 0;
    for (uint32_t j = 0; j < B; j++) {
      if (hst[j] == ST_BIG_KNOWN && hdl[j] <= big_t) {
        tdl[j] = hdl[j];
        tknown += hdl[j];
        hst[j] = ST_DONE;
      }
      unknown |= hst[j] == ST_BIG_UNKNOWN;
    }
    if (tknown) {
      if (!ctx->bfs.bytes) {  // the traversal state's first allocation: make room
        size_t fr = 0, tot = 0;
        pc_mem_info(ctx, &fr, &tot);
        if (fr < pc_select_state_bytes(ctx->nr, B) + ((size_t)1 << 30)) {
          PC_CUDA(cudaStreamSynchronize(ctx->stream));
          pc_free(ctx, ctx->Ltmp);
          pc_free(ctx, ctx->cwork);
        }
      }
      pc_traverse_slots(ctx, s, target, tdl.data());
    }
    known += tknown;
    if (tknown || changed)
      PC_CUDA(cudaMemcpyAsync(st, hst.data(), (size_t)B * 4, cudaMemcpyHostToDevice, ctx->stream));
    total += known;
  }
  if (hs[1]) {
    // big CCs without a center among the first QCAP vertices: rebuild the
    // labels of the affected batches, then dense passes
    std::vector<uint32_t> hst(B);
    PC_CUDA(cudaMemcpyAsync(hst.data(), st, (size_t)B * 4, cudaMemcpyDeviceToHost, ctx->stream));
    uint32_t srow = 0;
    PC_CUDA(cudaMemcpyAsync(&srow, ctx->cid.as<uint32_t>() + s, 4, cudaMemcpyDeviceToHost,
                            ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->Ltmp.bytes < (size_t)nr * ctx->Bb * 4) {  // released for the traversal state
      pc_free(ctx, ctx->cwork);
      ctx->Bb = choose_batch(ctx);
      pc_ensure(ctx, ctx->Ltmp, std::max<size_t>((size_t)nr * ctx->Bb, 1) * 4);
    }
    const uint32_t Bb = ctx->Bb;
    uint32_t *Lb = ctx->Ltmp.as<uint32_t>();
    pc_ensure(ctx, ctx->scratch2, (size_t)Bb * 24 + 64);
    unsigned long long *cnt = ctx->scratch2.as<unsigned long long>();
    uint32_t *sroot = reinterpret_cast<uint32_t *>(cnt + Bb), *clab = sroot + Bb, *seedf = clab + Bb;
    unsigned long long *ctr = ctx->counters.as<unsigned long long>();
    for (uint32_t j0 = 0; j0 < B; j0 += Bb) {
      const uint32_t bb = std::min(Bb, B - j0);
      bool any = false;
      for (uint32_t j = j0; j < j0 + bb; j++) any |= hst[j] != ST_DONE;
      if (!any) continue;
      pc_sketch_pass(ctx, Lb, j0, bb, ctr, nullptr);
      k_seed_roots<<<(bb + 255) / 256, 256, 0, ctx->stream>>>(Lb, bb, srow, sroot);
      PC_CUDA(cudaMemsetAsync(cnt, 0, (size_t)bb * 8, ctx->stream));
      PC_CUDA(cudaMemsetAsync(clab, 0xFF, (size_t)bb * 4, ctx->stream));
      PC_CUDA(cudaMemsetAsync(seedf, 0, (size_t)bb * 4, ctx->stream));
      k_big_analyze<<<pc_grid(ctx, (size_t)nr * bb, 256, 16), 256, 0, ctx->stream>>>(
          Lb, nr, bb, j0, B, st, sroot, ctx->rmap.as<uint32_t>(), ctx->center_of.as<uint32_t>(),
          ctx->clabel.as<uint32_t>(), ctx->is_seed.as<uint8_t>(), cnt, clab, seedf);
      k_big_decide<<<(bb + 255) / 256, 256, 0, ctx->stream>>>(bb, j0, B, st, dl, lab, cnt, clab,
                                                             seedf, ctx->csz.as<uint32_t>(),
                                                             sum);
      k_big_apply<<<pc_grid(ctx, (size_t)nr * 32, 256, 16), 256, 0, ctx->stream>>>(
          Lb, nr, bb, j0, st, dl, sroot, ctx->rmap.as<uint32_t>(), s,
          reinterpret_cast<long long *>(target), ctx->dlist);
      PC_CHECK_LAUNCH();
      ctx->launches += 4;
    }
    PC_CUDA(cudaMemcpyAsync(&total, sum, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    total += known;  // sum[0] holds the probe's and the rebuild's deltas
  }
  k_set_seed<<<1, 1, 0, ctx->stream>>>(reinterpret_cast<long long *>(target), ctx->is_seed.as<uint8_t>(),
                                       s, 0);
  PC_CHECK_LAUNCH();
  *local_gain = (int64_t)total;
}

void pc_select_compressed(pacim_ctx *ctx, uint32_t k, uint32_t *seeds, int64_t *gain_num,
                          int64_t *sigma_num) {
  const uint32_t n = ctx->n;
  cudaEvent_t e0, e1;
  PC_CUDA(cudaEventCreate(&e0));
  PC_CUDA(cudaEventCreate(&e1));
  PC_CUDA(cudaEventRecord(e0, ctx->stream));
  pc_ensure(ctx, ctx->gain, (size_t)n * 8);
  PC_CUDA(cudaMemcpyAsync(ctx->gain.p, ctx->gain0.p, (size_t)n * 8, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  pc_select_reset_compressed(ctx);
  ctx->stats.select_bfs_visits = 0;
  ctx->stats.select_center_visits = 0;
  ctx->stats.select_center_found = 0;
  ctx->stats.select_hotsum_steps = 0;
  ctx->launches = 0;
  long long run = 0;
  for (uint32_t i = 0; i < k; i++) {
    uint32_t s = 0;
    int64_t g = 0, got = 0;
    const void *dsel = pc_argmax_async(ctx, ctx->gain.as<int64_t>(), n);
    pc_cover_compressed(ctx, 0, ctx->gain.as<int64_t>(), &got, dsel, &s, &g);
    k_set_seed<<<1, 1, 0, ctx->stream>>>(ctx->gain.as<long long>(), ctx->is_seed.as<uint8_t>(), s,
                                         1);
    PC_CHECK_LAUNCH();
    ctx->launches += 3;
    PC_REQUIRE(got == g, PACIM_ECHECK,
               "compressed select: sum_r delta_r = " + std::to_string(got) +
                   " differs from the argmax gain " + std::to_string(g));
    seeds[i] = s;
    gain_num[i] = g;
    run += g;
    sigma_num[i] = run;
  }
  PC_CUDA(cudaEventRecord(e1, ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.t_select_ms = ms;
  ctx->stats.kernel_launches_select = ctx->launches;
}

void pc_get_center_sketch(pacim_ctx *ctx, uint32_t slot, uint32_t *label, uint32_t *size) {
  const uint32_t rho = ctx->rho, B = ctx->R_local;
  if (!rho) return;
  std::vector<uint32_t> a((size_t)rho * B), b((size_t)rho * B);
  PC_CUDA(cudaMemcpyAsync(a.data(), ctx->clabel.p, (size_t)rho * B * 4, cudaMemcpyDeviceToHost,
                          ctx->stream));
  PC_CUDA(cudaMemcpyAsync(b.data(), ctx->csz.p, (size_t)rho * B * 4, cudaMemcpyDeviceToHost,
                          ctx->stream));
  PC_CUDA(cudaStreamSynchronize(ctx->stream));
  for (uint32_t i = 0; i < rho; i++) {
    label[i] = a[(size_t)i * B + slot];
    const uint32_t x = b[(size_t)i * B + slot];
    size[i] = (x & 0x80000000u) ? 0u : x;  // covered in the last selection: 0
  }
}
