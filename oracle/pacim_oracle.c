/*
 * pacim_oracle.c — plain, slow, single-threaded CPU ORACLE for the PaC-IM hot
 * path (arXiv 2311.07554).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2311_07554_b200/ and never imports it.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n (section named beside
 * it); DESIGN.md §"Readings" (R1..R12) lists every choice the paper leaves open.
 *
 * Everything is integer; results are defined exactly (no tolerance).
 * Single-threaded except orc_verify, which may split its sketches over
 * threads ("sketch-parallel threads allowed").
 *
 * Functions and what pins them (tests/test_oracle_*.py):
 *   orc_mix64 ............ published splitmix64 output vectors (pinned)
 *   orc_t32_const/wic .... closed forms p=0,1/2,1 and 2/(du+dv) (pinned)
 *   orc_t32_uniform ...... R19, U(lo, hi) per edge from the edge key: lo = hi
 *                          reduces to the constant; range, mean and
 *                          uniformity checked statistically (pinned)
 *   orc_live ............. symmetry, p=0/1 extremes, live fraction ~ p (pinned, statistical)
 *   orc_live_decor ....... R20 decorrelated rule: live fraction ~ p, co-liveness of two
 *                          sketches ~ p^2 (pinned, statistical)
 *   orc_simulate_ic ...... R21 Monte-Carlo sigma(S): p = 0 / 1 closed forms, exact sigma by
 *                          world enumeration within 5 standard errors (pinned)
 *   orc_sketch_labels .... scipy connected_components on the materialised
 *                          sampled graph; p=0 / p=1 special cases (pinned)
 *   orc_greedy ........... brute-force set-union greedy on tiny inputs, closed
 *                          forms (p=0, p=1, star, path), (1-1/e)*OPT, exact
 *                          sigma by 2^m world enumeration across hash seeds (pinned)
 *   orc_verify ........... verify mode: certifies a claimed
 *                          (seed, gain) sequence with O(n) memory per thread;
 *                          pinned by verify(orc_greedy(x)) = accepted and by
 *                          rejection of every one-seed swap / gain +-1
 *   orc_compressed_sketch / orc_get_center / orc_greedy_alg3 ....
 *                          Alg. 3 transcribed; pinned by SPEC-style trivia and
 *                          by equality with orc_greedy (compression transparency)
 *   orc_gen_* ............ input generators (not method arithmetic); pinned by
 *                          structural invariants and exact edge counts.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

#define ORC_UNSET 0xFFFFFFFFu

/* ------------------------------------------------------------------------ */
/* Hash (Implementation notes; reading R1-R3 in DESIGN.md)            */
/* ------------------------------------------------------------------------ */

/* R1: `hash` is the splitmix64 finalizer (unnamed in P:3). */
uint64_t orc_mix64(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

/* R2: K = mix64(hash_seed); hash(r) = mix64((2^63 | r) xor K). */
uint64_t orc_hash_r(uint64_t hash_seed, uint32_t r)
{
    uint64_t K = orc_mix64(hash_seed);
    return orc_mix64(((1ull << 63) | (uint64_t)r) ^ K);
}

/* R2: hash(min(u,v) << 32 | max(u,v)) keyed by K (P:3). */
uint64_t orc_hash_e(uint64_t hash_seed, uint32_t u, uint32_t v)
{
    uint64_t K = orc_mix64(hash_seed);
    uint64_t a = u < v ? u : v, b = u < v ? v : u;
    return orc_mix64(((a << 32) | b) ^ K);
}

/* P:3: hash_edge(u,v,r) = hash(r) xor hash(min<<32|max). */
uint64_t orc_hash_edge(uint64_t hash_seed, uint32_t u, uint32_t v, uint32_t r)
{
    return orc_hash_r(hash_seed, r) ^ orc_hash_e(hash_seed, u, v);
}

/* R3: p quantised to T32 = floor(p * 2^32) in IEEE double; p=1 -> 2^32. */
uint64_t orc_t32_const(double p)
{
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return 1ull << 32;
    return (uint64_t)floor(p * 4294967296.0);
}

/* R4: WIC p(u,v) = 2/(d_u+d_v), capped at 1:
 *     T32 = min(2^32, floor(2^33 / (d_u + d_v))). */
uint64_t orc_t32_wic(uint64_t du, uint64_t dv)
{
    uint64_t s = du + dv;
    if (s == 0) return 1ull << 32;
    uint64_t t = (1ull << 33) / s;
    return t > (1ull << 32) ? (1ull << 32) : t;
}

/* R19 (NEXT f4): Uniform p(u,v) ~ U(lo, hi) ("draw a uniform random
 * number from x to y" per edge), drawn deterministically from the edge key
 * with a fixed key K_U (a graph property, independent of the
 * sketch hash seed):
 *     L = floor(lo 2^32), H = min(floor(hi 2^32), 2^32 - 1)   (IEEE double)
 *     u = hi32(mix64((min<<32 | max) xor K_U))                 uniform on [0, 2^32)
 *     T32(u,v) = L + floor((H - L) u / 2^32)                   in [L, H]
 * The model's parameter packs both bounds: t32 = H << 32 | L. */
#define ORC_K_U_SEED 0x5EED0F0DDBA11E55ull

uint64_t orc_t32_uniform(uint64_t packed, uint32_t u, uint32_t v)
{
    uint64_t L = packed & 0xFFFFFFFFull, H = packed >> 32;
    uint64_t a = u < v ? u : v, b = u < v ? v : u;
    uint64_t x = orc_mix64(((a << 32) | b) ^ orc_mix64(ORC_K_U_SEED)) >> 32;
    return L + (((H - L) * x) >> 32);
}

/* P:4: edge (u,v) is in the r-th sampled graph iff hash_edge(u,v,r) < p(u,v);
 * R3: with p quantised to T32 this is hash_edge < T32 * 2^32. */
int orc_live(uint64_t hash_seed, uint32_t u, uint32_t v, uint32_t r, uint64_t t32)
{
    uint64_t h = orc_hash_edge(hash_seed, u, v, r);
    if (t32 >= (1ull << 32)) return 1;
    return h < (t32 << 32);
}

/* R20 (NEXT f3): the decorrelated rule, an option beside the literal P:3-4:
 *     live'(u,v,r) <=> hi32(mix64(hash(r) xor hash(min<<32|max))) < T32
 * (the literal rule only compares leading bits, so sketches whose
 * hash(r) share those bits sample nearly the same edges). */
int orc_live_decor(uint64_t hash_seed, uint32_t u, uint32_t v, uint32_t r, uint64_t t32)
{
    if (t32 >= (1ull << 32)) return 1;
    return (orc_mix64(orc_hash_edge(hash_seed, u, v, r)) >> 32) < t32;
}

/* The oracle's model word: bits 0-7 the probability model (0 = constant T32,
 * 1 = WIC, 2 = Uniform U(lo, hi), R19, t32 = H << 32 | L), bits 8-15 the hash
 * rule (0 = literal P:3-4, 1 = decorrelated R20). */
static int live_m(int model, uint64_t hash_seed, uint32_t u, uint32_t v, uint32_t r,
                  uint64_t t32)
{
    return (model >> 8) == 1 ? orc_live_decor(hash_seed, u, v, r, t32)
                             : orc_live(hash_seed, u, v, r, t32);
}

static uint64_t edge_t32(int model, uint64_t t32, const uint64_t *off,
                         uint32_t u, uint32_t v)
{
    model &= 0xFF;
    if (model == 1)
        return orc_t32_wic(off[u + 1] - off[u], off[v + 1] - off[v]);
    if (model == 2)
        return orc_t32_uniform(t32, u, v);
    return t32;
}

/* ------------------------------------------------------------------------ */
/* Sketch(r): connected components of G'_r (Alg. 3)         */
/* ------------------------------------------------------------------------ */

/* The live test of P:3-4 (R3) / R20 on a precomputed h = hash_edge(u,v,r):
 * the same rule as orc_live / orc_live_decor with the sketch's constants
 * K = mix64(hash_seed) and hash(r) computed once per sketch. */
static int live_h(int model, uint64_t h, uint64_t T)
{
    if (T >= (1ull << 32)) return 1;
    if ((model >> 8) == 1) return (orc_mix64(h) >> 32) < T;
    return h < (T << 32);
}

/*
 * label[v] = smallest vertex id in v's CC of G'_r (reading R8: canonical
 * label); if size_of_v != NULL, size_of_v[v] = |C_r(v)|.  Plain BFS from every
 * unlabelled vertex in ascending id order, testing liveness of each adjacency
 * entry with the hash rule.  Returns the number of CCs, or -1 on OOM.
 * nbr_deg (optional, WIC only) = deg(nbr[e]) per adjacency entry, so the WIC
 * threshold of an entry needs no random read of off[] (verify mode at c4).
 */
static long sketch_labels(uint32_t n, const uint64_t *off, const uint32_t *nbr,
                          const uint32_t *nbr_deg, int model, uint64_t t32,
                          uint64_t hash_seed, uint32_t r, uint32_t *label,
                          uint32_t *size_of_v)
{
    uint32_t *queue = (uint32_t *)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
    if (!queue) return -1;
    const uint64_t K = orc_mix64(hash_seed);
    const uint64_t hr = orc_mix64(((1ull << 63) | (uint64_t)r) ^ K);   /* R2 */
    for (uint32_t v = 0; v < n; v++) label[v] = ORC_UNSET;
    long ncc = 0;
    for (uint32_t v = 0; v < n; v++) {
        if (label[v] != ORC_UNSET) continue;
        size_t head = 0, tail = 0;
        label[v] = v;
        queue[tail++] = v;
        while (head < tail) {
            uint32_t x = queue[head++];
            for (uint64_t e = off[x]; e < off[x + 1]; e++) {
                uint32_t w = nbr[e];
                uint64_t a = x < w ? x : w, b = x < w ? w : x;
                uint64_t h = hr ^ orc_mix64(((a << 32) | b) ^ K);      /* P:3 */
                uint64_t T = (nbr_deg && (model & 0xFF) == 1)
                                 ? orc_t32_wic(off[x + 1] - off[x], nbr_deg[e])
                                 : edge_t32(model, t32, off, x, w);
                if (!live_h(model, h, T)) continue;                   /* P:4 */
                if (label[w] != ORC_UNSET) continue;
                label[w] = v;
                queue[tail++] = w;
            }
        }
        if (size_of_v)
            for (size_t i = 0; i < tail; i++) size_of_v[queue[i]] = (uint32_t)tail;
        ncc++;
    }
    free(queue);
    return ncc;
}

long orc_sketch_labels(uint32_t n, const uint64_t *off, const uint32_t *nbr,
                       int model, uint64_t t32, uint64_t hash_seed, uint32_t r,
                       uint32_t *label, uint32_t *size_of_v)
{
    return sketch_labels(n, off, nbr, NULL, model, t32, hash_seed, r, label, size_of_v);
}

/* BFS of C_r(s) over live edges; writes members to out[], returns count.
 * stamp[] is a caller-owned visited array compared against `tag`. */
static size_t bfs_component(uint32_t s, const uint64_t *off, const uint32_t *nbr,
                            int model, uint64_t t32, uint64_t hash_seed,
                            uint32_t r, uint32_t *stamp, uint32_t tag,
                            uint32_t *out)
{
    size_t head = 0, tail = 0;
    stamp[s] = tag;
    out[tail++] = s;
    while (head < tail) {
        uint32_t x = out[head++];
        for (uint64_t e = off[x]; e < off[x + 1]; e++) {
            uint32_t w = nbr[e];
            if (stamp[w] == tag) continue;
            if (live_m(model, hash_seed, x, w, r, edge_t32(model, t32, off, x, w))) {
                stamp[w] = tag;
                out[tail++] = w;
            }
        }
    }
    return tail;
}

/* ------------------------------------------------------------------------ */
/* Greedy over R fixed sketches (P:396-401 GeneralGreedy;   */
/* memoised CC influence P:597-601; Alg. 1; tie by id P:2285-2286)  */
/* ------------------------------------------------------------------------ */

/*
 * Derive mode.  N(S) = sum_r |reach_{G'_r}(S)|.  gain[v] starts at
 * sum_r |C_r(v)| (= R * Marginal(empty, v)); each step picks the
 * smallest-id v not in S with maximal gain (R5, R6), records gain_num =
 * N(S+s) - N(S) and sigma_num = N(S+s), then for every sketch where C_r(s) is
 * not yet covered, marks it covered and subtracts |C_r(s)| from the gain of
 * each of its members (found by BFS over live edges).
 *
 * gain0 (optional, n entries) receives the initial gains.  Returns 0, -1 on
 * OOM, -2 if the per-step cross-check sum_r delta_r == gain[s] fails.
 */
int orc_greedy(uint32_t n, const uint64_t *off, const uint32_t *nbr, int model,
               uint64_t t32, uint32_t R, uint64_t hash_seed, uint32_t k,
               uint32_t *seeds, int64_t *gain_num, int64_t *sigma_num,
               int64_t *gain0)
{
    int rc = 0;
    uint32_t *labels = (uint32_t *)malloc((size_t)R * n * sizeof(uint32_t));
    uint32_t *sizev = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    int64_t *gain = (int64_t *)calloc(n, sizeof(int64_t));
    uint8_t *is_seed = (uint8_t *)calloc(n, 1);
    uint8_t *covered = (uint8_t *)calloc(((size_t)R * n + 7) / 8, 1);
    uint32_t *stamp = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint32_t *members = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    if (!labels || !sizev || !gain || !is_seed || !covered || !stamp || !members) {
        rc = -1;
        goto done;
    }
    /* Step 1 of Alg. 1: every sketch; gain[v] += |C_r(v)|. */
    for (uint32_t r = 0; r < R; r++) {
        if (orc_sketch_labels(n, off, nbr, model, t32, hash_seed, r,
                              labels + (size_t)r * n, sizev) < 0) {
            rc = -1;
            goto done;
        }
        for (uint32_t v = 0; v < n; v++) gain[v] += sizev[v];
    }
    if (gain0) memcpy(gain0, gain, (size_t)n * sizeof(int64_t));
    for (uint32_t v = 0; v < n; v++) stamp[v] = 0;
    uint32_t tag = 0;
    int64_t sigma = 0;
    /* Step 2 of Alg. 1: k greedy steps. */
    for (uint32_t i = 0; i < k; i++) {
        int64_t best = -1;
        uint32_t s = 0;
        for (uint32_t v = 0; v < n; v++)
            if (!is_seed[v] && gain[v] > best) { best = gain[v]; s = v; }
        int64_t dsum = 0;
        for (uint32_t r = 0; r < R; r++) {
            uint32_t c = labels[(size_t)r * n + s];
            size_t bit = (size_t)r * n + c;
            if (covered[bit >> 3] & (1u << (bit & 7))) continue; /* delta_r = 0 */
            covered[bit >> 3] |= (uint8_t)(1u << (bit & 7));
            if (++tag == 0) { /* wrap: reset stamps */
                for (uint32_t v = 0; v < n; v++) stamp[v] = 0;
                tag = 1;
            }
            size_t sz = bfs_component(s, off, nbr, model, t32, hash_seed, r,
                                      stamp, tag, members);
            dsum += (int64_t)sz;
            for (size_t j = 0; j < sz; j++) gain[members[j]] -= (int64_t)sz;
        }
        if (dsum != best) rc = -2;
        is_seed[s] = 1;
        sigma += best;
        seeds[i] = s;
        gain_num[i] = best;
        sigma_num[i] = sigma;
    }
done:
    free(labels); free(sizev); free(gain); free(is_seed); free(covered);
    free(stamp); free(members);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Verify mode (SURVEY §8(c) "Verify mode"; GeneralGreedy P:396-401, Alg. 1's */
/* NextSeed / MarkSeed loop P:524-530, tie by id P:2285-2286)                 */
/* ------------------------------------------------------------------------ */
/*
 * Certifies a CLAIMED greedy sequence (s_1..s_k, g_1..g_k) — e.g. the GPU's —
 * for configs whose derive mode is out of reach (c4, c5): O(n) memory per
 * thread, one BFS labelling per sketch, sketches split over `nthreads`
 * threads (sketch-parallel only; nothing else is parallel except the argmax
 * scan of step 2, whose result is order independent).
 *
 * With S_{i-1} = {s_1..s_{i-1}} and first_r(c) = the first i with s_i in CC c
 * of sketch r (none: infinity), the greedy's step-i gain of v is
 *     gain_i(v) = sum_r [first_r(C_r(v)) >= i] |C_r(v)|
 *               = gain0(v) - sum_{j<i} B_j(v),
 *     B_j(v)    = sum_{r : first_r(C_r(v)) = j} |C_r(v)|.
 * 1. For each sketch r: label it (sketch_labels, the derive mode's BFS),
 *    find first_r of the claimed seeds' CCs, add |C_r(v)| to gain0(v) for
 *    every v, and append (v, |C_r(v)|) to the list of step first_r(C_r(v))
 *    when that is finite (the members of C_r(s_j) first covered at step j).
 * 2. Sweep i = 1..k with acc = gain_i: check
 *    (a) acc[s_i] = g_i, and
 *    (b) s_i is the argmax of acc over v not in S_{i-1} under (gain desc,
 *        id asc) — derive mode's NextSeed;
 *    then subtract B_i.
 * By induction on i a sequence that passes is exactly derive mode's output.
 *
 * Returns 0 = certified, 1 = (a) fails, 2 = (b) fails, 3 = a claimed seed
 * repeats or is >= n, -1 = out of memory.  info[4] (may be NULL) receives
 * {failing step (0-based), the oracle's argmax at that step, its gain, the
 * claimed seed's true gain}; on success {k, 0, 0, sum of the B lists}.
 */
/* One step's list B_j of one thread: (v, |C_r(v)|) pairs, switched to a
 * dense int64[n] accumulator once it holds n pairs (giant CCs, e.g. c3's first
 * seed), so the memory stays below min(8 len, 8 n) bytes. */
typedef struct { uint32_t v, size; } orc_vs;
typedef struct { orc_vs *a; size_t len, cap; int64_t *dense; } orc_vs_list;

typedef struct {
    uint32_t n; const uint64_t *off; const uint32_t *nbr; const uint32_t *nbr_deg;
    int model; uint64_t t32;
    uint32_t R; uint64_t hash_seed; uint32_t k; const uint32_t *seeds;
    int64_t *gain0;                 /* shared, updated atomically */
    uint32_t next_r;                /* shared sketch counter */
    int oom;
} orc_vctx;

typedef struct {
    orc_vctx *c;
    orc_vs_list *steps;             /* k lists owned by this thread */
} orc_vthr;

static int vs_push(orc_vs_list *l, uint32_t n, uint32_t v, uint32_t size)
{
    if (l->dense) {
        l->dense[v] += size;
        l->len++;
        return 0;
    }
    if (l->len == n) {
        l->dense = (int64_t *)calloc(n, sizeof(int64_t));
        if (!l->dense) return -1;
        for (size_t j = 0; j < l->len; j++) l->dense[l->a[j].v] += l->a[j].size;
        free(l->a);
        l->a = NULL;
        l->cap = 0;
        l->dense[v] += size;
        l->len++;
        return 0;
    }
    if (l->len == l->cap) {
        size_t cap = l->cap ? 2 * l->cap : 64;
        if (cap > n) cap = n;
        orc_vs *a = (orc_vs *)realloc(l->a, cap * sizeof(orc_vs));
        if (!a) return -1;
        l->a = a;
        l->cap = cap;
    }
    l->a[l->len].v = v;
    l->a[l->len].size = size;
    l->len++;
    return 0;
}

static void *verify_worker(void *arg)
{
    orc_vthr *t = (orc_vthr *)arg;
    orc_vctx *c = t->c;
    uint32_t n = c->n;
    uint32_t *label = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint32_t *size = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint32_t *first = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    if (!label || !size || !first) {
        __atomic_store_n(&c->oom, 1, __ATOMIC_RELAXED);
        goto out;
    }
    for (uint32_t v = 0; v < n; v++) first[v] = ORC_UNSET;
    for (;;) {
        uint32_t r = __atomic_fetch_add(&c->next_r, 1, __ATOMIC_RELAXED);
        if (r >= c->R || __atomic_load_n(&c->oom, __ATOMIC_RELAXED)) break;
        if (sketch_labels(n, c->off, c->nbr, c->nbr_deg, c->model, c->t32, c->hash_seed, r,
                          label, size) < 0) {
            __atomic_store_n(&c->oom, 1, __ATOMIC_RELAXED);
            break;
        }
        /* first_r(c): the first step whose seed lies in CC c (labels are CC ids) */
        for (uint32_t i = 0; i < c->k; i++) {
            uint32_t cc = label[c->seeds[i]];
            if (first[cc] == ORC_UNSET) first[cc] = i;
        }
        for (uint32_t v = 0; v < n; v++) {
            __atomic_fetch_add(&c->gain0[v], (int64_t)size[v], __ATOMIC_RELAXED);
            uint32_t j = first[label[v]];
            if (j != ORC_UNSET && vs_push(&t->steps[j], n, v, size[v]) < 0) {
                __atomic_store_n(&c->oom, 1, __ATOMIC_RELAXED);
                break;
            }
        }
        for (uint32_t i = 0; i < c->k; i++) first[label[c->seeds[i]]] = ORC_UNSET;
    }
out:
    free(label); free(size); free(first);
    return NULL;
}

typedef struct { const uint64_t *off; const uint32_t *nbr; uint32_t *out; uint64_t lo, hi; } orc_degslice;

static void *degslice_worker(void *arg)
{
    orc_degslice *d = (orc_degslice *)arg;
    for (uint64_t e = d->lo; e < d->hi; e++)
        d->out[e] = (uint32_t)(d->off[d->nbr[e] + 1] - d->off[d->nbr[e]]);
    return NULL;
}

int orc_verify(uint32_t n, const uint64_t *off, const uint32_t *nbr, int model,
               uint64_t t32, uint32_t R, uint64_t hash_seed, uint32_t k,
               const uint32_t *seeds, const int64_t *gain_num, int nthreads,
               int64_t *info)
{
    int rc = 0;
    if (nthreads < 1) nthreads = 1;
    for (uint32_t i = 0; i < k; i++)
        if (seeds[i] >= n) {
            if (info) { info[0] = i; info[1] = info[2] = info[3] = -1; }
            return 3;
        }
    orc_vctx c = {n, off, nbr, NULL, model, t32, R, hash_seed, k, seeds, NULL, 0, 0};
    uint32_t *nbr_deg = NULL;
    if ((model & 0xFF) == 1) {   /* WIC: deg(nbr[e]) per entry, one pass (threads: slices) */
        nbr_deg = (uint32_t *)malloc((size_t)(off[n] ? off[n] : 1) * sizeof(uint32_t));
        pthread_t *dt = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
        orc_degslice *ds = (orc_degslice *)calloc((size_t)nthreads, sizeof(orc_degslice));
        if (!nbr_deg || !dt || !ds) { free(nbr_deg); free(dt); free(ds); return -1; }
        for (int t = 0; t < nthreads; t++) {
            ds[t].off = off; ds[t].nbr = nbr; ds[t].out = nbr_deg;
            ds[t].lo = off[n] * (uint64_t)t / (uint64_t)nthreads;
            ds[t].hi = off[n] * (uint64_t)(t + 1) / (uint64_t)nthreads;
            if (t) pthread_create(&dt[t], NULL, degslice_worker, &ds[t]);
        }
        degslice_worker(&ds[0]);
        for (int t = 1; t < nthreads; t++) pthread_join(dt[t], NULL);
        free(dt); free(ds);
        c.nbr_deg = nbr_deg;
    }
    c.gain0 = (int64_t *)calloc(n ? n : 1, sizeof(int64_t));
    uint8_t *is_seed = (uint8_t *)calloc(n ? n : 1, 1);
    orc_vthr *thr = (orc_vthr *)calloc((size_t)nthreads, sizeof(orc_vthr));
    pthread_t *tid = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!c.gain0 || !is_seed || !thr || !tid) { rc = -1; goto done; }
    for (int t = 0; t < nthreads; t++) {
        thr[t].c = &c;
        thr[t].steps = (orc_vs_list *)calloc(k ? k : 1, sizeof(orc_vs_list));
        if (!thr[t].steps) { rc = -1; goto done; }
    }
    /* Step 1: sketches, one BFS labelling each, split over the threads. */
    for (int t = 1; t < nthreads; t++) pthread_create(&tid[t], NULL, verify_worker, &thr[t]);
    verify_worker(&thr[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(tid[t], NULL);
    if (c.oom) { rc = -1; goto done; }
    /* Step 2: acc = gain_i, i = 1..k (acc reuses gain0's storage). */
    int64_t *acc = c.gain0;
    int64_t total = 0;
    for (uint32_t i = 0; i < k; i++) {
        uint32_t s = seeds[i];
        if (is_seed[s]) {
            if (info) { info[0] = i; info[1] = s; info[2] = -1; info[3] = -1; }
            rc = 3;
            goto done;
        }
        /* NextSeed: max gain over v not in S_{i-1}, smallest id on ties */
        int64_t best = -1;
        uint32_t arg = 0;
        for (uint32_t v = 0; v < n; v++)
            if (!is_seed[v] && acc[v] > best) { best = acc[v]; arg = v; }
        if (acc[s] != gain_num[i] || arg != s) {
            if (info) { info[0] = i; info[1] = arg; info[2] = best; info[3] = acc[s]; }
            rc = acc[s] != gain_num[i] ? 1 : 2;
            goto done;
        }
        is_seed[s] = 1;
        /* MarkSeed: the CCs first covered at step i leave every member's gain */
        for (int t = 0; t < nthreads; t++) {
            orc_vs_list *l = &thr[t].steps[i];
            if (l->dense)
                for (uint32_t v = 0; v < n; v++) acc[v] -= l->dense[v];
            else
                for (size_t j = 0; j < l->len; j++) acc[l->a[j].v] -= l->a[j].size;
            total += (int64_t)l->len;
        }
    }
    if (info) { info[0] = k; info[1] = 0; info[2] = 0; info[3] = total; }
done:
    if (thr)
        for (int t = 0; t < nthreads; t++) {
            if (!thr[t].steps) continue;
            for (uint32_t i = 0; i < k; i++) {
                free(thr[t].steps[i].a);
                free(thr[t].steps[i].dense);
            }
            free(thr[t].steps);
        }
    free(thr); free(tid); free(c.gain0); free(is_seed); free(nbr_deg);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Compressed sketches (Alg. 3; §3)       */
/* ------------------------------------------------------------------------ */

/* R9: v is a center iff hi32(mix64(v xor K_c)) < A32,
 *     K_c = mix64(hash_seed xor 0x9E3779B97F4A7C15). A32 >= 2^32: all. */
int orc_is_center(uint64_t hash_seed, uint32_t v, uint64_t a32)
{
    if (a32 >= (1ull << 32)) return 1;
    uint64_t Kc = orc_mix64(hash_seed ^ 0x9E3779B97F4A7C15ull);
    return (orc_mix64((uint64_t)v ^ Kc) >> 32) < a32;
}

/* centers c_0 < c_1 < ... in vertex order; returns rho.  center_of[v] = index
 * or ORC_UNSET.  ("randomly selected centers".) */
uint32_t orc_centers(uint32_t n, uint64_t hash_seed, uint64_t a32,
                     uint32_t *centers, uint32_t *center_of)
{
    uint32_t rho = 0;
    for (uint32_t v = 0; v < n; v++) {
        if (orc_is_center(hash_seed, v, a32)) {
            if (center_of) center_of[v] = rho;
            if (centers) centers[rho] = v;
            rho++;
        } else if (center_of) {
            center_of[v] = ORC_UNSET;
        }
    }
    return rho;
}

/*
 * Sketch(r) of Alg. 3: CCs of G'_r; for each center c_i,
 * label[i] = min{ j : c_j in the same CC as c_i };
 * size[i] = CC size of c_i when label[i] = i, else 0.
 * Sizes count all vertices of the CC (reading R10).
 */
int orc_compressed_sketch(uint32_t n, const uint64_t *off, const uint32_t *nbr,
                          int model, uint64_t t32, uint64_t hash_seed,
                          uint32_t r, uint64_t a32, uint32_t *clabel,
                          uint32_t *csize)
{
    uint32_t *label = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint32_t *sizev = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint32_t *first_center = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    if (!label || !sizev || !first_center) {
        free(label); free(sizev); free(first_center);
        return -1;
    }
    orc_sketch_labels(n, off, nbr, model, t32, hash_seed, r, label, sizev);
    for (uint32_t v = 0; v < n; v++) first_center[v] = ORC_UNSET;
    uint32_t i = 0;
    for (uint32_t v = 0; v < n; v++) {
        if (!orc_is_center(hash_seed, v, a32)) continue;
        uint32_t cc = label[v];
        if (first_center[cc] == ORC_UNSET) first_center[cc] = i; /* min j */
        clabel[i] = first_center[cc];
        csize[i] = (clabel[i] == i) ? sizev[v] : 0;
        i++;
    }
    free(label); free(sizev); free(first_center);
    return (int)i;
}

/*
 * GetCenter(S_r, v, S) of Alg. 3: BFS from v on
 * G'_r with a local queue.  Each dequeued vertex is first checked for
 * being a center (-> return <size[label[i]], label[i]>; reading R12/R13), then
 * for being a seed.  If the BFS exhausts the CC without a center it returns
 * <0,-1> when a seed was visited, else <n',-1>.  *visits = dequeued count.
 */
void orc_get_center(uint32_t n, const uint64_t *off, const uint32_t *nbr,
                    int model, uint64_t t32, uint64_t hash_seed, uint32_t r,
                    const uint32_t *center_of, const uint32_t *clabel,
                    const uint32_t *csize, const uint8_t *is_seed, uint32_t v,
                    int64_t *delta, int64_t *l, uint64_t *visits)
{
    uint32_t *queue = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint8_t *seen = (uint8_t *)calloc(n, 1);
    size_t head = 0, tail = 0;
    int seed_seen = 0;
    *delta = 0; *l = -1;
    seen[v] = 1;
    queue[tail++] = v;
    while (head < tail) {
        uint32_t x = queue[head++];
        if (center_of[x] != ORC_UNSET) {
            uint32_t lab = clabel[center_of[x]];
            *delta = csize[lab];
            *l = lab;
            *visits = head;
            free(queue); free(seen);
            return;
        }
        if (is_seed && is_seed[x]) seed_seen = 1;
        for (uint64_t e = off[x]; e < off[x + 1]; e++) {
            uint32_t w = nbr[e];
            if (seen[w]) continue;
            if (live_m(model, hash_seed, x, w, r, edge_t32(model, t32, off, x, w))) {
                seen[w] = 1;
                queue[tail++] = w;
            }
        }
    }
    *visits = head;
    *delta = seed_seen ? 0 : (int64_t)tail;
    *l = -1;
    free(queue); free(seen);
}

/*
 * Exhaustive greedy literally on Alg. 3's compressed sketches: every step
 * evaluates Marginal(S, v) = sum_r GetCenter(S_r, v, S).delta for
 * every v not in S, takes the argmax (smallest id on ties), then MarkSeed
 * (size[l] <- 0 when l is a valid label, R11).  Tiny inputs only.
 */
int orc_greedy_alg3(uint32_t n, const uint64_t *off, const uint32_t *nbr,
                    int model, uint64_t t32, uint32_t R, uint64_t hash_seed,
                    uint64_t a32, uint32_t k, uint32_t *seeds,
                    int64_t *gain_num, int64_t *sigma_num, uint64_t *visits_out)
{
    uint32_t *center_of = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint32_t rho = orc_centers(n, hash_seed, a32, NULL, center_of);
    uint32_t *clabel = (uint32_t *)malloc((size_t)R * (rho ? rho : 1) * sizeof(uint32_t));
    uint32_t *csize = (uint32_t *)malloc((size_t)R * (rho ? rho : 1) * sizeof(uint32_t));
    uint8_t *is_seed = (uint8_t *)calloc(n, 1);
    if (!center_of || !clabel || !csize || !is_seed) return -1;
    for (uint32_t r = 0; r < R; r++)
        orc_compressed_sketch(n, off, nbr, model, t32, hash_seed, r, a32,
                              clabel + (size_t)r * rho, csize + (size_t)r * rho);
    uint64_t visits = 0;
    int64_t sigma = 0;
    for (uint32_t i = 0; i < k; i++) {
        int64_t best = -1;
        uint32_t s = 0;
        for (uint32_t v = 0; v < n; v++) {
            if (is_seed[v]) continue;
            int64_t g = 0;
            for (uint32_t r = 0; r < R; r++) {
                int64_t d, l;
                uint64_t vis;
                orc_get_center(n, off, nbr, model, t32, hash_seed, r, center_of,
                               clabel + (size_t)r * rho, csize + (size_t)r * rho,
                               is_seed, v, &d, &l, &vis);
                g += d;
                visits += vis;
            }
            if (g > best) { best = g; s = v; }
        }
        /* MarkSeed(s) */
        for (uint32_t r = 0; r < R; r++) {
            int64_t d, l;
            uint64_t vis;
            orc_get_center(n, off, nbr, model, t32, hash_seed, r, center_of,
                           clabel + (size_t)r * rho, csize + (size_t)r * rho,
                           is_seed, s, &d, &l, &vis);
            if (l >= 0) csize[(size_t)r * rho + (size_t)l] = 0;
        }
        is_seed[s] = 1;
        sigma += best;
        seeds[i] = s;
        gain_num[i] = best;
        sigma_num[i] = sigma;
    }
    if (visits_out) *visits_out = visits;
    free(center_of); free(clabel); free(csize); free(is_seed);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Input generators (counter-based; DESIGN.md §"Input recipe").  Not method    */
/* arithmetic — the oracle's own copy of the recipe, compared bit-exactly      */
/* against the CUDA generator in the GPU tests.                                */
/* ------------------------------------------------------------------------ */

static uint64_t gen_key(uint64_t gen_seed)
{
    return orc_mix64(gen_seed ^ 0xD1B54A32D192ED03ull);
}

static int cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* ER: draw j = 0,1,2,...: w = mix64(Kg ^ j), u = (lo32(w)*n)>>32,
 * v = (hi32(w)*n)>>32; skip u == v; keep the first m distinct undirected
 * pairs.  keys_out (m entries) receives sorted keys min<<32|max.
 * Returns m, or -1 (OOM / m too large). */
long orc_gen_er(uint32_t n, uint64_t m, uint64_t gen_seed, uint64_t *keys_out)
{
    if (n < 2 || m > (uint64_t)n * (n - 1) / 2) return -1;
    uint64_t Kg = gen_key(gen_seed);
    size_t cap = 1;
    while (cap < 2 * m + 2) cap <<= 1;
    uint64_t *table = (uint64_t *)malloc(cap * sizeof(uint64_t));
    if (!table) return -1;
    for (size_t i = 0; i < cap; i++) table[i] = ~0ull;
    uint64_t got = 0;
    for (uint64_t j = 0; got < m; j++) {
        uint64_t w = orc_mix64(Kg ^ j);
        uint32_t u = (uint32_t)(((w & 0xFFFFFFFFull) * n) >> 32);
        uint32_t v = (uint32_t)(((w >> 32) * n) >> 32);
        if (u == v) continue;
        uint64_t a = u < v ? u : v, b = u < v ? v : u;
        uint64_t key = (a << 32) | b;
        size_t h = (size_t)(orc_mix64(key) & (cap - 1));
        int dup = 0;
        while (table[h] != ~0ull) {
            if (table[h] == key) { dup = 1; break; }
            h = (h + 1) & (cap - 1);
        }
        if (dup) continue;
        table[h] = key;
        keys_out[got++] = key;
    }
    free(table);
    qsort(keys_out, (size_t)m, sizeof(uint64_t), cmp_u64);
    return (long)m;
}

/* R-MAT permutation pi(x) = h(g2(h(g1(x)))) on [0, 2^s). */
static uint64_t rmat_perm(uint64_t x, int s)
{
    uint64_t mask = (s == 64) ? ~0ull : ((1ull << s) - 1);
    int sh = (s + 1) / 2;
    x = (x * 0x9E3779B97F4A7C15ull) & mask;
    x ^= x >> sh;
    x = (x * 0xBF58476D1CE4E5B9ull) & mask;
    x ^= x >> sh;
    return x;
}

/* R-MAT: samples i in [0, ef*2^s); level l in [0,s): y = mix64(Kg ^ (i*64+l)) >> 11
 * (53 bits); y < ta: quadrant a; < tab: b (v bit); < tabc: c (u bit); else d
 * (both bits); level l sets bit s-1-l.  Optional permutation pi of ids; then
 * drop loops, dedup.  keys_out capacity ef*2^s.  Returns m (distinct edges). */
long orc_gen_rmat(int scale, uint32_t ef, uint64_t ta, uint64_t tab,
                  uint64_t tabc, int permute, uint64_t gen_seed,
                  uint64_t *keys_out)
{
    uint64_t Kg = gen_key(gen_seed);
    uint64_t ns = (uint64_t)ef << scale;
    uint64_t cnt = 0;
    for (uint64_t i = 0; i < ns; i++) {
        uint64_t u = 0, v = 0;
        for (int l = 0; l < scale; l++) {
            uint64_t y = orc_mix64(Kg ^ (i * 64 + (uint64_t)l)) >> 11;
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
        if (permute) { u = rmat_perm(u, scale); v = rmat_perm(v, scale); }
        if (u == v) continue;
        uint64_t a = u < v ? u : v, b = u < v ? v : u;
        keys_out[cnt++] = (a << 32) | b;
    }
    qsort(keys_out, (size_t)cnt, sizeof(uint64_t), cmp_u64);
    uint64_t m = 0;
    for (uint64_t i = 0; i < cnt; i++)
        if (m == 0 || keys_out[m - 1] != keys_out[i]) keys_out[m++] = keys_out[i];
    return (long)m;
}

/* Grid W x H, id = i*W + j: edges (i,j)-(i,j+1), (i,j)-(i+1,j), and the
 * diagonal (i,j)-(i+1,j+1) iff hi32(mix64(Kg ^ (i*W+j))) < d32.  Keys are
 * emitted already sorted.  keys_out capacity 3*W*H.  Returns m. */
long orc_gen_grid(uint32_t W, uint32_t H, uint64_t d32, uint64_t gen_seed,
                  uint64_t *keys_out)
{
    uint64_t Kg = gen_key(gen_seed);
    uint64_t m = 0;
    for (uint64_t i = 0; i < H; i++) {
        for (uint64_t j = 0; j < W; j++) {
            uint64_t v = i * W + j;
            if (j + 1 < W) keys_out[m++] = (v << 32) | (v + 1);
            if (i + 1 < H) keys_out[m++] = (v << 32) | (v + W);
            if (i + 1 < H && j + 1 < W &&
                (orc_mix64(Kg ^ v) >> 32) < d32)
                keys_out[m++] = (v << 32) | (v + W + 1);
        }
    }
    return (long)m;
}

/* Symmetric CSR from sorted distinct keys (min<<32|max).  off: n+1,
 * nbr: 2m.  Neighbour lists come out sorted because keys are sorted. */
void orc_csr_from_keys(uint32_t n, uint64_t m, const uint64_t *keys,
                       uint64_t *off, uint32_t *nbr)
{
    for (uint32_t v = 0; v <= n; v++) off[v] = 0;
    for (uint64_t e = 0; e < m; e++) {
        off[(keys[e] >> 32) + 1]++;
        off[(keys[e] & 0xFFFFFFFFull) + 1]++;
    }
    for (uint32_t v = 0; v < n; v++) off[v + 1] += off[v];
    uint64_t *fill = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    for (uint32_t v = 0; v < n; v++) fill[v] = off[v];
    for (uint64_t e = 0; e < m; e++) {
        uint32_t a = (uint32_t)(keys[e] >> 32), b = (uint32_t)keys[e];
        nbr[fill[a]++] = b;
        nbr[fill[b]++] = a;
    }
    free(fill);
}

/* ------------------------------------------------------------------------ */
/* Threaded copy of the R-MAT input generator (same recipe, same output as    */
/* orc_gen_rmat + orc_csr_from_keys, checked bit for bit in the tests): the   */
/* c4 graph (1.6e9 samples) takes ~18 min single-threaded, too long for the   */
/* bench's reference arm.  Input generation only; no method arithmetic.       */
/* ------------------------------------------------------------------------ */

typedef struct {
    int scale, permute; uint64_t ta, tab, tabc, Kg;
    uint64_t lo, hi;              /* sample range */
    uint64_t *out; uint64_t cnt;  /* loop-free keys written at out[lo..] */
} orc_gen_slice;

static void *gen_slice_worker(void *arg)
{
    orc_gen_slice *g = (orc_gen_slice *)arg;
    uint64_t c = 0;
    for (uint64_t i = g->lo; i < g->hi; i++) {
        uint64_t u = 0, v = 0;
        for (int l = 0; l < g->scale; l++) {
            uint64_t y = orc_mix64(g->Kg ^ (i * 64 + (uint64_t)l)) >> 11;
            uint64_t bit = 1ull << (g->scale - 1 - l);
            if (y < g->ta) {
            } else if (y < g->tab) {
                v |= bit;
            } else if (y < g->tabc) {
                u |= bit;
            } else {
                u |= bit;
                v |= bit;
            }
        }
        if (g->permute) { u = rmat_perm(u, g->scale); v = rmat_perm(v, g->scale); }
        if (u == v) continue;
        uint64_t a = u < v ? u : v, b = u < v ? v : u;
        g->out[g->lo + c++] = (a << 32) | b;
    }
    g->cnt = c;
    return NULL;
}

/* LSD radix sort of u64 keys, 16-bit digits, T threads (per-thread digit
 * histograms of contiguous slices, so the scatter is stable). */
typedef struct {
    const uint64_t *src; uint64_t *dst; uint64_t lo, hi; int shift;
    uint64_t *hist;   /* 65536 counts, then the thread's write cursors */
    int phase;
} orc_rs_slice;

static void *rs_worker(void *arg)
{
    orc_rs_slice *r = (orc_rs_slice *)arg;
    if (r->phase == 0) {
        memset(r->hist, 0, 65536 * sizeof(uint64_t));
        for (uint64_t i = r->lo; i < r->hi; i++) r->hist[(r->src[i] >> r->shift) & 0xFFFF]++;
    } else {
        for (uint64_t i = r->lo; i < r->hi; i++) {
            uint64_t d = (r->src[i] >> r->shift) & 0xFFFF;
            r->dst[r->hist[d]++] = r->src[i];
        }
    }
    return NULL;
}

static int radix_sort_mt(uint64_t *a, uint64_t *tmp, uint64_t N, int T)
{
    orc_rs_slice *sl = (orc_rs_slice *)calloc((size_t)T, sizeof(orc_rs_slice));
    pthread_t *tid = (pthread_t *)calloc((size_t)T, sizeof(pthread_t));
    uint64_t *hist = (uint64_t *)malloc((size_t)T * 65536 * sizeof(uint64_t));
    if (!sl || !tid || !hist) { free(sl); free(tid); free(hist); return -1; }
    uint64_t *src = a, *dst = tmp;
    for (int shift = 0; shift < 64; shift += 16) {
        for (int ph = 0; ph < 2; ph++) {
            for (int t = 0; t < T; t++) {
                sl[t].src = src; sl[t].dst = dst; sl[t].shift = shift; sl[t].phase = ph;
                sl[t].lo = N * (uint64_t)t / (uint64_t)T;
                sl[t].hi = N * (uint64_t)(t + 1) / (uint64_t)T;
                sl[t].hist = hist + (size_t)t * 65536;
                if (t) pthread_create(&tid[t], NULL, rs_worker, &sl[t]);
            }
            rs_worker(&sl[0]);
            for (int t = 1; t < T; t++) pthread_join(tid[t], NULL);
            if (ph == 0) {  /* exclusive prefix over (digit, thread) */
                uint64_t run = 0;
                for (uint64_t d = 0; d < 65536; d++)
                    for (int t = 0; t < T; t++) {
                        uint64_t c = hist[(size_t)t * 65536 + d];
                        hist[(size_t)t * 65536 + d] = run;
                        run += c;
                    }
            }
        }
        uint64_t *x = src; src = dst; dst = x;
    }
    /* 4 passes: the sorted keys are back in a */
    free(sl); free(tid); free(hist);
    return 0;
}

typedef struct {
    const uint64_t *hi_keys, *lo_keys;  /* sorted by (min, max) and by (max, min) */
    uint64_t m; const uint64_t *off; uint32_t *nbr;
    uint32_t v0, v1; uint64_t ph, pl;   /* rows [v0, v1); key cursors at v0 */
} orc_csr_slice;

static void *csr_worker(void *arg)
{
    orc_csr_slice *c = (orc_csr_slice *)arg;
    uint64_t ph = c->ph, pl = c->pl;
    for (uint32_t x = c->v0; x < c->v1; x++) {
        uint64_t w = c->off[x];
        /* neighbours a < x: keys (a, x), listed by the (max, min) order */
        while (pl < c->m && (c->lo_keys[pl] >> 32) == x) c->nbr[w++] = (uint32_t)c->lo_keys[pl++];
        /* neighbours b > x: keys (x, b) */
        while (ph < c->m && (c->hi_keys[ph] >> 32) == x) c->nbr[w++] = (uint32_t)c->hi_keys[ph++];
    }
    return NULL;
}

static uint64_t lower_bound_hi(const uint64_t *k, uint64_t m, uint64_t x)
{
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if ((k[mid] >> 32) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* R-MAT graph -> CSR (off n+1, nbr 2m), threaded; keys_out (capacity ef 2^s)
 * receives the sorted distinct upper keys, tmp is scratch of the same size.
 * Returns m, or -1 on OOM. */
long orc_gen_rmat_csr_mt(int scale, uint32_t ef, uint64_t ta, uint64_t tab, uint64_t tabc,
                         int permute, uint64_t gen_seed, int T, uint64_t *keys_out,
                         uint64_t *tmp, uint64_t *off, uint32_t *nbr)
{
    if (T < 1) T = 1;
    uint64_t ns = (uint64_t)ef << scale, n = 1ull << scale;
    orc_gen_slice *gs = (orc_gen_slice *)calloc((size_t)T, sizeof(orc_gen_slice));
    pthread_t *tid = (pthread_t *)calloc((size_t)T, sizeof(pthread_t));
    if (!gs || !tid) { free(gs); free(tid); return -1; }
    for (int t = 0; t < T; t++) {
        gs[t] = (orc_gen_slice){scale, permute, ta, tab, tabc, gen_key(gen_seed),
                                ns * (uint64_t)t / (uint64_t)T, ns * (uint64_t)(t + 1) / (uint64_t)T,
                                keys_out, 0};
        if (t) pthread_create(&tid[t], NULL, gen_slice_worker, &gs[t]);
    }
    gen_slice_worker(&gs[0]);
    for (int t = 1; t < T; t++) pthread_join(tid[t], NULL);
    uint64_t cnt = 0;
    for (int t = 0; t < T; t++) {
        memmove(keys_out + cnt, keys_out + gs[t].lo, gs[t].cnt * sizeof(uint64_t));
        cnt += gs[t].cnt;
    }
    free(gs);
    if (radix_sort_mt(keys_out, tmp, cnt, T) < 0) { free(tid); return -1; }
    uint64_t m = 0;
    for (uint64_t i = 0; i < cnt; i++)
        if (m == 0 || keys_out[m - 1] != keys_out[i]) keys_out[m++] = keys_out[i];
    /* degrees and offsets */
    for (uint64_t v = 0; v <= n; v++) off[v] = 0;
    for (uint64_t e = 0; e < m; e++) {
        off[(keys_out[e] >> 32) + 1]++;
        off[(keys_out[e] & 0xFFFFFFFFull) + 1]++;
    }
    for (uint64_t v = 0; v < n; v++) off[v + 1] += off[v];
    /* the (max, min) order: swapped keys, sorted */
    for (uint64_t e = 0; e < m; e++) tmp[e] = (keys_out[e] << 32) | (keys_out[e] >> 32);
    uint64_t *tmp2 = (uint64_t *)malloc((size_t)(m ? m : 1) * sizeof(uint64_t));
    if (!tmp2 || radix_sort_mt(tmp, tmp2, m, T) < 0) { free(tmp2); free(tid); return -1; }
    free(tmp2);
    orc_csr_slice *cs = (orc_csr_slice *)calloc((size_t)T, sizeof(orc_csr_slice));
    if (!cs) { free(tid); return -1; }
    for (int t = 0; t < T; t++) {
        uint32_t v0 = (uint32_t)(n * (uint64_t)t / (uint64_t)T);
        uint32_t v1 = (uint32_t)(n * (uint64_t)(t + 1) / (uint64_t)T);
        cs[t] = (orc_csr_slice){keys_out, tmp, m, off, nbr, v0, v1,
                                lower_bound_hi(keys_out, m, v0), lower_bound_hi(tmp, m, v0)};
        if (t) pthread_create(&tid[t], NULL, csr_worker, &cs[t]);
    }
    csr_worker(&cs[0]);
    for (int t = 1; t < T; t++) pthread_join(tid[t], NULL);
    free(cs); free(tid);
    return (long)m;
}

/* ------------------------------------------------------------------------ */
/* Monte-Carlo sigma(S) (NEXT f3; IC simulation P:375-377, the paper's        */
/* "Influence ... 20000 simulations" column P:1335)           */
/* ------------------------------------------------------------------------ */
/*
 * R21: simulation i draws a fresh world: edge e = (u,v) is live iff
 *     hi32(mix64(mix64(K_mc xor i) xor (min<<32|max))) < T32(e)
 * with K_mc = mix64(mc_seed xor 0x4D435349434D4353) (T32 = 2^32: always).
 * Returns the total number of vertices reached from S over the nsims worlds
 * (sigma_hat(S) = total / nsims), or UINT64_MAX on OOM.
 */
uint64_t orc_simulate_ic(uint32_t n, const uint64_t *off, const uint32_t *nbr, int model,
                         uint64_t t32, const uint32_t *seeds, uint32_t ns, uint32_t nsims,
                         uint64_t mc_seed)
{
    uint32_t *stamp = (uint32_t *)calloc(n ? n : 1, sizeof(uint32_t));
    uint32_t *queue = (uint32_t *)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
    if (!stamp || !queue) {
        free(stamp);
        free(queue);
        return UINT64_MAX;
    }
    const uint64_t Kmc = orc_mix64(mc_seed ^ 0x4D435349434D4353ull);
    uint64_t total = 0;
    for (uint32_t i = 0; i < nsims; i++) {
        const uint32_t tag = i + 1;
        const uint64_t Ki = orc_mix64(Kmc ^ (uint64_t)i);
        size_t head = 0, tail = 0;
        for (uint32_t k = 0; k < ns; k++)
            if (stamp[seeds[k]] != tag) {
                stamp[seeds[k]] = tag;
                queue[tail++] = seeds[k];
            }
        while (head < tail) {
            uint32_t x = queue[head++];
            for (uint64_t e = off[x]; e < off[x + 1]; e++) {
                uint32_t w = nbr[e];
                if (stamp[w] == tag) continue;
                uint64_t T = edge_t32(model, t32, off, x, w);
                uint64_t a = x < w ? x : w, b = x < w ? w : x;
                if (T >= (1ull << 32) || (orc_mix64(Ki ^ ((a << 32) | b)) >> 32) < T) {
                    stamp[w] = tag;
                    queue[tail++] = w;
                }
            }
        }
        total += tail;
    }
    free(stamp);
    free(queue);
    return total;
}
