// api.cu — the extern "C" boundary declared in include/pacim.h.
// Argument validation, state machine (load -> build -> select), error
// capture; all compute is delegated to graph.cu / build.cu / select.cu.
#include <cmath>
#include <cstring>
#include <iterator>

#include "pacim_internal.cuh"

static std::string g_create_err;

// Device allocation: cudaMalloc, or first-fit sub-allocation from the
// caller's workspace (pacim_create's torch-owned buffer, SURVEY 8(b)
// ownership: "the ctx owns every device allocation, which it sub-allocates
// from the torch workspace when one is given").  256-byte alignment.
static void *ws_alloc(pacim_ctx *ctx, size_t bytes) {
  bytes = (bytes + 255) & ~(size_t)255;
  for (auto it = ctx->ws_free.begin(); it != ctx->ws_free.end(); ++it) {
    if (it->second < bytes) continue;
    const size_t off = it->first, len = it->second;
    ctx->ws_free.erase(it);
    if (len > bytes) ctx->ws_free[off + bytes] = len - bytes;
    ctx->ws_used[off] = bytes;
    return (char *)ctx->ws_base + off;
  }
  return nullptr;
}

static void ws_release(pacim_ctx *ctx, void *p) {
  const size_t off = (size_t)((char *)p - (char *)ctx->ws_base);
  auto u = ctx->ws_used.find(off);
  if (u == ctx->ws_used.end()) return;
  size_t start = off, len = u->second;
  ctx->ws_used.erase(u);
  auto nx = ctx->ws_free.lower_bound(start);
  if (nx != ctx->ws_free.end() && nx->first == start + len) {  // merge with the next hole
    len += nx->second;
    nx = ctx->ws_free.erase(nx);
  }
  if (nx != ctx->ws_free.begin()) {  // and with the previous one
    auto pv = std::prev(nx);
    if (pv->first + pv->second == start) {
      start = pv->first;
      len += pv->second;
      ctx->ws_free.erase(pv);
    }
  }
  ctx->ws_free[start] = len;
}

void pc_mem_info(pacim_ctx *ctx, size_t *fr, size_t *tot) {
  if (ctx->ws_base) {
    *fr = pc_mem_free(ctx);
    *tot = ctx->ws_bytes;
    return;
  }
  if (!ctx->mi_valid) {
    cudaMemGetInfo(&ctx->mi_free, &ctx->mi_total);
    ctx->mi_dev_bytes = ctx->device_bytes;
    ctx->mi_valid = true;
  }
  // the free bytes at the query, minus what this ctx allocated since
  const int64_t d = (int64_t)ctx->device_bytes - (int64_t)ctx->mi_dev_bytes;
  *fr = d >= (int64_t)ctx->mi_free ? 0 : (size_t)((int64_t)ctx->mi_free - d);
  *tot = ctx->mi_total;
}

size_t pc_mem_free(pacim_ctx *ctx) {
  if (ctx->ws_base) {
    size_t best = 0;
    for (auto &h : ctx->ws_free) best = std::max(best, h.second);
    return best;
  }
  size_t fr = 0, tot = 0;
  pc_mem_info(ctx, &fr, &tot);
  return fr;
}

void pc_ensure(pacim_ctx *ctx, DevBuf &b, size_t bytes) {
  if (bytes <= b.bytes && b.p) return;
  if (b.p) pc_free(ctx, b);
  if (bytes == 0) bytes = 16;
  if (ctx->ws_base) {
    // stream-ordered reuse: work already queued may still read a block that
    // was released, so a workspace allocation waits for the stream first
    cudaStreamSynchronize(ctx->stream);
    b.p = ws_alloc(ctx, bytes);
    if (!b.p)
      throw PacimError{PACIM_ENOMEM, "workspace: no free block of " + std::to_string(bytes) +
                                         " bytes (largest " + std::to_string(pc_mem_free(ctx)) +
                                         ")"};
  } else {
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      ctx->mi_valid = false;  // the tracked free memory was wrong: query again
      b.p = nullptr;
      throw PacimError{PACIM_ENOMEM, "cudaMalloc(" + std::to_string(bytes) +
                                         " bytes) failed: " + cudaGetErrorString(e)};
    }
  }
  b.bytes = bytes;
  ctx->device_bytes += bytes;
  ctx->device_peak = std::max(ctx->device_peak, ctx->device_bytes);
}

void pc_free(pacim_ctx *ctx, DevBuf &b) {
  if (b.p) {
    if (ctx->ws_base) {
      cudaStreamSynchronize(ctx->stream);
      ws_release(ctx, b.p);
    } else {
      cudaFree(b.p);
    }
    ctx->device_bytes -= b.bytes;
  }
  b.p = nullptr;
  b.bytes = 0;
}

template <typename F>
static int guarded(pacim_ctx *ctx, F &&f) {
  if (!ctx) return PACIM_EINVAL;
  ctx->err.clear();
  try {
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) throw PacimError{PACIM_ECUDA, cudaGetErrorString(e)};
    f();
    return PACIM_OK;
  } catch (const PacimError &pe) {
    ctx->err = pe.msg;
    return pe.code;
  } catch (const std::exception &ex) {
    ctx->err = ex.what();
    return PACIM_ECUDA;
  } catch (...) {
    ctx->err = "unknown error";
    return PACIM_ECUDA;
  }
}

// Dropping keeps the device buffers as capacity for the next load/build
// (pc_ensure reuses them); they are released by pacim_destroy.
static void drop_sketches(pacim_ctx *ctx) {
  ctx->built = false;
  ctx->dist_cov_valid = false;  // a new store: no covered flags to restore
  ctx->dist_cov_n = 0;
  ctx->hla_ok = false;
  ctx->sel_list_valid = false;  // the covered list refers to the old store
}

void pc_graph_loaded(pacim_ctx *ctx) {
  ctx->graph_gen++;
  uint64_t sig = pc_mix64(ctx->n);
  for (uint64_t x : {ctx->m, (uint64_t)ctx->nr, (uint64_t)ctx->pmodel, ctx->t32, (uint64_t)ctx->lean})
    sig = pc_mix64(sig ^ x);
  if (sig != ctx->graph_sig || ctx->hint_gen == 0) ctx->hint_gen++;
  ctx->graph_sig = sig;
}

static void drop_graph(pacim_ctx *ctx) {
  drop_sketches(ctx);
  ctx->has_graph = false;
  ctx->upper_src = false;  // (an upper load sets both again)
  ctx->sym_pending = false;
}

static void free_all(pacim_ctx *ctx) {
  DevBuf *bufs[] = {&ctx->off,   &ctx->nbr,        &ctx->keys,     &ctx->tm1, &ctx->ckeys, &ctx->cid, &ctx->rmap,      &ctx->L,
                    &ctx->csize, &ctx->csize_work, &ctx->coff,     &ctx->cfill,    &ctx->perm,
                    &ctx->clabel, &ctx->csz,       &ctx->csz_work, &ctx->Ltmp,     &ctx->d_shr,
                    &ctx->d_hot, &ctx->centers, &ctx->is_seed, &ctx->cwork,

                    &ctx->d_tab, &ctx->gain0,      &ctx->gain,     &ctx->center_of, &ctx->counters,
                    &ctx->scratch, &ctx->scratch2, &ctx->sel_seeds, &ctx->sel_gain,
                    &ctx->sel_partial, &ctx->sel_list, &ctx->sel_flag, &ctx->argmax_part, &ctx->bfs, &ctx->tcsr, &ctx->hidx, &ctx->hub_tab, &ctx->hla_off, &ctx->hla_row, &ctx->hla_raw, &ctx->d_smap, &ctx->pkeys, &ctx->cprobe, &ctx->cseed, &ctx->d_hr64, &ctx->crow, &ctx->vinfo, &ctx->hotsum, &ctx->d_hot_size,
                    &ctx->cs_rec, &ctx->cs_soff, &ctx->cs_ecrow, &ctx->cs_E, &ctx->cs_vid,
                    &ctx->cs_diag, &ctx->cs_cnt, &ctx->cs_plist, &ctx->edge_work, &ctx->wt_buf, &ctx->dist_ghot, &ctx->dist_buf, &ctx->dist_cov_old, &ctx->ep_tab, &ctx->ep_send, &ctx->ep_cnt, &ctx->hk_list, &ctx->uoff, &ctx->ucrow, &ctx->rk, &ctx->unbr, &ctx->ud16, &ctx->uvrow, &ctx->ucrowr};
  for (DevBuf *b : bufs) pc_free(ctx, *b);
  pc_sym_free(ctx);
}

extern "C" {

const char *pacim_version(void) { return "pacim-b200 0.1 (sm_100a)"; }

uint64_t pacim_threshold_uniform(double lo, double hi) {
  lo = std::isnan(lo) ? 0.0 : std::min(1.0, std::max(0.0, lo));
  hi = std::isnan(hi) ? 0.0 : std::min(1.0, std::max(0.0, hi));
  if (lo > hi) std::swap(lo, hi);
  const uint64_t H = std::min<uint64_t>(pacim_threshold_from_p(hi), 0xFFFFFFFFull);
  const uint64_t L = std::min<uint64_t>(pacim_threshold_from_p(lo), H);
  return (H << 32) | L;
}

uint64_t pacim_threshold_from_p(double p) {
  if (!(p > 0.0)) return 0;
  if (p >= 1.0) return 1ull << 32;
  return (uint64_t)std::floor(p * 4294967296.0);
}

int pacim_create(pacim_ctx **out, int device, void *workspace, size_t ws_bytes,
                 void *cuda_stream) {
  if (!out) return PACIM_EINVAL;
  *out = nullptr;
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  if (e != cudaSuccess) {
    g_create_err = std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e);
    return PACIM_ECUDA;
  }
  if (device < 0 || device >= cnt) {
    g_create_err = "no such CUDA device";
    return PACIM_EINVAL;
  }
  if ((workspace == nullptr) != (ws_bytes == 0)) {
    g_create_err = "workspace and ws_bytes must be given together";
    return PACIM_EINVAL;
  }
  if (workspace && ((uintptr_t)workspace & 255)) {
    g_create_err = "workspace must be 256-byte aligned";
    return PACIM_EINVAL;
  }
  pacim_ctx *ctx = new pacim_ctx();
  ctx->device = device;
  if (workspace) {
    ctx->ws_base = workspace;
    ctx->ws_bytes = ws_bytes & ~(size_t)255;
    ctx->ws_free[0] = ctx->ws_bytes;
  }
  e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount,
                                                   device);
  if (e == cudaSuccess) {
    if (cuda_stream) {
      ctx->stream = (cudaStream_t)cuda_stream;
    } else {
      e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
      ctx->own_stream = true;
    }
  }
  if (e != cudaSuccess) {
    g_create_err = cudaGetErrorString(e);
    delete ctx;
    return PACIM_ECUDA;
  }
  *out = ctx;
  return PACIM_OK;
}

void pacim_destroy(pacim_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
    cudaEventDestroy(ctx->released);
    for (auto &g : ctx->stage) {
      if (g.done) cudaEventDestroy(g.done);
      pc_free(ctx, g.off);
      pc_free(ctx, g.nbr);
    }
  }
  pc_free_comm(ctx);
  free_all(ctx);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int pacim_nccl_unique_id(void *id_out) {
  if (!id_out) return PACIM_EINVAL;
  try {
    pc_nccl_unique_id(id_out);
  } catch (const PacimError &pe) {
    g_create_err = pe.msg;
    return pe.code;
  }
  return PACIM_OK;
}

int pacim_init_comm(pacim_ctx *ctx, int rank, int world, const void *nccl_unique_id) {
  return guarded(ctx, [&] {
    PC_REQUIRE(world >= 1 && rank >= 0 && rank < world && nccl_unique_id, PACIM_EINVAL,
               "need 0 <= rank < world and a 128-byte NCCL unique id");
    pc_init_comm(ctx, rank, world, nccl_unique_id);
  });
}

const char *pacim_last_error(const pacim_ctx *ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

static void check_model(int pmodel, uint64_t t32) {
  PC_REQUIRE(pmodel == PACIM_P_CONST || pmodel == PACIM_P_WIC || pmodel == PACIM_P_UNIFORM,
             PACIM_EINVAL, "pmodel must be PACIM_P_CONST, PACIM_P_WIC or PACIM_P_UNIFORM");
  PC_REQUIRE(pmodel != PACIM_P_CONST || t32 <= (1ull << 32), PACIM_EINVAL, "t32 > 2^32");
  PC_REQUIRE(pmodel != PACIM_P_UNIFORM || (t32 & 0xFFFFFFFFull) <= (t32 >> 32), PACIM_EINVAL,
             "uniform model: L > H in t32 = H << 32 | L");
}

static void load_common(pacim_ctx *ctx, uint32_t n, uint64_t nnz, int pmodel, uint64_t t32,
                        bool want_nbr = true) {
  PC_REQUIRE(n >= 1, PACIM_EINVAL, "n must be >= 1");
  PC_REQUIRE(n < (1u << 31), PACIM_EINVAL, "n must be < 2^31 (R2 key packing)");
  PC_REQUIRE((nnz & 1) == 0, PACIM_EINVAL, "nnz must be even (symmetric CSR)");
  check_model(pmodel, t32);
  drop_graph(ctx);
  ctx->n = n;
  ctx->m = nnz / 2;
  ctx->pmodel = pmodel;
  ctx->t32 = t32;
  pc_ensure(ctx, ctx->off, ((size_t)n + 1) * 8);
  if (want_nbr) pc_ensure(ctx, ctx->nbr, std::max<uint64_t>(nnz, 1) * 4);
  else pc_free(ctx, ctx->nbr);  // an upper load: built on first use (pc_ensure_sym)
}

// commit the oldest pending asynchronous load (no-op without one)
static void commit_staged(pacim_ctx *ctx) {
  StagedGraph &st = ctx->stage[ctx->stage_commit];
  if (!st.pending) return;
  st.pending = false;
  ctx->stage_commit ^= 1;
  drop_graph(ctx);  // (the model was checked when the load was enqueued)
  ctx->n = st.n;
  ctx->m = st.nnz / 2;
  ctx->pmodel = st.pmodel;
  ctx->t32 = st.t32;
  PC_CUDA(cudaStreamWaitEvent(ctx->stream, st.done, 0));
  if (st.upper) {
    // the upper CSR becomes the graph's (the old uoff / unbr buffers are the
    // slot's next staging area); the symmetric offsets from the degrees, the
    // symmetric lists only when something reads them (pc_ensure_sym)
    std::swap(ctx->uoff, st.off);
    std::swap(ctx->unbr, st.nbr);
    pc_free(ctx, ctx->nbr);  // an earlier graph's lists
    pc_upper_degrees(ctx);
  } else {
    std::swap(ctx->off, st.off);  // the staged CSR becomes the graph; the old
    std::swap(ctx->nbr, st.nbr);  // buffers are the slot's next staging area
  }
  pc_graph_finish_load(ctx, 0);
  ctx->has_graph = true;
  pc_graph_loaded(ctx);
  PC_CUDA(cudaEventRecord(ctx->released, ctx->stream));
}

// a synchronous load replaces anything still pending (and releases the
// staging buffers: a graph loaded synchronously may need all the memory)
static void drop_staged(pacim_ctx *ctx) {
  if (ctx->copy_stream) PC_CUDA(cudaStreamSynchronize(ctx->copy_stream));
  for (auto &g : ctx->stage) {
    g.pending = false;
    pc_free(ctx, g.off);
    pc_free(ctx, g.nbr);
  }
  ctx->stage_fill = ctx->stage_commit = 0;
}

int pacim_load_graph(pacim_ctx *ctx, uint32_t n, uint64_t nnz, const uint64_t *offsets,
                     const uint32_t *neighbors, int pmodel, uint64_t t32, int validate) {
  return guarded(ctx, [&] {
    PC_REQUIRE(offsets && (neighbors || nnz == 0), PACIM_EINVAL, "NULL CSR array");
    PC_REQUIRE(n >= 1, PACIM_EINVAL, "n must be >= 1");
    PC_REQUIRE(offsets[0] == 0, PACIM_EINVAL, "offsets[0] != 0");
    PC_REQUIRE(offsets[n] == nnz, PACIM_EINVAL, "offsets[n] != nnz");
    drop_staged(ctx);
    pc_sym_free(ctx);  // the upper loads' scratch
    ctx->mi_valid = false;  // free device memory queried afresh (pc_mem_info)
    load_common(ctx, n, nnz, pmodel, t32);
    PC_CUDA(cudaMemcpyAsync(ctx->off.p, offsets, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice,
                            ctx->stream));
    if (nnz)
      PC_CUDA(cudaMemcpyAsync(ctx->nbr.p, neighbors, nnz * 4, cudaMemcpyHostToDevice, ctx->stream));
    pc_graph_finish_load(ctx, validate);
    ctx->has_graph = true;
  pc_graph_loaded(ctx);
  });
}

// enqueue the host -> device copies of a graph on the copy stream (committed
// by the next build): the symmetric CSR (nnz = 2m entries) or, upper, the
// upper CSR (nnz = m entries, symmetrized on the device at commit)
static void load_async(pacim_ctx *ctx, uint32_t n, uint64_t nnz, const uint64_t *offsets,
                       const uint32_t *neighbors, int pmodel, uint64_t t32, bool upper) {
  PC_REQUIRE(offsets && (neighbors || nnz == 0), PACIM_EINVAL, "NULL CSR array");
  PC_REQUIRE(n >= 1, PACIM_EINVAL, "n must be >= 1");
  PC_REQUIRE(n < (1u << 31), PACIM_EINVAL, "n must be < 2^31 (R2 key packing)");
  PC_REQUIRE(upper || (nnz & 1) == 0, PACIM_EINVAL, "nnz must be even (symmetric CSR)");
  PC_REQUIRE(offsets[0] == 0, PACIM_EINVAL, "offsets[0] != 0");
  PC_REQUIRE(offsets[n] == nnz, PACIM_EINVAL, upper ? "offsets[n] != m" : "offsets[n] != nnz");
  check_model(pmodel, t32);
  StagedGraph &st = ctx->stage[ctx->stage_fill];
  PC_REQUIRE(!st.pending, PACIM_ESTATE, "two graph loads are already pending");
  if (!ctx->copy_stream) {
    PC_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    PC_CUDA(cudaEventCreateWithFlags(&ctx->released, cudaEventDisableTiming));
    for (auto &g : ctx->stage) PC_CUDA(cudaEventCreateWithFlags(&g.done, cudaEventDisableTiming));
    PC_CUDA(cudaEventRecord(ctx->released, ctx->stream));
  }
  pc_ensure(ctx, st.off, ((size_t)n + 1) * 8);
  pc_ensure(ctx, st.nbr, std::max<uint64_t>(nnz, 1) * 4);
  // the slot's buffers may have been the graph before the last commit (or
  // the source of its symmetrization)
  PC_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->released, 0));
  PC_CUDA(cudaMemcpyAsync(st.off.p, offsets, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice,
                          ctx->copy_stream));
  if (nnz)
    PC_CUDA(cudaMemcpyAsync(st.nbr.p, neighbors, nnz * 4, cudaMemcpyHostToDevice,
                            ctx->copy_stream));
  PC_CUDA(cudaEventRecord(st.done, ctx->copy_stream));
  st.pending = true;
  st.upper = upper;
  st.n = n;
  st.nnz = upper ? 2 * nnz : nnz;
  st.pmodel = pmodel;
  st.t32 = t32;
  ctx->stage_fill ^= 1;
}

int pacim_load_graph_async(pacim_ctx *ctx, uint32_t n, uint64_t nnz, const uint64_t *offsets,
                           const uint32_t *neighbors, int pmodel, uint64_t t32) {
  return guarded(ctx, [&] { load_async(ctx, n, nnz, offsets, neighbors, pmodel, t32, false); });
}

int pacim_load_graph_upper_async(pacim_ctx *ctx, uint32_t n, uint64_t m, const uint64_t *uoffsets,
                                 const uint32_t *uneighbors, int pmodel, uint64_t t32) {
  return guarded(ctx, [&] { load_async(ctx, n, m, uoffsets, uneighbors, pmodel, t32, true); });
}

int pacim_load_graph_upper(pacim_ctx *ctx, uint32_t n, uint64_t m, const uint64_t *uoffsets,
                           const uint32_t *uneighbors, int pmodel, uint64_t t32, int validate) {
  return guarded(ctx, [&] {
    PC_REQUIRE(uoffsets && (uneighbors || m == 0), PACIM_EINVAL, "NULL CSR array");
    PC_REQUIRE(n >= 1, PACIM_EINVAL, "n must be >= 1");
    PC_REQUIRE(uoffsets[0] == 0, PACIM_EINVAL, "offsets[0] != 0");
    PC_REQUIRE(uoffsets[n] == m, PACIM_EINVAL, "offsets[n] != m");
    drop_staged(ctx);
    ctx->mi_valid = false;  // free device memory queried afresh (pc_mem_info)
    load_common(ctx, n, 2 * m, pmodel, t32, false);
    pc_ensure(ctx, ctx->uoff, ((size_t)n + 1) * 8);
    pc_ensure(ctx, ctx->unbr, std::max<uint64_t>(m, 1) * 4);
    PC_CUDA(cudaMemcpyAsync(ctx->uoff.p, uoffsets, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice,
                            ctx->stream));
    if (m)
      PC_CUDA(cudaMemcpyAsync(ctx->unbr.p, uneighbors, m * 4, cudaMemcpyHostToDevice, ctx->stream));
    if (validate) pc_validate_upper(ctx, ctx->uoff.as<uint64_t>(), ctx->unbr.as<uint32_t>(), n);
    pc_upper_degrees(ctx);
    pc_graph_finish_load(ctx, 0);
    ctx->has_graph = true;
    pc_graph_loaded(ctx);
  });
}

int pacim_load_graph_device(pacim_ctx *ctx, uint32_t n, uint64_t nnz, const uint64_t *d_offsets,
                            const uint32_t *d_neighbors, int pmodel, uint64_t t32, int validate) {
  return guarded(ctx, [&] {
    PC_REQUIRE(d_offsets && (d_neighbors || nnz == 0), PACIM_EINVAL, "NULL CSR array");
    drop_staged(ctx);
    ctx->mi_valid = false;  // free device memory queried afresh (pc_mem_info)
    load_common(ctx, n, nnz, pmodel, t32);
    PC_CUDA(cudaMemcpyAsync(ctx->off.p, d_offsets, ((size_t)n + 1) * 8, cudaMemcpyDeviceToDevice,
                            ctx->stream));
    if (nnz)
      PC_CUDA(cudaMemcpyAsync(ctx->nbr.p, d_neighbors, nnz * 4, cudaMemcpyDeviceToDevice,
                              ctx->stream));
    uint64_t ends[2];
    PC_CUDA(cudaMemcpyAsync(&ends[0], ctx->off.as<uint64_t>(), 8, cudaMemcpyDeviceToHost,
                            ctx->stream));
    PC_CUDA(cudaMemcpyAsync(&ends[1], ctx->off.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost,
                            ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    PC_REQUIRE(ends[0] == 0, PACIM_EINVAL, "offsets[0] != 0");
    PC_REQUIRE(ends[1] == nnz, PACIM_EINVAL, "offsets[n] != nnz");
    pc_graph_finish_load(ctx, validate);
    ctx->has_graph = true;
  pc_graph_loaded(ctx);
  });
}

int pacim_generate_graph(pacim_ctx *ctx, int kind, const uint64_t *params, int nparams,
                         uint64_t gen_seed, int pmodel, uint64_t t32) {
  return guarded(ctx, [&] {
    PC_REQUIRE(params || nparams == 0, PACIM_EINVAL, "NULL params");
    check_model(pmodel, t32);
    drop_staged(ctx);
    ctx->mi_valid = false;  // free device memory queried afresh (pc_mem_info)
    drop_graph(ctx);
    ctx->pmodel = pmodel;
    ctx->t32 = t32;
    pc_generate(ctx, kind, params, nparams, gen_seed);
    ctx->has_graph = true;
  pc_graph_loaded(ctx);
  });
}

int pacim_graph_info(pacim_ctx *ctx, uint32_t *n, uint64_t *m) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->has_graph, PACIM_ESTATE, "no graph loaded");
    if (n) *n = ctx->n;
    if (m) *m = ctx->m;
  });
}

int pacim_get_graph(pacim_ctx *ctx, uint64_t *offsets_out, uint32_t *neighbors_out) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->has_graph, PACIM_ESTATE, "no graph loaded");
    if (neighbors_out) pc_ensure_sym(ctx);
    if (offsets_out)
      PC_CUDA(cudaMemcpyAsync(offsets_out, ctx->off.p, ((size_t)ctx->n + 1) * 8,
                              cudaMemcpyDeviceToHost, ctx->stream));
    if (neighbors_out && ctx->m)
      PC_CUDA(cudaMemcpyAsync(neighbors_out, ctx->nbr.p, 2 * ctx->m * 4, cudaMemcpyDeviceToHost,
                              ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int pacim_build_sketches(pacim_ctx *ctx, uint32_t R, uint64_t hash_seed, uint64_t center_a32,
                         uint32_t shard_rank, uint32_t shard_world) {
  return guarded(ctx, [&] {
    commit_staged(ctx);
    PC_REQUIRE(ctx->has_graph, PACIM_ESTATE, "build before load_graph");
    PC_REQUIRE(R >= 1, PACIM_EINVAL, "R must be >= 1");
    PC_REQUIRE(shard_world >= 1 && shard_rank < shard_world, PACIM_EINVAL,
               "need 0 <= shard_rank < shard_world");
    PC_REQUIRE(shard_rank < R, PACIM_EINVAL, "shard holds no sketch (shard_rank >= R)");
    drop_sketches(ctx);
    ctx->device_peak = ctx->device_bytes;  // high-water mark of this build + select

    ctx->R = R;
    ctx->rank = shard_rank;
    ctx->world = shard_world;
    ctx->R_local = (R - shard_rank + shard_world - 1) / shard_world;
    ctx->hash_seed = hash_seed;
    ctx->K = pc_mix64(hash_seed);  // R2
    ctx->a32 = center_a32;
    ctx->compressed = center_a32 < (1ull << 32);
    if (ctx->compressed)
      pc_build_compressed(ctx);
    else
      pc_build(ctx);
    pc_dist_build_finish(ctx);  // sharded with a communicator: gain0 all-reduced
    ctx->built = true;
  });
}

int pacim_select_seeds(pacim_ctx *ctx, uint32_t k, uint32_t *seeds_out, int64_t *gain_num_out,
                       int64_t *sigma_num_out, double *sigma_out) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->built, PACIM_ESTATE, "select before build_sketches");
    PC_REQUIRE(k >= 1 && k <= ctx->n, PACIM_EINVAL, "k must be in [1, n]");
    PC_REQUIRE(seeds_out && gain_num_out && sigma_num_out, PACIM_EINVAL, "NULL output");
    if (ctx->world > 1 || pc_dist_active(ctx)) {
      // sharded build: the greedy loop over NCCL (dist.cu); without a
      // communicator the per-rank step primitives remain (dist.py)
      pc_dist_select(ctx, k, seeds_out, gain_num_out);
      int64_t run = 0;
      for (uint32_t i = 0; i < k; i++) sigma_num_out[i] = run += gain_num_out[i];
    } else if (ctx->compressed) {
      pc_select_compressed(ctx, k, seeds_out, gain_num_out, sigma_num_out);
    } else {
      // selector 3 (auto): the Win-Tree under WIC (a few re-evaluations per
      // step: c4 needs ~1.5), else the incremental selector
      // (constant / uniform p on social graphs re-evaluate ~n vertices)
      const int sel = ctx->selector == 3 ? (ctx->pmodel == PACIM_P_WIC ? 2 : 0) : ctx->selector;
      if (sel == 2 && ctx->cs)
        pc_cs_select_wintree(ctx, k, seeds_out, gain_num_out, sigma_num_out);
      else if (sel == 2)
        pc_select_wintree_dense(ctx, k, seeds_out, gain_num_out, sigma_num_out);
      else if (sel == 1)
        pc_select_lazy(ctx, k, seeds_out, gain_num_out, sigma_num_out);
      else
        pc_select(ctx, k, seeds_out, gain_num_out, sigma_num_out);
    }
    if (sigma_out)
      for (uint32_t i = 0; i < k; i++) sigma_out[i] = (double)sigma_num_out[i] / (double)ctx->R;
  });
}

int pacim_gain0_to_device(pacim_ctx *ctx, int64_t *d_out) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->built, PACIM_ESTATE, "no sketches");
    PC_REQUIRE(d_out, PACIM_EINVAL, "NULL output");
    PC_CUDA(cudaMemcpyAsync(d_out, ctx->gain0.p, (size_t)ctx->n * 8, cudaMemcpyDeviceToDevice,
                            ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int pacim_select_reset(pacim_ctx *ctx) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->built, PACIM_ESTATE, "no sketches");
    if (ctx->compressed)
      pc_select_reset_compressed(ctx);
    else
      pc_select_reset(ctx);
  });
}

int pacim_cover_local(pacim_ctx *ctx, uint32_t s, int64_t *d_delta, int64_t *local_gain) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->built, PACIM_ESTATE, "no sketches");
    PC_REQUIRE(s < ctx->n && d_delta && local_gain, PACIM_EINVAL, "bad argument");
    if (ctx->compressed) {
      pc_cover_compressed(ctx, s, d_delta, local_gain);
      PC_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
      pc_cover_local(ctx, s, d_delta, local_gain);
    }
  });
}

int pacim_cover_local_sparse(pacim_ctx *ctx, uint32_t s, int64_t *d_delta, uint32_t *d_list_v,
                             int64_t *d_list_d, uint64_t cap, uint64_t *count,
                             int64_t *local_gain) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->built, PACIM_ESTATE, "no sketches");
    PC_REQUIRE(s < ctx->n && d_delta && local_gain && count && d_list_v && d_list_d,
               PACIM_EINVAL, "bad argument");
    // the list counter lives in the ctx (reset per call)
    pc_ensure(ctx, ctx->sel_flag, 64);
    unsigned long long *cnt = ctx->sel_flag.as<unsigned long long>() + 4;
    PC_CUDA(cudaMemsetAsync(cnt, 0, 8, ctx->stream));
    ctx->dlist.v = d_list_v;
    ctx->dlist.d = reinterpret_cast<long long *>(d_list_d);
    ctx->dlist.cnt = cnt;
    ctx->dlist.cap = cap;
    try {
      if (ctx->compressed) {
        pc_cover_compressed(ctx, s, d_delta, local_gain);
        PC_CUDA(cudaStreamSynchronize(ctx->stream));
      } else {
        pc_cover_local(ctx, s, d_delta, local_gain);
      }
    } catch (...) {
      ctx->dlist = DeltaList{};
      throw;
    }
    ctx->dlist = DeltaList{};
    unsigned long long h = 0;
    PC_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
    *count = h;
  });
}

int pacim_simulate_ic(pacim_ctx *ctx, const uint32_t *seeds, uint32_t ns, uint32_t nsims,
                      uint64_t mc_seed, uint64_t *total) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->has_graph, PACIM_ESTATE, "simulate before a graph is loaded");
    PC_REQUIRE(total && (ns == 0 || seeds), PACIM_EINVAL, "bad argument");
    pc_simulate_ic(ctx, seeds, ns, nsims, mc_seed, total);
  });
}

int pacim_set_selector(pacim_ctx *ctx, int selector) {
  return guarded(ctx, [&] {
    PC_REQUIRE(selector >= 0 && selector <= 3, PACIM_EINVAL,
               "selector must be 0 (incremental), 1 (prefix doubling), 2 (Win-Tree) or 3 (auto)");
    ctx->selector = selector;
  });
}

int pacim_set_hash_rule(pacim_ctx *ctx, int rule) {
  return guarded(ctx, [&] {
    PC_REQUIRE(rule == 0 || rule == 1, PACIM_EINVAL, "hash rule must be 0 (P:3-4) or 1 (R20)");
    if (rule != ctx->hash_rule) drop_sketches(ctx);
    ctx->hash_rule = rule;
  });
}

int pacim_apply_deltas(pacim_ctx *ctx, int64_t *d_gain, const uint32_t *d_v, const int64_t *d_d,
                       uint64_t count, uint32_t s) {
  return guarded(ctx, [&] {
    PC_REQUIRE(d_gain && (count == 0 || (d_v && d_d)), PACIM_EINVAL, "bad argument");
    pc_apply_deltas(ctx, d_gain, d_v, d_d, count, s);
  });
}

int pacim_apply_dense(pacim_ctx *ctx, int64_t *d_gain, int64_t *d_delta, uint32_t n, uint32_t s) {
  return guarded(ctx, [&] {
    PC_REQUIRE(d_gain && d_delta && n >= 1, PACIM_EINVAL, "bad argument");
    pc_apply_dense(ctx, d_gain, d_delta, n, s);
  });
}

int pacim_clear_deltas(pacim_ctx *ctx, int64_t *d_delta, const uint32_t *d_v, uint64_t count) {
  return guarded(ctx, [&] {
    PC_REQUIRE(d_delta && (count == 0 || d_v), PACIM_EINVAL, "bad argument");
    pc_clear_deltas(ctx, d_delta, d_v, count);
  });
}

int pacim_argmax_device(pacim_ctx *ctx, const int64_t *d_gain, uint32_t n, uint32_t *s_out,
                        int64_t *g_out) {
  return guarded(ctx, [&] {
    PC_REQUIRE(d_gain && s_out && g_out && n >= 1, PACIM_EINVAL, "bad argument");
    pc_argmax(ctx, d_gain, n, s_out, g_out);
  });
}

int pacim_get_gain0(pacim_ctx *ctx, int64_t *out) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->built, PACIM_ESTATE, "no sketches");
    PC_REQUIRE(out, PACIM_EINVAL, "NULL output");
    PC_CUDA(cudaMemcpyAsync(out, ctx->gain0.p, (size_t)ctx->n * 8, cudaMemcpyDeviceToHost,
                            ctx->stream));
    PC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int pacim_get_labels(pacim_ctx *ctx, uint32_t r, uint32_t *out) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->built, PACIM_ESTATE, "no sketches");
    PC_REQUIRE(!ctx->compressed, PACIM_ENOTIMPL, "labels are not stored in compressed mode");
    PC_REQUIRE(out && r < ctx->R && ctx->r_slot[r] >= 0, PACIM_EINVAL,
               "sketch r is not held by this ctx");
    pc_get_labels(ctx, (uint32_t)ctx->r_slot[r], out);
  });
}

int pacim_get_center_sketch(pacim_ctx *ctx, uint32_t r, uint32_t *label_out, uint32_t *size_out) {
  return guarded(ctx, [&] {
    PC_REQUIRE(ctx->built, PACIM_ESTATE, "no sketches");
    PC_REQUIRE(ctx->compressed, PACIM_ESTATE, "not a compressed store");
    (void)r;
    (void)label_out;
    (void)size_out;
    PC_REQUIRE(label_out && size_out && r < ctx->R && ctx->r_slot[r] >= 0, PACIM_EINVAL,
               "sketch r is not held by this ctx");
    pc_get_center_sketch(ctx, (uint32_t)ctx->r_slot[r], label_out, size_out);
  });
}

int pacim_get_stats(pacim_ctx *ctx, pacim_stats *out) {
  return guarded(ctx, [&] {
    PC_REQUIRE(out, PACIM_EINVAL, "NULL output");
    pacim_stats s = ctx->stats;
    s.n = ctx->n;
    s.m = ctx->m;
    s.R = ctx->R;
    s.R_local = ctx->R_local;
    s.rho = ctx->compressed ? ctx->rho : ctx->n;
    s.compressed = ctx->compressed ? 1 : 0;
    s.ncomp = ctx->ncomp;
    s.nmember = ctx->nmember;
    s.rows = ctx->nr;
    s.batch_slots = ctx->compressed ? ctx->Bb : 0;
    s.hla_entries = ctx->hla_ok ? ctx->hla_n : 0;
    s.hubs = ctx->nhub;
    s.lean = ctx->lean ? 1u : 0u;
    s.store = ctx->compressed ? 2u : (ctx->cs ? 1u : 0u);
    s.nnonsingle = ctx->nnonsingle;
    s.device_bytes = ctx->device_bytes;
    s.device_peak_bytes = ctx->device_peak;
    *out = s;
  });
}

}  // extern "C"
