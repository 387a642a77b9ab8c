// capi.cu -- the extern "C" boundary of libbgmf.so (declared in
// include/bgmf.h).  Host-side orchestration only; kernels live in
// partition.cu / sgd.cu / eval.cu.

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>

#include "bgmf_internal.cuh"

namespace bgmf {

thread_local std::string g_err;  // errors of calls without a context

int fail(bgmf_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg; else g_err = msg;
  return code;
}

int cuda_fail(bgmf_ctx* ctx, cudaError_t e, const char* what) {
  std::string msg = std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                    cudaGetErrorString(e) + ") in " + what;
  cudaGetLastError();  // clear sticky-free errors
  return fail(ctx, e == cudaErrorMemoryAllocation ? BGMF_ERR_NOMEM : BGMF_ERR_CUDA, msg);
}

void prof_mark(bgmf_ctx* c, const char* what) {
  const bool on = getenv("BGMF_PROFILE") != nullptr;
  if (!on) return;
  static thread_local std::chrono::steady_clock::time_point last;
  if (c && c->stream) cudaStreamSynchronize(c->stream);
  const auto now = std::chrono::steady_clock::now();
  if (what)
    fprintf(stderr, "[bgmf]   %-30s %9.2f ms\n", what,
            std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

void record_begin(bgmf_ctx* c, int kind, double bytes, TimedLaunch** slot) {
  if (c->events_used == c->events.size()) {
    TimedLaunch t;
    cudaEventCreate(&t.a);
    cudaEventCreate(&t.b);
    c->events.push_back(t);
  }
  TimedLaunch* t = &c->events[c->events_used++];
  t->kind = kind;
  t->bytes = bytes;
  cudaEventRecord(t->a, c->stream);
  *slot = t;
}

void record_end(bgmf_ctx* c, TimedLaunch* slot) { cudaEventRecord(slot->b, c->stream); }

void harvest_timing(bgmf_ctx* c) {
  for (size_t i = 0; i < c->events_used; ++i) {
    TimedLaunch& t = c->events[i];
    float ms = 0.f;
    cudaEventSynchronize(t.b);
    cudaEventElapsedTime(&ms, t.a, t.b);
    if (t.kind == 0) { c->t_sgd_ms += ms; c->n_sgd++; c->t_bytes += t.bytes; }
    else { c->t_sse_ms += ms; c->n_sse++; }
  }
  c->events_used = 0;
}

namespace {

void free_factors(bgmf_ctx* c) {
  if (!c->bound) {
    if (c->d_u) dfree(c->d_u, c->stream);
    if (c->d_v) dfree(c->d_v, c->stream);
  }
  if (c->d_u64) dfree(c->d_u64, c->stream);
  if (c->d_v64) dfree(c->d_v64, c->stream);
  c->d_u = c->d_v = nullptr;
  c->d_u64 = c->d_v64 = nullptr;
  c->bound = false;
  c->have_factors = false;
}

void free_holdout(bgmf_ctx* c) {
  if (c->d_hrow) dfree(c->d_hrow, c->stream);
  if (c->d_hcol) dfree(c->d_hcol, c->stream);
  if (c->d_hval) dfree(c->d_hval, c->stream);
  if (c->d_hval64) dfree(c->d_hval64, c->stream);
  if (c->d_hcold) dfree(c->d_hcold, c->stream);
  c->d_hrow = c->d_hcol = nullptr;
  c->d_hval = nullptr;
  c->d_hval64 = nullptr;
  c->d_hcold = nullptr;
  c->hcount = 0;
}

int check_step_ready(bgmf_ctx* c) {
  if (!c->partitioned) return fail(c, BGMF_ERR_STATE, "bgmf_partition has not been called");
  if (!c->have_factors) return fail(c, BGMF_ERR_STATE, "bgmf_set_factors has not been called");
  if (c->exact && (!c->d_val64 || !c->d_u64))
    return fail(c, BGMF_ERR_STATE, "exact mode must be enabled before partition and set_factors");
  if (!c->exact && !c->d_u) return fail(c, BGMF_ERR_STATE, "fast-mode factors missing");
  return BGMF_OK;
}

void fill_bad(bgmf_ctx* c, int64_t* bad_out) {
  const unsigned long long b = *c->h_bad;
  if (b == kNoBad) {
    bad_out[0] = bad_out[1] = bad_out[2] = -1;
  } else {
    bad_out[0] = (int64_t)(b >> 48);
    bad_out[1] = (int64_t)(b & 0xFFFFFFFFull);
    bad_out[2] = (int64_t)((b >> 32) & 0xFFFF);
  }
}

// Per-thread scratch context for the stateless drop-in entry points.
bgmf_ctx* scratch_ctx(int* rc) {
  thread_local std::unique_ptr<bgmf_ctx, void (*)(bgmf_ctx*)> ctx(nullptr, bgmf_destroy);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) { *rc = cuda_fail(nullptr, e, "cudaGetDevice"); return nullptr; }
  if (!ctx || ctx->device != dev) {
    bgmf_ctx* c = nullptr;
    *rc = bgmf_create(dev, nullptr, &c);
    if (*rc) return nullptr;
    ctx.reset(c);
  }
  *rc = BGMF_OK;
  return ctx.get();
}

}  // namespace
}  // namespace bgmf

using namespace bgmf;

extern "C" {

int bgmf_version(void) { return 100; }

int bgmf_create(int device, void* stream, bgmf_ctx** out) {
  if (!out) return fail(nullptr, BGMF_ERR_ARG, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(nullptr, BGMF_ERR_ARG, "no such CUDA device");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
  {  // keep freed device memory in the pool (see dmalloc)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  auto* c = new bgmf_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete c; return cuda_fail(nullptr, e, "cudaStreamCreate"); }
    c->own_stream = true;
  }
  *out = c;
  return BGMF_OK;
}

void bgmf_destroy(bgmf_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  prof_mark(c, nullptr);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (int h = 0; h < 2; ++h)
    if (c->ws_done[h]) cudaEventDestroy(c->ws_done[h]);
  peer_release(c);
  prof_mark(c, "destroy: sync");
  free_factors(c);
  free_holdout(c);
  stream_free(c);
  order_release(c);
  prof_mark(c, "destroy: factors/holdout/stream");
  dfree(c->d_lrow, c->stream); dfree(c->d_lcol, c->stream); dfree(c->d_val, c->stream); dfree(c->d_val64, c->stream);
  dfree(c->d_order, c->stream); dfree(c->d_fuse, c->stream); dfree(c->d_cstate, c->stream); conv_graphs_release(c); dfree(c->d_sse, c->stream); dfree(c->d_bad, c->stream); dfree(c->d_work, c->stream);
  dfree(c->d_partials, c->stream);
  dfree(c->d_priv, c->stream);
  cudaStreamSynchronize(c->stream);
  if (c->d_dyn) cudaFree(c->d_dyn);
  prof_mark(c, "destroy: device frees");
  pinned_free(c->h_work);
  pinned_free(c->h_sse);
  pinned_free(c->h_bad);
  prof_mark(nullptr, "destroy: pinned frees");
  for (auto& t : c->events) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* bgmf_last_error(const bgmf_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

int bgmf_set_option(bgmf_ctx* c, const char* key, double value) {
  if (!c || !key) return fail(c, BGMF_ERR_ARG, "NULL argument");
  if (!strcmp(key, "exact")) c->exact = value != 0.0;
  else if (!strcmp(key, "min_chunk")) c->min_chunk = value < 1 ? 1 : (int)value;
  else if (!strcmp(key, "timing")) c->timing = value != 0.0;
  else if (!strcmp(key, "warps_per_sm")) c->warps_per_sm = value < 0 ? 0 : (int)value;
  else if (!strcmp(key, "fused")) c->fused = value < 0 ? -1 : (value != 0.0 ? 1 : 0);
  else if (!strcmp(key, "bulk_red")) c->bulk_red = value != 0.0;
  else if (!strcmp(key, "sse_wide")) c->sse_wide = value != 0.0;
  else if (!strcmp(key, "sse_async")) c->sse_async = value != 0.0;
  else if (!strcmp(key, "stagger")) c->stagger = (int)value;
  else if (!strcmp(key, "sparse_min_chunk")) c->sparse_min_chunk = value < 0 ? 0 : (int)value;
  else if (!strcmp(key, "col_ratio")) c->col_ratio = value > 0 ? value : 0.6;
  else if (!strcmp(key, "ordered")) c->ord_mode = value < 0 ? -1 : (value != 0.0 ? 1 : 0);
  else if (!strcmp(key, "ord_row_split")) c->ord_row_split = value;
  else if (!strcmp(key, "no_val8")) c->no_val8 = value != 0.0;
  else if (!strcmp(key, "fuse_sse")) c->fuse_sse = value != 0.0;
  else if (!strcmp(key, "u_ring")) c->u_ring = value < 0.0 ? -1 : (value != 0.0 ? 1 : 0);
  else if (!strcmp(key, "u_prefetch")) { c->u_prefetch = value < 0.0 ? -1 : value != 0.0; c->upf_key = -1; }
  else if (!strcmp(key, "spread")) c->spread = value != 0.0;
  else if (!strcmp(key, "nt_download")) c->nt_download = value != 0.0;
  else if (!strcmp(key, "snap")) c->snap_cap = value < 0.0 ? 0 : value > 4096.0 ? 4096 : (int)value;
  else if (!strcmp(key, "dyn_split")) {
    c->dyn_split = value < 1.0 ? 1 : value > 16.0 ? 16 : (int)value;
    if (c->dyn_split > 1 && !c->d_dyn) {  // the ticket counters, zeroed once
      cudaSetDevice(c->device);
      cudaError_t e = cudaMalloc(&c->d_dyn, 2 * sizeof(unsigned));
      if (e == cudaSuccess) e = cudaMemset(c->d_dyn, 0, 2 * sizeof(unsigned));
      if (e != cudaSuccess) { c->dyn_split = 1; return cuda_fail(c, e, "dyn_split counters"); }
    }
  }
  else if (!strcmp(key, "pdl")) c->pdl = value != 0.0;
  else if (!strcmp(key, "conv_graph")) c->conv_graph = value != 0.0;
  else if (!strcmp(key, "ord_col_conc")) c->ord_col_conc = value;
  else if (!strcmp(key, "ord_fill_ctas")) c->ord_fill_ctas = value < 1 ? 1 : (int)value;
  else if (!strcmp(key, "ord_warp")) c->ord_warp = value != 0.0;
  else if (!strcmp(key, "ord_stage_ratings"))
    c->ord_stage_ratings = value < 1 ? 1 : (int64_t)value;
  else if (!strcmp(key, "l2_wave_bytes")) c->l2_wave_bytes = value < 0 ? 0 : (int64_t)value;
  else if (!strcmp(key, "fused_max_batch")) c->fused_max_batch = (int64_t)value;
  else return fail(c, BGMF_ERR_ARG, std::string("unknown option ") + key);
  return BGMF_OK;
}

int bgmf_partition(bgmf_ctx* c, const int64_t* rows, const int64_t* cols, const double* vals,
                   int64_t nnz, int64_t n, int64_t m, int grid_i, int grid_j) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  cudaSetDevice(c->device);
  if (c->streaming) stream_free(c);
  // the step scratch is sized by the grid
  dfree(c->d_sse, c->stream); pinned_free(c->h_sse); dfree(c->d_fuse, c->stream); c->d_fuse = nullptr; dfree(c->d_cstate, c->stream); c->d_cstate = nullptr; c->cstate_cap = 0; conv_graphs_release(c); dfree(c->d_bad, c->stream); pinned_free(c->h_bad);
  c->d_sse = nullptr; c->h_sse = nullptr; c->d_bad = nullptr; c->h_bad = nullptr;
  return partition_device(c, rows, cols, vals, nnz, n, m, grid_i, grid_j);
}

int bgmf_partition_rows(bgmf_ctx* c, const int64_t* rows, const int64_t* cols,
                        const double* vals, int64_t nnz, int64_t n, int64_t m, int grid_i,
                        int grid_j, int64_t row_lo, int64_t row_hi) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  cudaSetDevice(c->device);
  if (c->streaming) stream_free(c);
  dfree(c->d_sse, c->stream); pinned_free(c->h_sse); dfree(c->d_fuse, c->stream); c->d_fuse = nullptr; dfree(c->d_cstate, c->stream); c->d_cstate = nullptr; c->cstate_cap = 0; conv_graphs_release(c); dfree(c->d_bad, c->stream); pinned_free(c->h_bad);
  c->d_sse = nullptr; c->h_sse = nullptr; c->d_bad = nullptr; c->h_bad = nullptr;
  return partition_device(c, rows, cols, vals, nnz, n, m, grid_i, grid_j, false, row_lo, row_hi);
}

int bgmf_synth_partition(bgmf_ctx* c, int64_t n, int64_t m, int64_t nnz, uint64_t seed,
                         int grid_i, int grid_j) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (n < 1 || m < 1 || nnz < 0 || (uint64_t)nnz > (uint64_t)n * (uint64_t)m)
    return fail(c, BGMF_ERR_ARG, "bad synthetic shape");
  cudaSetDevice(c->device);
  if (c->streaming) stream_free(c);
  dfree(c->d_sse, c->stream); pinned_free(c->h_sse); dfree(c->d_fuse, c->stream); c->d_fuse = nullptr; dfree(c->d_cstate, c->stream); c->d_cstate = nullptr; c->cstate_cap = 0; conv_graphs_release(c); dfree(c->d_bad, c->stream); pinned_free(c->h_bad);
  c->d_sse = nullptr; c->h_sse = nullptr; c->d_bad = nullptr; c->h_bad = nullptr;
  const size_t N = (size_t)(nnz > 0 ? nnz : 1);
  int64_t *r = nullptr, *q = nullptr;
  double* v = nullptr;
  cudaError_t e = dmalloc(&r, N * 8, c->stream);
  if (e == cudaSuccess) e = dmalloc(&q, N * 8, c->stream);
  if (e == cudaSuccess) e = dmalloc(&v, N * 8, c->stream);
  if (e != cudaSuccess) { dfree(r, c->stream); dfree(q, c->stream); dfree(v, c->stream); return cuda_fail(c, e, "synth alloc"); }
  int rc = synth_lowrank_device(c, n, m, nnz, 0, seed, r, q, v);
  if (rc) { dfree(r, c->stream); dfree(q, c->stream); dfree(v, c->stream); return rc; }
  return partition_device(c, r, q, v, nnz, n, m, grid_i, grid_j, /*dev_in=*/true);
}

int bgmf_synth(int64_t n, int64_t m, int64_t nnz, int64_t start, uint64_t seed, int64_t* rows,
               int64_t* cols, double* vals) {
  int rc;
  bgmf_ctx* c = scratch_ctx(&rc);
  if (!c) return rc;
  if (nnz <= 0) return BGMF_OK;
  int64_t *r = nullptr, *q = nullptr;
  double* v = nullptr;
  cudaError_t e = dmalloc(&r, nnz * 8, c->stream);
  if (e == cudaSuccess) e = dmalloc(&q, nnz * 8, c->stream);
  if (e == cudaSuccess) e = dmalloc(&v, nnz * 8, c->stream);
  if (e == cudaSuccess) {
    rc = synth_lowrank_device(c, n, m, nnz, start, seed, r, q, v);
    if (!rc) {
      e = cudaMemcpy(rows, r, nnz * 8, cudaMemcpyDeviceToHost);
      if (e == cudaSuccess) e = cudaMemcpy(cols, q, nnz * 8, cudaMemcpyDeviceToHost);
      if (e == cudaSuccess) e = cudaMemcpy(vals, v, nnz * 8, cudaMemcpyDeviceToHost);
    }
  }
  dfree(r, c->stream); dfree(q, c->stream); dfree(v, c->stream);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "bgmf_synth");
  if (rc) { g_err = c->err; return rc; }
  return BGMF_OK;
}

int bgmf_partition_export(bgmf_ctx* c, int64_t* offsets, int64_t* order, int32_t* lrows,
                          int32_t* lcols) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (!c->partitioned) return fail(c, BGMF_ERR_STATE, "bgmf_partition has not been called");
  cudaSetDevice(c->device);
  if (offsets) memcpy(offsets, c->h_offsets.data(), c->h_offsets.size() * 8);
  const int64_t n = c->nnz;
  if (n == 0) return BGMF_OK;
  if (c->streaming) return stream_export(c, order, lrows, lcols);  // pinned host copy
  if (lrows) BGMF_CK(c, cudaMemcpyAsync(lrows, c->d_lrow, n * 4, cudaMemcpyDeviceToHost, c->stream));
  if (lcols) BGMF_CK(c, cudaMemcpyAsync(lcols, c->d_lcol, n * 4, cudaMemcpyDeviceToHost, c->stream));
  if (order) {
    std::vector<uint32_t> o((size_t)n);
    BGMF_CK(c, cudaMemcpyAsync(o.data(), c->d_order, n * 4, cudaMemcpyDeviceToHost, c->stream));
    BGMF_CK(c, cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < n; ++i) order[i] = (int64_t)o[i];
  }
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  return BGMF_OK;
}

int bgmf_release_host_cache(void) {
  big_pinned_trim();
  return BGMF_OK;
}

int bgmf_partition_values(bgmf_ctx* c, double* vals) {
  if (!c || !vals) return fail(c, BGMF_ERR_ARG, "ctx or vals is NULL");
  if (!c->partitioned) return fail(c, BGMF_ERR_STATE, "bgmf_partition has not been called");
  if (c->streaming) return fail(c, BGMF_ERR_STATE, "the ratings stream from host memory");
  cudaSetDevice(c->device);
  const int64_t n = c->nnz;
  if (n == 0) return BGMF_OK;
  if (c->d_val64) {
    BGMF_CK(c, cudaMemcpyAsync(vals, c->d_val64, n * 8, cudaMemcpyDeviceToHost, c->stream));
    BGMF_CK(c, cudaStreamSynchronize(c->stream));
    return BGMF_OK;
  }
  std::vector<float> f((size_t)n);
  BGMF_CK(c, cudaMemcpyAsync(f.data(), c->d_val, n * 4, cudaMemcpyDeviceToHost, c->stream));
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  for (int64_t i = 0; i < n; ++i) vals[i] = (double)f[i];
  return BGMF_OK;
}

int bgmf_set_factors(bgmf_ctx* c, const double* u, const double* v, int64_t n, int64_t m, int k) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (!u || !v || k < 1 || n < 1 || m < 1) return fail(c, BGMF_ERR_ARG, "bad factor arguments");
  if (c->partitioned && (n != c->n || m != c->m))
    return fail(c, BGMF_ERR_ARG, "factor shapes do not match the partitioned dataset");
  cudaSetDevice(c->device);
  if (c->exact) {
    free_factors(c);
    c->k = k; c->kp = k;
    BGMF_CK(c, dmalloc(&c->d_u64, (size_t)n * k * 8, c->stream));
    BGMF_CK(c, dmalloc(&c->d_v64, (size_t)m * k * 8, c->stream));
    BGMF_CK(c, cudaMemcpyAsync(c->d_u64, u, (size_t)n * k * 8, cudaMemcpyHostToDevice, c->stream));
    BGMF_CK(c, cudaMemcpyAsync(c->d_v64, v, (size_t)m * k * 8, cudaMemcpyHostToDevice, c->stream));
    BGMF_CK(c, cudaStreamSynchronize(c->stream));
    c->have_factors = true;
    return BGMF_OK;
  }
  const int kp = (k + 3) / 4 * 4;
  if (kp > 512) return fail(c, BGMF_ERR_ARG, "fast mode supports k <= 512 (use exact mode)");
  if (!(c->bound && c->k == k)) {
    free_factors(c);
    c->k = k; c->kp = kp;
    BGMF_CK(c, dmalloc(&c->d_u, (size_t)n * kp * 4, c->stream));
    BGMF_CK(c, dmalloc(&c->d_v, (size_t)m * kp * 4, c->stream));
  }
  int rc = upload_rows(c, u, c->d_u, n, k, c->kp);
  if (!rc) rc = upload_rows(c, v, c->d_v, m, k, c->kp);
  if (rc) return rc;
  c->have_factors = true;
  return BGMF_OK;
}

int bgmf_init_factors(bgmf_ctx* c, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                      uint64_t inc_lo, int64_t n, int64_t m, int k) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (k < 1 || n < 1 || m < 1) return fail(c, BGMF_ERR_ARG, "n, m, k must all be >= 1");
  if (c->partitioned && (n != c->n || m != c->m))
    return fail(c, BGMF_ERR_ARG, "factor shapes do not match the partitioned dataset");
  cudaSetDevice(c->device);
  if (c->exact) {
    free_factors(c);
    c->k = k; c->kp = k;
    BGMF_CK(c, dmalloc(&c->d_u64, (size_t)n * k * 8, c->stream));
    BGMF_CK(c, dmalloc(&c->d_v64, (size_t)m * k * 8, c->stream));
  } else {
    const int kp = (k + 3) / 4 * 4;
    if (kp > 512) return fail(c, BGMF_ERR_ARG, "fast mode supports k <= 512 (use exact mode)");
    if (!(c->bound && c->k == k)) {
      free_factors(c);
      c->k = k; c->kp = kp;
      BGMF_CK(c, dmalloc(&c->d_u, (size_t)n * kp * 4, c->stream));
      BGMF_CK(c, dmalloc(&c->d_v, (size_t)m * kp * 4, c->stream));
    }
  }
  int rc = init_factors_device(c, state_hi, state_lo, inc_hi, inc_lo, n, m, k);
  if (rc) return rc;
  c->have_factors = true;
  return BGMF_OK;
}

int bgmf_bind_factors(bgmf_ctx* c, void* u_dev, void* v_dev, int64_t n, int64_t m, int k, int kp) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (c->exact) return fail(c, BGMF_ERR_STATE, "bind_factors is fast-mode only");
  if (!u_dev || !v_dev || k < 1 || kp < k || kp % 4 || kp > 512)
    return fail(c, BGMF_ERR_ARG, "bad bind (need k <= kp <= 512, kp % 4 == 0)");
  if (((uintptr_t)u_dev | (uintptr_t)v_dev) & 15) return fail(c, BGMF_ERR_ARG, "unaligned factors");
  if (c->partitioned && (n != c->n || m != c->m))
    return fail(c, BGMF_ERR_ARG, "factor shapes do not match the partitioned dataset");
  free_factors(c);
  c->d_u = (float*)u_dev;
  c->d_v = (float*)v_dev;
  c->k = k; c->kp = kp;
  c->bound = true;
  c->have_factors = true;
  return BGMF_OK;
}

int bgmf_get_factors(bgmf_ctx* c, double* u, double* v) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (!c->have_factors) return fail(c, BGMF_ERR_STATE, "no factors on the device");
  cudaSetDevice(c->device);
  const int64_t n = c->n, m = c->m;
  if (c->exact) {
    if (u) BGMF_CK(c, cudaMemcpyAsync(u, c->d_u64, (size_t)n * c->k * 8, cudaMemcpyDeviceToHost, c->stream));
    if (v) BGMF_CK(c, cudaMemcpyAsync(v, c->d_v64, (size_t)m * c->k * 8, cudaMemcpyDeviceToHost, c->stream));
    BGMF_CK(c, cudaStreamSynchronize(c->stream));
    return BGMF_OK;
  }
  int rc = BGMF_OK;
  if (u) rc = download_rows(c, c->d_u, u, n, c->k, c->kp);
  if (!rc && v) rc = download_rows(c, c->d_v, v, m, c->k, c->kp);
  return rc;
}

int bgmf_run_step(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off, int nbatch,
                  int inner_iters, double alpha, double beta, double* sse_out, int64_t* bad_out) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (!plan || !batch_off || nbatch < 0 || !sse_out || !bad_out)
    return fail(c, BGMF_ERR_ARG, "NULL argument");
  if (inner_iters < 1 || inner_iters > 65535) return fail(c, BGMF_ERR_ARG, "inner_iters out of range");
  int rc = check_step_ready(c);
  if (rc) return rc;
  cudaSetDevice(c->device);
  if (c->exact)
    rc = run_step_exact(c, plan, batch_off, nbatch, inner_iters, alpha, beta);
  else if (c->streaming)
    rc = run_step_stream(c, plan, batch_off, nbatch, inner_iters, (float)alpha, (float)beta);
  else
    rc = run_step_fast(c, plan, batch_off, nbatch, inner_iters, (float)alpha, (float)beta);
  if (rc) return rc;
  const int nb = c->I * c->J;
  for (int b = 0; b < nb; ++b) sse_out[b] = c->h_sse[b];
  fill_bad(c, bad_out);
  return BGMF_OK;
}

int bgmf_run_steps(bgmf_ctx* c, int nsteps, const int32_t* plans, const int32_t* batch_offs,
                   const int32_t* nbatch, const int32_t* inner_iters, double alpha, double beta,
                   double* sse_out, int64_t* bad_out, float* step_ms) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (nsteps < 0 || (nsteps > 0 && (!plans || !batch_offs || !nbatch || !inner_iters ||
                                    !sse_out)) || !bad_out)
    return fail(c, BGMF_ERR_ARG, "NULL argument");
  int rc = check_step_ready(c);
  if (rc) return rc;
  cudaSetDevice(c->device);
  return run_steps(c, nsteps, plans, batch_offs, nbatch, inner_iters, (float)alpha, (float)beta,
                   sse_out, bad_out, step_ms);
}

int bgmf_step_begin(bgmf_ctx* c, int max_blocks) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  int rc = check_step_ready(c);
  if (rc) return rc;
  cudaSetDevice(c->device);
  return step_begin(c, max_blocks);
}

int bgmf_step_batch(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off, int nbatch,
                    int inner_iters, double alpha, double beta) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (!plan || !batch_off || nbatch < 0) return fail(c, BGMF_ERR_ARG, "NULL argument");
  if (inner_iters < 1 || inner_iters > 65535) return fail(c, BGMF_ERR_ARG, "inner_iters out of range");
  for (int q = 0; q < batch_off[nbatch]; ++q)
    if (plan[q] < 0 || plan[q] >= c->I * c->J) return fail(c, BGMF_ERR_ARG, "plan block id out of range");
  cudaSetDevice(c->device);
  return step_batch(c, plan, batch_off, nbatch, inner_iters, (float)alpha, (float)beta);
}

int bgmf_step_end(bgmf_ctx* c, double* sse_out, int64_t* bad_out) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (!sse_out || !bad_out) return fail(c, BGMF_ERR_ARG, "NULL argument");
  cudaSetDevice(c->device);
  return step_end(c, sse_out, bad_out);
}

int bgmf_step_end_async(bgmf_ctx* c, double* d_sse_out, uint64_t* d_bad_out) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (!d_sse_out || !d_bad_out) return fail(c, BGMF_ERR_ARG, "NULL argument");
  cudaSetDevice(c->device);
  return step_end_async(c, d_sse_out, reinterpret_cast<unsigned long long*>(d_bad_out));
}

int bgmf_run_sync_parallel_step(bgmf_ctx* c, const int64_t* shard_edges, int nshards,
                                double alpha, double beta, double* sse_out, int64_t* bad_out) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  int rc = check_step_ready(c);
  if (rc) return rc;
  if (c->streaming) return fail(c, BGMF_ERR_STATE, "sync-parallel steps do not stream");
  cudaSetDevice(c->device);
  return run_sync_parallel_step(c, shard_edges, nshards, alpha, beta, sse_out, bad_out);
}

int bgmf_run_step_converge(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off,
                           int nbatch, double tol, int64_t cap, double alpha, double beta,
                           double* sse_out, int64_t* iters_out, int32_t* capped_out,
                           int64_t* bad_out) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (!plan || !batch_off || !sse_out || !iters_out || !capped_out || !bad_out)
    return fail(c, BGMF_ERR_ARG, "NULL argument");
  if (!(tol > 0) || cap < 1) return fail(c, BGMF_ERR_ARG, "converge mode needs tol > 0, cap >= 1");
  int rc = check_step_ready(c);
  if (rc) return rc;
  cudaSetDevice(c->device);
  rc = c->streaming ? run_step_stream_converge(c, plan, batch_off, nbatch, tol, cap, alpha,
                                                beta, iters_out, capped_out)
     : c->exact ? run_step_converge_exact(c, plan, batch_off, nbatch, tol, cap, alpha, beta,
                                          iters_out, capped_out)
                : run_step_converge_fast(c, plan, batch_off, nbatch, tol, cap, alpha, beta,
                                         iters_out, capped_out);
  if (rc) return rc;
  const int nb = c->I * c->J;
  for (int b = 0; b < nb; ++b) sse_out[b] = c->h_sse[b];
  fill_bad(c, bad_out);
  return BGMF_OK;
}

int bgmf_train_sse(bgmf_ctx* c, double* sse_out) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  int rc = check_step_ready(c);
  if (rc) return rc;
  cudaSetDevice(c->device);
  rc = ensure_step_scratch(c, 1);
  if (rc) return rc;
  if (c->streaming) {  // zero sweeps: every block's SSE of the current factors
    const int nb = c->I * c->J;
    std::vector<int32_t> plan(nb), off{0, nb};
    for (int b = 0; b < nb; ++b) plan[b] = b;
    rc = run_step_stream(c, plan.data(), off.data(), 1, 0, 0.f, 0.f);
    if (rc) return rc;
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += c->h_sse[b];
    *sse_out = acc;
    return BGMF_OK;
  }
  return c->exact ? train_sse_exact(c, sse_out) : train_sse_fast(c, sse_out);
}

int bgmf_holdout_set(bgmf_ctx* c, const int64_t* rows, const int64_t* cols, const double* vals,
                     const uint8_t* cold, int64_t count, double fallback) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  if (count < 0 || (count > 0 && (!rows || !cols || !vals)))
    return fail(c, BGMF_ERR_ARG, "bad holdout arguments");
  cudaSetDevice(c->device);
  free_holdout(c);
  const size_t N = (size_t)(count > 0 ? count : 1);
  std::vector<int32_t> r(N), q(N);
  for (int64_t i = 0; i < count; ++i) {
    if (rows[i] < 0 || rows[i] >= c->n || cols[i] < 0 || cols[i] >= c->m)
      return fail(c, BGMF_ERR_DATA, "holdout index outside the matrix");
    r[i] = (int32_t)rows[i];
    q[i] = (int32_t)cols[i];
  }
  std::vector<float> vf(N);
  for (int64_t i = 0; i < count; ++i) vf[i] = (float)vals[i];
  BGMF_CK(c, dmalloc(&c->d_hrow, N * 4, c->stream));
  BGMF_CK(c, dmalloc(&c->d_hcol, N * 4, c->stream));
  BGMF_CK(c, dmalloc(&c->d_hval, N * 4, c->stream));
  BGMF_CK(c, dmalloc(&c->d_hval64, N * 8, c->stream));
  BGMF_CK(c, dmalloc(&c->d_hcold, N, c->stream));
  if (count > 0) {
    BGMF_CK(c, cudaMemcpyAsync(c->d_hrow, r.data(), count * 4, cudaMemcpyHostToDevice, c->stream));
    BGMF_CK(c, cudaMemcpyAsync(c->d_hcol, q.data(), count * 4, cudaMemcpyHostToDevice, c->stream));
    BGMF_CK(c, cudaMemcpyAsync(c->d_hval, vf.data(), count * 4, cudaMemcpyHostToDevice, c->stream));
    BGMF_CK(c, cudaMemcpyAsync(c->d_hval64, vals, count * 8, cudaMemcpyHostToDevice, c->stream));
    if (cold) BGMF_CK(c, cudaMemcpyAsync(c->d_hcold, cold, count, cudaMemcpyHostToDevice, c->stream));
    else BGMF_CK(c, cudaMemsetAsync(c->d_hcold, 0, count, c->stream));
  }
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  c->hcount = count;
  c->hfallback = fallback;
  return BGMF_OK;
}

int bgmf_holdout_sse(bgmf_ctx* c, double* sse_out) {
  if (!c || !sse_out) return fail(c, BGMF_ERR_ARG, "NULL argument");
  if (!c->have_factors) return fail(c, BGMF_ERR_STATE, "no factors on the device");
  if (!c->d_hrow) return fail(c, BGMF_ERR_STATE, "bgmf_holdout_set has not been called");
  cudaSetDevice(c->device);
  if (c->hcount == 0) { *sse_out = 0.0; return BGMF_OK; }
  if (c->exact)
    return eval_sse_f64(c, c->d_u64, c->d_v64, c->k, c->d_hrow, c->d_hcol, c->d_hval64, c->d_hcold,
                        c->hfallback, c->hcount, sse_out);
  return eval_sse_f32(c, c->d_hrow, c->d_hcol, c->d_hval, c->d_hcold, c->hfallback, c->hcount,
                      sse_out);
}

int bgmf_partition_ooc(bgmf_ctx* c, const int64_t* rows, const int64_t* cols,
                       const double* vals, int64_t nnz, int64_t n, int64_t m, int grid_i,
                       int grid_j, int64_t device_budget, int64_t slot_ratings, int nslots,
                       int64_t row_lo, int64_t row_hi) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  cudaSetDevice(c->device);
  prof_mark(c, nullptr);
  dfree(c->d_sse, c->stream); pinned_free(c->h_sse); dfree(c->d_fuse, c->stream); c->d_fuse = nullptr; dfree(c->d_cstate, c->stream); c->d_cstate = nullptr; c->cstate_cap = 0; conv_graphs_release(c); dfree(c->d_bad, c->stream); pinned_free(c->h_bad);
  c->d_sse = nullptr; c->h_sse = nullptr; c->d_bad = nullptr; c->h_bad = nullptr;
  return partition_ooc(c, rows, cols, vals, nnz, n, m, grid_i, grid_j, device_budget,
                       slot_ratings, nslots, row_lo, row_hi);
}

int bgmf_mem_stats(bgmf_ctx* c, int64_t* out2, int reset) {
  if (!c || !out2) return fail(c, BGMF_ERR_ARG, "NULL argument");
  cudaSetDevice(c->device);
  cudaMemPool_t pool;
  BGMF_CK(c, cudaDeviceGetDefaultMemPool(&pool, c->device));
  unsigned long long used = 0, high = 0;
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  BGMF_CK(c, cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  BGMF_CK(c, cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high));
  out2[0] = (int64_t)used;
  out2[1] = (int64_t)high;
  if (reset) {
    unsigned long long zero = 0;
    BGMF_CK(c, cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero));
  }
  return BGMF_OK;
}

int bgmf_stream_ratings(bgmf_ctx* c, int64_t slot_ratings, int nslots) {
  if (!c) return fail(nullptr, BGMF_ERR_ARG, "ctx is NULL");
  cudaSetDevice(c->device);
  return stream_enable(c, slot_ratings, nslots);
}

int bgmf_stream_stats(bgmf_ctx* c, double* h2d_bytes) {
  if (!c || !h2d_bytes) return fail(c, BGMF_ERR_ARG, "NULL argument");
  *h2d_bytes = c->h2d_bytes;
  return BGMF_OK;
}

int bgmf_kernel_stats(bgmf_ctx* c, double* out5, int reset) {
  if (!c || !out5) return fail(c, BGMF_ERR_ARG, "NULL argument");
  if (c->events_used) {  // launches timed since the last synchronising call
    cudaSetDevice(c->device);
    harvest_timing(c);
  }
  out5[0] = c->t_sgd_ms;
  out5[1] = c->t_sse_ms;
  out5[2] = (double)c->n_sgd;
  out5[3] = (double)c->n_sse;
  out5[4] = c->t_bytes;
  if (reset) { c->t_sgd_ms = c->t_sse_ms = c->t_bytes = 0; c->n_sgd = c->n_sse = 0; }
  return BGMF_OK;
}

// ---------------------------------------------------------------- stateless

int bgmf_sgd_sweeps(const int64_t* rows, const int64_t* cols, const double* vals, int64_t count,
                    double* u, int64_t u_rows, double* v, int64_t v_rows, int k, double alpha,
                    double beta, int iters, double* sse_before, double* sse_after,
                    int64_t* bad_entry, int64_t* bad_iter) {
  int rc;
  bgmf_ctx* c = scratch_ctx(&rc);
  if (!c) return rc;
  if (iters < 0) return fail(nullptr, BGMF_ERR_ARG, "iters must be >= 0");
  double o[6];
  rc = block_exact(c, rows, cols, vals, count, u, u_rows, v, v_rows, k, alpha, beta, 0, iters,
                   0.0, 0, o);
  if (rc) { g_err = c->err; return rc; }
  *sse_before = o[0]; *sse_after = o[1];
  *bad_entry = (int64_t)o[4]; *bad_iter = (int64_t)o[5];
  return BGMF_OK;
}

int bgmf_gradient_steps(const int64_t* rows, const int64_t* cols, const double* vals,
                        int64_t count, double* u, int64_t u_rows, double* v, int64_t v_rows,
                        int k, double alpha, double beta, int iters, double* sse_before,
                        double* sse_after, int64_t* bad_entry, int64_t* bad_iter) {
  int rc;
  bgmf_ctx* c = scratch_ctx(&rc);
  if (!c) return rc;
  if (!sse_before || !sse_after || !bad_entry || !bad_iter)
    return fail(nullptr, BGMF_ERR_ARG, "NULL out-parameter");
  double o[4];
  rc = gradient_steps(c, rows, cols, vals, count, u, u_rows, v, v_rows, k, alpha, beta, iters, o);
  if (rc) { g_err = c->err; return rc; }
  *sse_before = o[0]; *sse_after = o[1];
  *bad_entry = (int64_t)o[2]; *bad_iter = (int64_t)o[3];
  return BGMF_OK;
}

int bgmf_block_gradients(const int64_t* rows, const int64_t* cols, const double* vals,
                         int64_t count, const double* u, int64_t u_rows, const double* v,
                         int64_t v_rows, int k, double beta, double* gu, double* gv,
                         double* sse, double* sq_norms) {
  int rc;
  bgmf_ctx* c = scratch_ctx(&rc);
  if (!c) return rc;
  if (!sse || !sq_norms) return fail(nullptr, BGMF_ERR_ARG, "NULL out-parameter");
  double o[2];
  rc = block_gradients(c, rows, cols, vals, count, u, u_rows, v, v_rows, k, beta, gu, gv, o);
  if (rc) { g_err = c->err; return rc; }
  *sse = o[0];
  *sq_norms = o[1];
  return BGMF_OK;
}

int bgmf_sgd_converge(const int64_t* rows, const int64_t* cols, const double* vals, int64_t count,
                      double* u, int64_t u_rows, double* v, int64_t v_rows, int k, double alpha,
                      double beta, double tol, int64_t cap, double* sse_before, double* sse_after,
                      int64_t* iters_used, int32_t* capped, int64_t* bad_entry,
                      int64_t* bad_iter) {
  int rc;
  bgmf_ctx* c = scratch_ctx(&rc);
  if (!c) return rc;
  double o[6];
  rc = block_exact(c, rows, cols, vals, count, u, u_rows, v, v_rows, k, alpha, beta, 1, 0, tol,
                   cap, o);
  if (rc) { g_err = c->err; return rc; }
  *sse_before = o[0]; *sse_after = o[1];
  *iters_used = (int64_t)o[2]; *capped = (int32_t)o[3];
  *bad_entry = (int64_t)o[4]; *bad_iter = (int64_t)o[5];
  return BGMF_OK;
}

int bgmf_block_sse(const int64_t* rows, const int64_t* cols, const double* vals, int64_t count,
                   const double* u, int64_t u_rows, const double* v, int64_t v_rows, int k,
                   double* sse) {
  int rc;
  bgmf_ctx* c = scratch_ctx(&rc);
  if (!c) return rc;
  double o[6];
  rc = block_exact(c, rows, cols, vals, count, const_cast<double*>(u), u_rows,
                   const_cast<double*>(v), v_rows, k, 0.0, 0.0, 2, 0, 0.0, 0, o);
  if (rc) { g_err = c->err; return rc; }
  *sse = o[0];
  return BGMF_OK;
}

namespace {

// upload u, v (f64) and int32 copies of rows/cols; caller frees via cleanup
struct EvalBufs {
  double *u = nullptr, *v = nullptr, *vals = nullptr, *pred = nullptr;
  int32_t *r = nullptr, *q = nullptr;
  uint8_t* cold = nullptr;
  ~EvalBufs() {
    cudaFree(u); cudaFree(v); cudaFree(vals); cudaFree(pred); cudaFree(r); cudaFree(q);
    cudaFree(cold);
  }
};

int eval_upload(bgmf_ctx* c, EvalBufs& b, const double* u, int64_t n, const double* v, int64_t m,
                int k, const int64_t* rows, const int64_t* cols, int64_t count) {
  if (!u || !v || k < 1 || n < 1 || m < 1 || count < 0 || n >= INT32_MAX || m >= INT32_MAX)
    return fail(c, BGMF_ERR_ARG, "bad model/dataset shapes");
  const size_t N = (size_t)(count > 0 ? count : 1);
  std::vector<int32_t> r(N), q(N);
  for (int64_t i = 0; i < count; ++i) {
    if (rows[i] < 0 || rows[i] >= n || cols[i] < 0 || cols[i] >= m)
      return fail(c, BGMF_ERR_DATA, "index outside the model");
    r[i] = (int32_t)rows[i];
    q[i] = (int32_t)cols[i];
  }
  BGMF_CK(c, dmalloc(&b.u, (size_t)n * k * 8, c->stream));
  BGMF_CK(c, dmalloc(&b.v, (size_t)m * k * 8, c->stream));
  BGMF_CK(c, dmalloc(&b.r, N * 4, c->stream));
  BGMF_CK(c, dmalloc(&b.q, N * 4, c->stream));
  BGMF_CK(c, cudaMemcpyAsync(b.u, u, (size_t)n * k * 8, cudaMemcpyHostToDevice, c->stream));
  BGMF_CK(c, cudaMemcpyAsync(b.v, v, (size_t)m * k * 8, cudaMemcpyHostToDevice, c->stream));
  if (count > 0) {
    BGMF_CK(c, cudaMemcpyAsync(b.r, r.data(), count * 4, cudaMemcpyHostToDevice, c->stream));
    BGMF_CK(c, cudaMemcpyAsync(b.q, q.data(), count * 4, cudaMemcpyHostToDevice, c->stream));
  }
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  return BGMF_OK;
}

}  // namespace

int bgmf_predict(const double* u, int64_t n, const double* v, int64_t m, int k,
                 const int64_t* rows, const int64_t* cols, int64_t count, double* out) {
  int rc;
  bgmf_ctx* c = scratch_ctx(&rc);
  if (!c) return rc;
  EvalBufs b;
  rc = eval_upload(c, b, u, n, v, m, k, rows, cols, count);
  if (rc) { g_err = c->err; return rc; }
  if (count == 0) return BGMF_OK;
  cudaError_t e = dmalloc(&b.pred, (size_t)count * 8, c->stream);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaMalloc");
  rc = predict_f64(c, b.u, b.v, k, b.r, b.q, count, b.pred);
  if (rc) { g_err = c->err; return rc; }
  e = cudaMemcpyAsync(out, b.pred, (size_t)count * 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "predict download");
  return BGMF_OK;
}

int bgmf_sse(const double* u, int64_t n, const double* v, int64_t m, int k, const int64_t* rows,
             const int64_t* cols, const double* vals, const uint8_t* cold, double fallback,
             int64_t count, double* sse) {
  int rc;
  bgmf_ctx* c = scratch_ctx(&rc);
  if (!c) return rc;
  EvalBufs b;
  rc = eval_upload(c, b, u, n, v, m, k, rows, cols, count);
  if (rc) { g_err = c->err; return rc; }
  if (count == 0) { *sse = 0.0; return BGMF_OK; }
  const size_t N = (size_t)count;
  cudaError_t e = dmalloc(&b.vals, N * 8, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(b.vals, vals, N * 8, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess && cold) {
    e = dmalloc(&b.cold, N, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(b.cold, cold, N, cudaMemcpyHostToDevice, c->stream);
  }
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "sse upload");
  rc = eval_sse_f64(c, b.u, b.v, k, b.r, b.q, b.vals, b.cold, fallback, count, sse);
  if (rc) { g_err = c->err; return rc; }
  return BGMF_OK;
}

}  // extern "C"
