// gradient.cu -- the reference's verification kernels on the GPU:
//   _kernels.gradient_steps (reference _kernels.py:103-140), called by
//   kernel.batch_gradient_block (kernel.py:142-158), and the pure
//   block_objective / block_gradients (kernel.py:161-179).
//
// gradient_steps is full-batch gradient descent on one block: per iteration
// du, dv accumulate 2e*v / 2e*u over the entries in stored order (pre-update
// factors), then every row moves u += a(du - b u), v += a(dv - b v).  Here one
// CTA owns the block; thread g owns latent dimension g, so every (row, g)
// accumulator sees the entries in the reference's order, and the residual is
// reduced serially over g by one thread with explicitly rounded fp64 ops:
// bit-identical to numba's fastmath=False loops.  A verification path, not a
// throughput path (one CTA; the serial residual is O(k) per entry).

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

constexpr int kGradThreads = 256;

// block_sse (_kernels.py:16-28), sequential.
__device__ double sse_seq(const int32_t* rows, const int32_t* cols, const double* vals,
                          int64_t count, const double* u, const double* v, int k) {
  double s = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    const double* ur = u + (int64_t)rows[i] * k;
    const double* vc = v + (int64_t)cols[i] * k;
    double e = vals[i];
    for (int g = 0; g < k; ++g) e = __dsub_rn(e, __dmul_rn(ur[g], vc[g]));
    s = __dadd_rn(s, __dmul_rn(e, e));
  }
  return s;
}

// Residual of entry i: x - sum_g u[r,g] v[c,g], subtracted in g order.  The
// products are formed in parallel (one per thread), the chain by thread 0.
__device__ double residual(const double* ur, const double* vc, double x, int k, double* sprod,
                           double* se) {
  for (int g = threadIdx.x; g < k; g += blockDim.x) sprod[g] = __dmul_rn(ur[g], vc[g]);
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = x;
    for (int g = 0; g < k; ++g) e = __dsub_rn(e, sprod[g]);
    *se = e;
  }
  __syncthreads();
  return *se;
}

// out: {sse_before, sse_after, bad_entry, bad_iter}
__global__ void __launch_bounds__(kGradThreads)
gradient_steps_kernel(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                      const double* __restrict__ vals, int64_t count, double* u, int64_t nu,
                      double* v, int64_t nv, int k, double alpha, double beta, int iters,
                      double* du, double* dv, double* out) {
  extern __shared__ double sprod[];
  __shared__ double se;
  __shared__ double s_sb;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  if (threadIdx.x == 0) s_sb = sse_seq(rows, cols, vals, count, u, v, k);
  __syncthreads();
  const double sb = s_sb;
  for (int it = 0; it < iters; ++it) {
    for (int64_t i = threadIdx.x; i < nu * k; i += blockDim.x) du[i] = 0.0;
    for (int64_t i = threadIdx.x; i < nv * k; i += blockDim.x) dv[i] = 0.0;
    __syncthreads();
    for (int64_t idx = 0; idx < count; ++idx) {
      const int64_t r = rows[idx], c = cols[idx];
      double* ur = u + r * k;
      double* vc = v + c * k;
      const double e = residual(ur, vc, vals[idx], k, sprod, &se);
      if (!isfinite(e)) {
        if (threadIdx.x == 0) { out[0] = sb; out[1] = nan; out[2] = (double)idx; out[3] = it; }
        return;
      }
      const double e2 = __dmul_rn(2.0, e);
      for (int g = threadIdx.x; g < k; g += blockDim.x) {
        du[r * k + g] = __dadd_rn(du[r * k + g], __dmul_rn(e2, vc[g]));
        dv[c * k + g] = __dadd_rn(dv[c * k + g], __dmul_rn(e2, ur[g]));
      }
      // the next entry's products read u/v only; du/dv rows are per thread
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < nu * k; i += blockDim.x)
      u[i] = __dadd_rn(u[i], __dmul_rn(alpha, __dsub_rn(du[i], __dmul_rn(beta, u[i]))));
    for (int64_t i = threadIdx.x; i < nv * k; i += blockDim.x)
      v[i] = __dadd_rn(v[i], __dmul_rn(alpha, __dsub_rn(dv[i], __dmul_rn(beta, v[i]))));
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double sa = sse_seq(rows, cols, vals, count, u, v, k);
    out[0] = sb;
    if (!isfinite(sa)) {
      out[1] = nan; out[2] = (double)(count - 1); out[3] = iters - 1;
    } else {
      out[1] = sa; out[2] = -1.0; out[3] = -1.0;
    }
  }
}

// block_gradients / block_objective (kernel.py:161-179), fp64:
//   e = x - u[r].v[c];  gu = beta u;  gu[r] += (-2e) v[c] in entry order (np.add.at);
//   gv likewise;  objective = e.e + (beta/2)(|u|^2 + |v|^2).
// out: {sum e^2, sum u^2 + sum v^2}
__global__ void __launch_bounds__(kGradThreads)
block_gradients_kernel(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                       const double* __restrict__ vals, int64_t count, const double* u,
                       int64_t nu, const double* v, int64_t nv, int k, double beta, double* gu,
                       double* gv, double* out) {
  extern __shared__ double sprod[];
  __shared__ double se;
  for (int64_t i = threadIdx.x; i < nu * k; i += blockDim.x) gu[i] = __dmul_rn(beta, u[i]);
  for (int64_t i = threadIdx.x; i < nv * k; i += blockDim.x) gv[i] = __dmul_rn(beta, v[i]);
  __syncthreads();
  double ee = 0.0;
  for (int64_t idx = 0; idx < count; ++idx) {
    const int64_t r = rows[idx], c = cols[idx];
    const double* ur = u + r * k;
    const double* vc = v + c * k;
    const double e = residual(ur, vc, vals[idx], k, sprod, &se);
    ee = __dadd_rn(ee, __dmul_rn(e, e));
    const double m2e = __dmul_rn(-2.0, e);
    for (int g = threadIdx.x; g < k; g += blockDim.x) {
      gu[r * k + g] = __dadd_rn(gu[r * k + g], __dmul_rn(m2e, vc[g]));
      gv[c * k + g] = __dadd_rn(gv[c * k + g], __dmul_rn(m2e, ur[g]));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double reg = 0.0;
    for (int64_t i = 0; i < nu * k; ++i) reg = __dadd_rn(reg, __dmul_rn(u[i], u[i]));
    double reg_v = 0.0;
    for (int64_t i = 0; i < nv * k; ++i) reg_v = __dadd_rn(reg_v, __dmul_rn(v[i], v[i]));
    out[0] = ee;
    out[1] = __dadd_rn(reg, reg_v);
  }
}

struct GradBufs {
  cudaStream_t s;
  int32_t *r = nullptr, *c = nullptr;
  double *x = nullptr, *u = nullptr, *v = nullptr, *du = nullptr, *dv = nullptr, *out = nullptr;
  explicit GradBufs(cudaStream_t st) : s(st) {}
  ~GradBufs() {
    dfree(r, s); dfree(c, s); dfree(x, s); dfree(u, s); dfree(v, s); dfree(du, s);
    dfree(dv, s); dfree(out, s);
  }
};

// Upload a block (int64 local indices -> int32, range-checked) and its slices.
int grad_upload(bgmf_ctx* c, GradBufs& b, const int64_t* rows, const int64_t* cols,
                const double* vals, int64_t count, const double* u, int64_t nu, const double* v,
                int64_t nv, int k) {
  if (count < 0 || nu < 0 || nv < 0 || k < 1 || nu >= INT32_MAX || nv >= INT32_MAX)
    return fail(c, BGMF_ERR_ARG, "bad block shapes");
  if (count > 0 && (!rows || !cols || !vals)) return fail(c, BGMF_ERR_ARG, "NULL entries");
  if ((nu > 0 && !u) || (nv > 0 && !v)) return fail(c, BGMF_ERR_ARG, "NULL factor slice");
  std::vector<int32_t> r32((size_t)count), c32((size_t)count);
  for (int64_t i = 0; i < count; ++i) {
    if (rows[i] < 0 || rows[i] >= nu || cols[i] < 0 || cols[i] >= nv)
      return fail(c, BGMF_ERR_DATA, "entry index outside the factor slices");
    r32[i] = (int32_t)rows[i];
    c32[i] = (int32_t)cols[i];
  }
  const size_t N = (size_t)(count > 0 ? count : 1);
  const size_t U = (size_t)(nu > 0 ? nu : 1) * k, V = (size_t)(nv > 0 ? nv : 1) * k;
  cudaStream_t s = c->stream;
  BGMF_CK(c, dmalloc(&b.r, N * 4, s));
  BGMF_CK(c, dmalloc(&b.c, N * 4, s));
  BGMF_CK(c, dmalloc(&b.x, N * 8, s));
  BGMF_CK(c, dmalloc(&b.u, U * 8, s));
  BGMF_CK(c, dmalloc(&b.v, V * 8, s));
  BGMF_CK(c, dmalloc(&b.du, U * 8, s));
  BGMF_CK(c, dmalloc(&b.dv, V * 8, s));
  BGMF_CK(c, dmalloc(&b.out, 4 * 8, s));
  if (count > 0) {
    BGMF_CK(c, cudaMemcpyAsync(b.r, r32.data(), count * 4, cudaMemcpyHostToDevice, s));
    BGMF_CK(c, cudaMemcpyAsync(b.c, c32.data(), count * 4, cudaMemcpyHostToDevice, s));
    BGMF_CK(c, cudaMemcpyAsync(b.x, vals, count * 8, cudaMemcpyHostToDevice, s));
  }
  if (nu > 0) BGMF_CK(c, cudaMemcpyAsync(b.u, u, (size_t)nu * k * 8, cudaMemcpyHostToDevice, s));
  if (nv > 0) BGMF_CK(c, cudaMemcpyAsync(b.v, v, (size_t)nv * k * 8, cudaMemcpyHostToDevice, s));
  return BGMF_OK;
}

// k products, padded: thread 0 reads them back with vectorised shared loads
size_t grad_smem(int k) { return ((size_t)k + 2) * sizeof(double); }

}  // namespace

int gradient_steps(bgmf_ctx* c, const int64_t* rows, const int64_t* cols, const double* vals,
                   int64_t count, double* u, int64_t nu, double* v, int64_t nv, int k,
                   double alpha, double beta, int iters, double* out4) {
  if (iters < 1) return fail(c, BGMF_ERR_ARG, "iters must be >= 1");
  GradBufs b(c->stream);
  int rc = grad_upload(c, b, rows, cols, vals, count, u, nu, v, nv, k);
  if (rc) return rc;
  const size_t smem = grad_smem(k);
  if (smem > 48 * 1024)
    BGMF_CK(c, cudaFuncSetAttribute(gradient_steps_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gradient_steps_kernel<<<1, kGradThreads, smem, c->stream>>>(b.r, b.c, b.x, count, b.u, nu, b.v,
                                                              nv, k, alpha, beta, iters, b.du,
                                                              b.dv, b.out);
  BGMF_CK(c, cudaGetLastError());
  BGMF_CK(c, cudaMemcpyAsync(out4, b.out, 4 * 8, cudaMemcpyDeviceToHost, c->stream));
  if (nu > 0) BGMF_CK(c, cudaMemcpyAsync(u, b.u, (size_t)nu * k * 8, cudaMemcpyDeviceToHost, c->stream));
  if (nv > 0) BGMF_CK(c, cudaMemcpyAsync(v, b.v, (size_t)nv * k * 8, cudaMemcpyDeviceToHost, c->stream));
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  return BGMF_OK;
}

int block_gradients(bgmf_ctx* c, const int64_t* rows, const int64_t* cols, const double* vals,
                    int64_t count, const double* u, int64_t nu, const double* v, int64_t nv,
                    int k, double beta, double* gu, double* gv, double* out2) {
  GradBufs b(c->stream);
  int rc = grad_upload(c, b, rows, cols, vals, count, u, nu, v, nv, k);
  if (rc) return rc;
  const size_t smem = grad_smem(k);
  if (smem > 48 * 1024)
    BGMF_CK(c, cudaFuncSetAttribute(block_gradients_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  block_gradients_kernel<<<1, kGradThreads, smem, c->stream>>>(b.r, b.c, b.x, count, b.u, nu,
                                                               b.v, nv, k, beta, b.du, b.dv,
                                                               b.out);
  BGMF_CK(c, cudaGetLastError());
  BGMF_CK(c, cudaMemcpyAsync(out2, b.out, 2 * 8, cudaMemcpyDeviceToHost, c->stream));
  if (gu && nu > 0)
    BGMF_CK(c, cudaMemcpyAsync(gu, b.du, (size_t)nu * k * 8, cudaMemcpyDeviceToHost, c->stream));
  if (gv && nv > 0)
    BGMF_CK(c, cudaMemcpyAsync(gv, b.dv, (size_t)nv * k * 8, cudaMemcpyDeviceToHost, c->stream));
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  return BGMF_OK;
}

}  // namespace bgmf
