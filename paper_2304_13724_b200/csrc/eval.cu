// eval.cu -- RMSE / prediction kernels (reference metrics.py:39-86,
// core.py:163-165).
//
// Squared errors are accumulated in fp64 per worker, reduced per CTA in a
// fixed order into partials[blockIdx.x], and the (few hundred) partials are
// summed on the host in index order: the result is deterministic for a given
// grid (the reference uses numpy's pairwise sum; both are within a few ulp of
// the exact sum).  Cold entries (HoldoutEvaluator, metrics.py:68-79) predict
// the training mean.

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

constexpr int EVAL_THREADS = 256;

__device__ __forceinline__ double block_sum(double x, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  if (lane == 0) smem[warp] = x;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < EVAL_THREADS / 32; ++w) s += smem[w];
  return s;
}

// fp32 device factors (row stride kp), group of L lanes per entry.
template <int L, int V4>
__global__ void __launch_bounds__(EVAL_THREADS)
eval_f32_kernel(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                const float* __restrict__ vals, const uint8_t* __restrict__ cold,
                double fallback, int64_t count, const float* __restrict__ U,
                const float* __restrict__ V, int kp, double* __restrict__ partials) {
  __shared__ double smem[EVAL_THREADS / 32];
  const int lane = threadIdx.x & 31;
  const int gl = lane & (L - 1);
  const int64_t groups = (int64_t)gridDim.x * EVAL_THREADS / L;
  const int64_t g = ((int64_t)blockIdx.x * EVAL_THREADS + threadIdx.x) / L;
  const int64_t stride = groups;
  const int64_t rounds = (count + stride - 1) / stride;
  double acc = 0.0;
  for (int64_t r = 0; r < rounds; ++r) {
    const int64_t i = r * stride + g;
    const bool valid = i < count;
    float dot = 0.f;
    if (valid) {
      const float* up = U + (int64_t)rows[i] * kp;
      const float* vp = V + (int64_t)cols[i] * kp;
#pragma unroll
      for (int q = 0; q < V4; ++q) {
        if (4 * (q * L + gl) >= kp) continue;  // lane past the padded row
        const float4 a = __ldg(reinterpret_cast<const float4*>(up + 4 * (q * L + gl)));
        const float4 b = __ldg(reinterpret_cast<const float4*>(vp + 4 * (q * L + gl)));
        dot = fmaf(a.x, b.x, dot);
        dot = fmaf(a.y, b.y, dot);
        dot = fmaf(a.z, b.z, dot);
        dot = fmaf(a.w, b.w, dot);
      }
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(kFull, dot, o);
    if (valid && gl == 0) {
      const double pred = (cold && cold[i]) ? fallback : (double)dot;
      const double e = (double)vals[i] - pred;
      acc += e * e;
    }
  }
  const double s = block_sum(acc, smem);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// fp64 factors of arbitrary k (row stride k), one warp per entry.
template <typename IT>
__global__ void __launch_bounds__(EVAL_THREADS)
eval_f64_kernel(const IT* __restrict__ rows, const IT* __restrict__ cols,
                const double* __restrict__ vals, const uint8_t* __restrict__ cold,
                double fallback, int64_t count, const double* __restrict__ U,
                const double* __restrict__ V, int k, double* __restrict__ partials,
                double* __restrict__ pred_out) {
  __shared__ double smem[EVAL_THREADS / 32];
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * EVAL_THREADS / 32;
  const int64_t w = ((int64_t)blockIdx.x * EVAL_THREADS + threadIdx.x) >> 5;
  double acc = 0.0;
  for (int64_t i = w; i < count; i += warps) {
    const double* up = U + (int64_t)rows[i] * k;
    const double* vp = V + (int64_t)cols[i] * k;
    double d = 0.0;
    for (int q = lane; q < k; q += 32) d = fma(up[q], vp[q], d);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(kFull, d, o);
    if (lane == 0) {
      if (pred_out) pred_out[i] = d;
      if (vals) {
        const double pred = (cold && cold[i]) ? fallback : d;
        const double e = vals[i] - pred;
        acc += e * e;
      }
    }
  }
  const double s = block_sum(acc, smem);
  if (partials && threadIdx.x == 0) partials[blockIdx.x] = s;
}

int eval_grid(bgmf_ctx* c) { return c->num_sms * 4; }

int ensure_partials(bgmf_ctx* c) {
  if (!c->d_partials) {
    BGMF_CK(c, dmalloc(&c->d_partials, sizeof(double) * eval_grid(c), c->stream));
  }
  return BGMF_OK;
}

int sum_partials(bgmf_ctx* c, double* out) {
  const int G = eval_grid(c);
  std::vector<double> h(G);
  BGMF_CK(c, cudaMemcpyAsync(h.data(), c->d_partials, sizeof(double) * G, cudaMemcpyDeviceToHost,
                             c->stream));
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  double s = 0.0;
  for (int i = 0; i < G; ++i) s += h[i];
  *out = s;
  return BGMF_OK;
}

}  // namespace

int eval_sse_f32(bgmf_ctx* c, const int32_t* rows, const int32_t* cols, const float* vals,
                 const uint8_t* cold, double fallback, int64_t count, double* out) {
  int rc = ensure_partials(c);
  if (rc) return rc;
  const int f4 = c->kp / 4;
  const dim3 grid(eval_grid(c));
  cudaStream_t s = c->stream;
#define EV(LL, VV)                                                                             \
  eval_f32_kernel<LL, VV><<<grid, EVAL_THREADS, 0, s>>>(rows, cols, vals, cold, fallback, count, \
                                                        c->d_u, c->d_v, c->kp, c->d_partials)
  if (f4 <= 1) EV(1, 1);
  else if (f4 <= 2) EV(2, 1);
  else if (f4 <= 4) EV(4, 1);
  else if (f4 <= 8) EV(8, 1);
  else if (f4 <= 16) EV(16, 1);
  else if (f4 <= 32) EV(32, 1);
  else if (f4 <= 64) EV(32, 2);
  else if (f4 <= 128) EV(32, 4);
  else EV(32, 8);
#undef EV
  BGMF_CK(c, cudaGetLastError());
  return sum_partials(c, out);
}

int eval_sse_f64(bgmf_ctx* c, const double* u, const double* v, int k, const int32_t* rows,
                 const int32_t* cols, const double* vals, const uint8_t* cold, double fallback,
                 int64_t count, double* out) {
  int rc = ensure_partials(c);
  if (rc) return rc;
  eval_f64_kernel<int32_t><<<eval_grid(c), EVAL_THREADS, 0, c->stream>>>(
      rows, cols, vals, cold, fallback, count, u, v, k, c->d_partials, nullptr);
  BGMF_CK(c, cudaGetLastError());
  return sum_partials(c, out);
}

int predict_f64(bgmf_ctx* c, const double* u, const double* v, int k, const int32_t* rows,
                const int32_t* cols, int64_t count, double* out_dev) {
  eval_f64_kernel<int32_t><<<eval_grid(c), EVAL_THREADS, 0, c->stream>>>(
      rows, cols, nullptr, nullptr, 0.0, count, u, v, k, nullptr, out_dev);
  BGMF_CK(c, cudaGetLastError());
  return BGMF_OK;
}

}  // namespace bgmf
