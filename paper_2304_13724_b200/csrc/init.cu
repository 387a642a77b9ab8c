// init.cu -- init_factors on the device, bit-identical to the reference
// (core.py:179-193: rng = np.random.default_rng(seed); u = rng.random((n, k))
// / sqrt(k); then v the same way).
//
// numpy's default generator is PCG64: a 128-bit LCG s <- s*A + inc, output
// XSL-RR (rotr64(hi ^ lo, s >> 122)) of the new state; Generator.random()
// maps a draw x to (x >> 11) * 2^-53.  Draw i of the stream is reached from the
// seeded state by LCG jump-ahead (Brown's O(log i) power), so every thread
// produces its own contiguous run of draws independently.  The host passes
// the seeded (state, inc) that numpy's SeedSequence produced.

#include <cmath>

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

typedef unsigned __int128 u128;

constexpr uint64_t kMulHi = 0x2360ED051FC65DA4ull;
constexpr uint64_t kMulLo = 0x4385DF649FCCF645ull;
constexpr int kDrawsPerThread = 64;

__device__ __forceinline__ u128 mk(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

// state after `delta` LCG steps
__device__ u128 advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = mk(kMulHi, kMulLo), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned r = (unsigned)(s >> 122);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// fills U (n x k) then V (m x k); fp32 rows of stride kp (fast) and/or fp64
// rows of stride k (exact).  Padding columns are zeroed by the host first.
__global__ void pcg64_factors(uint64_t shi, uint64_t slo, uint64_t ihi, uint64_t ilo, int64_t n,
                              int64_t m, int k, int kp, double scale, float* __restrict__ u32,
                              float* __restrict__ v32, double* __restrict__ u64,
                              double* __restrict__ v64) {
  const int64_t total = (n + m) * (int64_t)k;
  const int64_t first = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kDrawsPerThread;
  if (first >= total) return;
  const u128 inc = mk(ihi, ilo);
  const u128 mult = mk(kMulHi, kMulLo);
  u128 s = advance(mk(shi, slo), inc, (uint64_t)first);
  const int64_t last = first + kDrawsPerThread < total ? first + kDrawsPerThread : total;
  const int64_t nk = n * (int64_t)k;
  for (int64_t i = first; i < last; ++i) {
    s = s * mult + inc;
    const double d = (double)(xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0);
    const double x = __dmul_rn(d, scale);
    const bool in_u = i < nk;
    const int64_t j = in_u ? i : i - nk;
    const int64_t row = j / k;
    const int col = (int)(j - row * k);
    if (in_u) {
      if (u32) u32[row * kp + col] = (float)x;
      if (u64) u64[row * k + col] = x;
    } else {
      if (v32) v32[row * kp + col] = (float)x;
      if (v64) v64[row * k + col] = x;
    }
  }
}

}  // namespace

int init_factors_device(bgmf_ctx* c, uint64_t shi, uint64_t slo, uint64_t ihi, uint64_t ilo,
                        int64_t n, int64_t m, int k) {
  cudaStream_t s = c->stream;
  const double scale = 1.0 / std::sqrt((double)k);
  float *u32 = c->d_u, *v32 = c->d_v;
  double *u64 = c->d_u64, *v64 = c->d_v64;
  if (u32) BGMF_CK(c, cudaMemsetAsync(u32, 0, (size_t)n * c->kp * 4, s));
  if (v32) BGMF_CK(c, cudaMemsetAsync(v32, 0, (size_t)m * c->kp * 4, s));
  const int64_t total = (n + m) * (int64_t)k;
  const int64_t threads = (total + kDrawsPerThread - 1) / kDrawsPerThread;
  if (threads > 0)
    pcg64_factors<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
        shi, slo, ihi, ilo, n, m, k, c->kp, scale, u32, v32, u64, v64);
  BGMF_CK(c, cudaGetLastError());
  BGMF_CK(c, cudaStreamSynchronize(s));
  return BGMF_OK;
}

}  // namespace bgmf
