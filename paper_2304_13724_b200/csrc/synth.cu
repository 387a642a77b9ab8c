// synth.cu -- device-side synthetic workload generator (benchmark / test
// input only; not part of the factorization path).  Needed for C5 (2e9
// ratings), whose host generation would take minutes and ~50 GB.
//
// Cells: the keyed Feistel bijection of workloads.feistel_cells (same integer
// math, cycle walking), i.e. sampling without replacement in scrambled order.
// Values: the workloads.lowrank generative model -- 3.53 + user bias + item
// bias (N(0,.55)) + rank-6 taste (N(0,.6/sqrt 6)) + noise N(0,.8), rint, clip
// 1..5 -- but with counter-based normals (splitmix64 hash of (seed, index) ->
// Box-Muller), so any rating is computable independently on the device.

#include <cmath>

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Feistel {
  int lo_bits;
  uint64_t lo_mask, hi_mask, key[4];
};

__device__ __forceinline__ uint64_t feistel_perm(const Feistel& f, uint64_t x) {
  uint64_t hi = x >> f.lo_bits, lo = x & f.lo_mask;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if ((r & 1) == 0) hi = (hi ^ mix64(lo ^ f.key[r])) & f.hi_mask;
    else lo = (lo ^ mix64(hi ^ f.key[r])) & f.lo_mask;
  }
  return (hi << f.lo_bits) | lo;
}

// standard normal from two hashed uniforms (Box-Muller, cosine branch)
__device__ __forceinline__ double hnormal(uint64_t seed, uint64_t stream, uint64_t idx) {
  const uint64_t a = mix64(seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + idx);
  const uint64_t b = mix64(a ^ 0xA0761D6478BD642Full);
  const double u1 = ((a >> 11) + 1) * (1.0 / 9007199254740993.0);  // (0, 1]
  const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

__global__ void synth_kernel(Feistel f, uint64_t total, int64_t m, int64_t nnz, int64_t start,
                             uint64_t seed, int64_t* __restrict__ rows, int64_t* __restrict__ cols,
                             double* __restrict__ vals) {
  const double s_bias = 0.55, s_taste = 0.6 / sqrt(6.0), s_noise = 0.8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t y = feistel_perm(f, (uint64_t)(start + i));
    while (y >= total) y = feistel_perm(f, y);  // cycle walking
    const int64_t r = (int64_t)(y / (uint64_t)m), c = (int64_t)(y % (uint64_t)m);
    double x = 3.53 + s_bias * hnormal(seed, 1, r) + s_bias * hnormal(seed, 2, c);
    double taste = 0.0;
#pragma unroll
    for (int q = 0; q < 6; ++q)
      taste += (s_taste * hnormal(seed, 3 + q, r)) * (s_taste * hnormal(seed, 9 + q, c));
    x += taste + s_noise * hnormal(seed, 15, (uint64_t)(start + i));
    x = rint(x);
    rows[i] = r;
    cols[i] = c;
    vals[i] = x < 1.0 ? 1.0 : (x > 5.0 ? 5.0 : x);
  }
}

}  // namespace

int synth_lowrank_device(bgmf_ctx* c, int64_t n, int64_t m, int64_t nnz, int64_t start,
                         uint64_t seed, int64_t* rows, int64_t* cols, double* vals) {
  const uint64_t total = (uint64_t)n * (uint64_t)m;
  int bits = 2;
  while (bits < 64 && ((total - 1) >> bits) != 0) ++bits;
  Feistel f;
  f.lo_bits = bits / 2;
  const int hi_bits = bits - f.lo_bits;
  f.lo_mask = (1ull << f.lo_bits) - 1;
  f.hi_mask = (1ull << hi_bits) - 1;
  for (int r = 0; r < 4; ++r)
    f.key[r] = seed * 0x9E3779B97F4A7C15ull + (uint64_t)r * 0xD1B54A32D192ED03ull + 1;
  synth_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(f, total, m, nnz, start, seed, rows, cols,
                                                      vals);
  BGMF_CK(c, cudaGetLastError());
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  return BGMF_OK;
}

}  // namespace bgmf
