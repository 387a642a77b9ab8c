// rows.cuh -- lane geometry of a worker group and fp32 row arithmetic shared
// by the stratum kernels (sgd.cu: chunked sweep / SSE; ordered.cu: ordered
// slab sweep).  A group of L lanes owns one rating at a time; lane gl holds
// float4s gl, gl+L, ... (V4 of them) of a padded factor row of kp floats.
#pragma once

#include "bgmf_internal.cuh"

namespace bgmf {

struct Shape {
  int L, V4;
};

inline Shape shape_for(int kp) {
  // A group of L lanes owns one rating; lane gl holds float4s gl, gl+L, ...
  // of the row (V4 of them), so one warp instruction moves a 16L-byte
  // contiguous segment of each of 32/L rows.  L >= 4 keeps that segment at 64
  // bytes or more (two full sectors): with k = 16 on one lane per rating the
  // sweep ran at half the speed, k = 32 on two lanes 21% slower
  // (scripts/k_sweep.py, B200).  Beyond that, up to 4 float4 per lane keeps
  // several independent groups per warp and few shuffles per rating.
  const int f4 = kp / 4;  // float4 per row
  // rows of 3 * 2^j float4 (k = 24, 48, 96, 192, 384): 3 float4 per lane fit
  // exactly, where the power-of-two shape would predicate a quarter of the
  // lanes off (k = 96: SSE 4.2 ms vs 2.6 at k = 64 on C4; k = 24 on 2 lanes of
  // 3 beats 4 lanes of 2 with one masked: 4.06 vs 4.33 ms)
  if (f4 >= 6 && f4 % 3 == 0 && ((f4 / 3) & (f4 / 3 - 1)) == 0 && f4 / 3 <= 32)
    return {f4 / 3, 3};
  if (f4 <= 2) return {f4 < 1 ? 1 : f4, 1};
  int L = 4;
  while (L * 4 < f4 && L < 32) L <<= 1;
  int v4 = 1;
  while (v4 * L < f4) v4 <<= 1;
  return {L, v4};
}

#define BGMF_SHAPES(X)                                                                    \
  X(1, 1, false) X(2, 1, false) X(2, 3, false) X(4, 1, true) X(4, 1, false) X(4, 2, true) \
  X(4, 2, false)                                                                          \
  X(4, 3, false) X(4, 4, true) X(4, 4, false) X(8, 3, false) X(8, 4, true)                \
  X(8, 4, false) X(16, 3, false) X(16, 4, true) X(16, 4, false) X(32, 3, false)           \
  X(32, 4, true) X(32, 4, false)

// kp == 4*L*V4: every lane owns a full slice of the row, no predication
inline bool needs_mask(const Shape& sh, int kp) { return 4 * sh.L * sh.V4 != kp; }

// Lane geometry of a group.  kMask: the padded row kp is narrower than the
// group's 4*L*V4 floats, so some lanes/vectors sit past the row and are
// predicated off (only for odd k; k = 32/64/128 run unmasked).
template <int L, int V4, bool kMask>
struct Lanes {
  int gl, gbase;
  bool on_[V4];
  __device__ __forceinline__ Lanes(int kp) {
    const int lane = threadIdx.x & 31;
    gl = lane & (L - 1);
    gbase = lane & ~(L - 1);
#pragma unroll
    for (int q = 0; q < V4; ++q) on_[q] = !kMask || 4 * (q * L + gl) < kp;
  }
  __device__ __forceinline__ bool on(int q) const { return !kMask || on_[q]; }
  __device__ __forceinline__ int off(int q) const { return 4 * (q * L + gl); }
};

__device__ __forceinline__ float4 zero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }

__device__ __forceinline__ float2 lo2(const float4& a) { return make_float2(a.x, a.y); }
__device__ __forceinline__ float2 hi2(const float4& a) { return make_float2(a.z, a.w); }
__device__ __forceinline__ float4 cat4(const float2& a, const float2& b) {
  return make_float4(a.x, a.y, b.x, b.y);
}

// partial dot of the lane's slice with packed FFMA2 (two fp32 lanes per op)
template <int V4>
__device__ __forceinline__ float dot_slice(const float4 (&u)[V4], const float4 (&v)[V4]) {
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int q = 0; q < V4; ++q) {
    acc = __ffma2_rn(lo2(u[q]), lo2(v[q]), acc);
    acc = __ffma2_rn(hi2(u[q]), hi2(v[q]), acc);
  }
  return acc.x + acc.y;
}

// butterfly sum over the group's L lanes (every lane gets the same bits)
template <int L>
__device__ __forceinline__ float group_sum(float x) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// the same over a sub-warp mask (groups that run independently of the
// other groups of their warp: the ordered sweep)
template <int L>
__device__ __forceinline__ float group_sum_m(float x, unsigned mask) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) x += __shfl_xor_sync(mask, x, o);
  return x;
}

}  // namespace bgmf
