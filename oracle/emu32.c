/*
 * emu32.c -- the reference's sequential block sweep (_kernels.py:31-59,
 * entries in stored order, both updates from pre-update values) evaluated in
 * fp32 with the operation shapes of the GPU fast path.
 *
 * TEST INFRASTRUCTURE ONLY (like bgmf_oracle.c): nothing in the package links
 * or calls it.  tests/test_gpu_ordered.py uses it to show that the ordered
 * stratum kernel (csrc/ordered.cu) applies every update in the reference's
 * order: its factors must equal this sequential walk BIT FOR BIT.
 *
 * The GPU arithmetic restated (csrc/rows.cuh dot_slice/group_sum and the
 * update in ordered.cu): a group of L lanes, lane g holds float4s g, g+L, ...
 * (V4 of them; vectors past kp are zero); per lane two fp32 FMA chains
 * (x/z and y/w components... see dot_lane), the lane partial acc.x + acc.y,
 * then a butterfly over the lanes; e = x - dot; g = (2a) e; with nab = -(a b):
 * dv = fma(g, u, nab v), du = fma(g, v, nab u), u += du, v += dv (fp32,
 * nab v and nab u rounded first).  Build with -ffp-contract=off.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static float dot_group(const float* u, const float* v, int kp, int L, int V4) {
  float part[32];
  for (int g = 0; g < L; ++g) {
    float ax = 0.f, ay = 0.f;
    for (int q = 0; q < V4; ++q) {
      const int o = 4 * (q * L + g);
      const float u0 = o < kp ? u[o] : 0.f, u1 = o < kp ? u[o + 1] : 0.f;
      const float u2 = o < kp ? u[o + 2] : 0.f, u3 = o < kp ? u[o + 3] : 0.f;
      const float v0 = o < kp ? v[o] : 0.f, v1 = o < kp ? v[o + 1] : 0.f;
      const float v2 = o < kp ? v[o + 2] : 0.f, v3 = o < kp ? v[o + 3] : 0.f;
      ax = fmaf(u0, v0, ax);
      ay = fmaf(u1, v1, ay);
      ax = fmaf(u2, v2, ax);
      ay = fmaf(u3, v3, ay);
    }
    part[g] = ax + ay;
  }
  for (int o = L / 2; o > 0; o >>= 1) {
    float nx[32];
    for (int g = 0; g < L; ++g) nx[g] = part[g] + part[g ^ o];
    memcpy(part, nx, sizeof(float) * L);
  }
  return part[0];
}

/* One outer step: `iters` sweeps of every block of plan[0..nplan) in plan
 * order (blocks of a stratum are independent, so plan order is as good as
 * any), then -- per block, right after its sweeps -- the post-sweep SSE in
 * fp64.  U is n x kp, V is m x kp (fp32, padded rows).  Returns the first
 * plan position whose sweep met a non-finite residual, or -1. */
int64_t emu32_step(const int32_t* lrow, const int32_t* lcol, const float* val,
                   const int64_t* offsets, const int64_t* row_bounds, const int64_t* col_bounds,
                   int J, const int32_t* plan, int nplan, float* U, float* V, int kp, int L,
                   int V4, float alpha, float beta, int iters, double* sse_out) {
  const float two_a = 2.0f * alpha;
  const float nab = -alpha * beta;
  int64_t bad = -1;
  for (int p = 0; p < nplan; ++p) {
    const int b = plan[p];
    const int64_t beg = offsets[b], end = offsets[b + 1];
    float* Ub = U + row_bounds[b / J] * (int64_t)kp;
    float* Vb = V + col_bounds[b % J] * (int64_t)kp;
    for (int it = 0; it < iters; ++it)
      for (int64_t i = beg; i < end; ++i) {
        float* u = Ub + (int64_t)lrow[i] * kp;
        float* v = Vb + (int64_t)lcol[i] * kp;
        const float e = val[i] - dot_group(u, v, kp, L, V4);
        if (!isfinite(e) && bad < 0) bad = p;
        const float g = two_a * e;
        for (int j = 0; j < kp; ++j) {
          const float uo = u[j], vo = v[j];
          const float dv = fmaf(g, uo, nab * vo);
          const float du = fmaf(g, vo, nab * uo);
          u[j] = uo + du;
          v[j] = vo + dv;
        }
      }
    double s = 0.0;
    for (int64_t i = beg; i < end; ++i) {
      const float d = dot_group(Ub + (int64_t)lrow[i] * kp, Vb + (int64_t)lcol[i] * kp, kp, L, V4);
      const double ed = (double)val[i] - (double)d;
      s += ed * ed;
    }
    sse_out[b] = s;
  }
  return bad;
}
