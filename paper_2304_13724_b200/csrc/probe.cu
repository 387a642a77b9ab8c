// probe.cu -- the SM<->L2 ceiling of the sweep's access pattern.
//
// The sweep (sgd.cu) moves, per rating, one V row in (ld.global.cg, 4k bytes)
// and one V-row delta out (red.global.add.v4.f32, 4k bytes) against a V block
// that is L2-resident; its DRAM traffic is ~25x below its algorithmic bytes
// (profiles/r01_ncu_c4.md), so HBM is not its roofline.  This kernel issues
// exactly that traffic -- random rows of an L2-resident matrix, k floats per
// row, groups of L lanes with 16-byte vectors, no arithmetic dependency
// between rows, several rows in flight per group -- to measure what the SM->L2
// interface sustains for it on this GPU.  bench.py reports the sweep's
// achieved row bytes against this measured ceiling next to the HBM roofline.

#include <cooperative_groups.h>

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// mode 0: read rows; 1: read rows + reduce-add a delta into other rows;
// 2: reduce-add only; 3: two reads + one reduce per rating; 4: even warps do
// mode 1 over `ratings`, odd warps mode 0 over another `ratings` (a sweep and
// an SSE sharing the SMs).  L = 8 lanes x 4 float4 = 128 floats per row.
template <int MODE>
__device__ __forceinline__ void l2_probe_body(float* __restrict__ V, uint32_t rows,
                                              int64_t ratings, int64_t group, int64_t ngroups,
                                              int gl, float& acc);

template <int MODE>
__global__ void __launch_bounds__(256) l2_probe_kernel(float* __restrict__ V, uint32_t rows,
                                                       int64_t ratings, float* __restrict__ sink) {
  constexpr int L = 8;
  const int lane = threadIdx.x & 31, gl = lane & (L - 1);
  float acc = 0.f;
  if (MODE == 4) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t group = (gw >> 1) * (32 / L) + lane / L;
    const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / L / 2;
    if (gw & 1) l2_probe_body<0>(V, rows, ratings, group, ngroups, gl, acc);
    else l2_probe_body<1>(V, rows, ratings, group, ngroups, gl, acc);
  } else {
    const int64_t group = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / L;
    const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / L;
    l2_probe_body<MODE>(V, rows, ratings, group, ngroups, gl, acc);
  }
  if (acc == 12345.678f) sink[0] = acc;  // keeps the loads alive
}

template <int MODE>
__device__ __forceinline__ void l2_probe_body(float* __restrict__ V, uint32_t rows,
                                              int64_t ratings, int64_t group, int64_t ngroups,
                                              int gl, float& acc) {
  constexpr int L = 8, V4 = 4, D = 4;
  for (int64_t t0 = group * D; t0 < ratings; t0 += ngroups * D) {
    float4 v[D][V4];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const uint32_t c = mix32((uint32_t)(t0 + d)) % rows;
      const float4* row = reinterpret_cast<const float4*>(V + (int64_t)c * (4 * L * V4));
#pragma unroll
      for (int q = 0; q < V4; ++q) v[d][q] = MODE == 2 ? make_float4(1e-30f, 0.f, 0.f, 0.f)
                                                       : __ldcg(row + q * L + gl);
      if (MODE == 3) {  // a second, independent row read (the SSE's) per rating
        const uint32_t c2 = mix32((uint32_t)(t0 + d) ^ 0x5bd1e995u) % rows;
        const float4* row2 = reinterpret_cast<const float4*>(V + (int64_t)c2 * (4 * L * V4));
#pragma unroll
        for (int q = 0; q < V4; ++q) {
          const float4 w = __ldcg(row2 + q * L + gl);
          v[d][q].x += w.x; v[d][q].y += w.y; v[d][q].z += w.z; v[d][q].w += w.w;
        }
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (MODE == 1 || MODE == 2 || MODE == 3) {
        const uint32_t c = mix32((uint32_t)(t0 + d) ^ 0x9e3779b9u) % rows;
        float* row = V + (int64_t)c * (4 * L * V4);
#pragma unroll
        for (int q = 0; q < V4; ++q) {
          const float4 z = make_float4(v[d][q].x * 0.f, v[d][q].y * 0.f, v[d][q].z * 0.f,
                                       v[d][q].w * 0.f);
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + 4 * (q * L + gl)),
                       "f"(z.x), "f"(z.y), "f"(z.z), "f"(z.w)
                       : "memory");
        }
      } else {
#pragma unroll
        for (int q = 0; q < V4; ++q) acc += v[d][q].x + v[d][q].y + v[d][q].z + v[d][q].w;
      }
    }
  }
}

// DSMEM alternative to L2 for the sweep's V block: a
// cluster of CS CTAs holds one V block of `rows` rows x 128 floats in its
// distributed shared memory (row c in CTA c % CS).  Per rating a group reads
// one random row (ld through the mapped shared::cluster address) and -- the
// lossless update -- adds a delta into another random row with fp32 atomics
// (there is no vector red for shared::cluster).  MODE 5: remote rows
// (anywhere in the cluster); 6: rows of the CTA's own slice only (the best
// case: ratings pre-sorted by column slab); 7: remote reads only.
template <int CS, int MODE>
__global__ void __launch_bounds__(256) dsmem_probe_kernel(uint32_t rows, int64_t ratings,
                                                          float* __restrict__ sink) {
  namespace cg = cooperative_groups;
  constexpr int L = 8, V4 = 4, D = 4;
  extern __shared__ __align__(16) float slice[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank();
  const uint32_t per = (rows + CS - 1) / CS;  // rows held by each CTA
  for (uint32_t i = threadIdx.x; i < per * 128; i += blockDim.x) slice[i] = 0.f;
  cl.sync();
  const int lane = threadIdx.x & 31, gl = lane & (L - 1);
  const int64_t group = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / L;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / L;
  float acc = 0.f;
  for (int64_t t0 = group * D; t0 < ratings; t0 += ngroups * D) {
    float4 v[D][V4];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const uint32_t c = mix32((uint32_t)(t0 + d)) % rows;
      const unsigned owner = MODE == 6 ? me : c % CS;
      const float* base = cl.map_shared_rank(slice, owner);
      const float4* row = reinterpret_cast<const float4*>(base + (size_t)((c / CS) % per) * 128);
#pragma unroll
      for (int q = 0; q < V4; ++q) v[d][q] = row[q * L + gl];
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (MODE == 7) {
#pragma unroll
        for (int q = 0; q < V4; ++q) acc += v[d][q].x + v[d][q].y + v[d][q].z + v[d][q].w;
        continue;
      }
      const uint32_t c = mix32((uint32_t)(t0 + d) ^ 0x9e3779b9u) % rows;
      const unsigned owner = MODE == 6 ? me : c % CS;
      float* base = cl.map_shared_rank(slice, owner);
      float* row = base + (size_t)((c / CS) % per) * 128;
#pragma unroll
      for (int q = 0; q < V4; ++q) {
        float* p = row + 4 * (q * L + gl);
        atomicAdd(p, v[d][q].x * 0.f);
        atomicAdd(p + 1, v[d][q].y * 0.f);
        atomicAdd(p + 2, v[d][q].z * 0.f);
        atomicAdd(p + 3, v[d][q].w * 0.f);
      }
    }
  }
  cl.sync();  // no CTA leaves while others may still touch its slice
  if (acc == 12345.678f) sink[0] = acc;
}

template <int CS, int MODE>
cudaError_t launch_dsmem_probe(int sms, int ctas_per_sm, uint32_t rows, int64_t ratings,
                               float* sink) {
  const size_t smem = (size_t)((rows + CS - 1) / CS) * 128 * 4;
  cudaError_t e = cudaFuncSetAttribute(&dsmem_probe_kernel<CS, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && CS > 8)
    e = cudaFuncSetAttribute(&dsmem_probe_kernel<CS, MODE>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  int clusters = sms * (ctas_per_sm > 0 ? ctas_per_sm : 1) / CS;
  cfg.gridDim = dim3(clusters * CS);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int maxc = 0;
  if (cudaOccupancyMaxActiveClusters(&maxc, &dsmem_probe_kernel<CS, MODE>, &cfg) == cudaSuccess &&
      maxc > 0 && clusters > maxc)
    cfg.gridDim = dim3(maxc * CS);
  return cudaLaunchKernelEx(&cfg, &dsmem_probe_kernel<CS, MODE>, rows, ratings, sink);
}

}  // namespace
}  // namespace bgmf

using namespace bgmf;

// modes 5-7 (DSMEM, see dsmem_probe_kernel); `rows` = rows of one V block
// (C4: 1113), cluster size cs in {2, 4, 8, 16}.
extern "C" int bgmf_probe_dsmem(int device, int64_t rows, int64_t ratings, int mode, int cs,
                                int ctas_per_sm, double* ms_out) {
  if (!ms_out || rows < 1 || ratings < 1 || mode < 5 || mode > 7)
    return fail(nullptr, BGMF_ERR_ARG, "bgmf_probe_dsmem: bad argument");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* sink = nullptr;
  cudaEvent_t a = nullptr, b = nullptr;
  e = cudaMalloc(&sink, 4);
  if (e == cudaSuccess) e = cudaEventCreate(&a);
  if (e == cudaSuccess) e = cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4 && e == cudaSuccess; ++rep) {
    cudaEventRecord(a);
#define BGMF_DS(CSV)                                                                          \
  if (cs == CSV) {                                                                            \
    if (mode == 5) e = launch_dsmem_probe<CSV, 5>(sms, ctas_per_sm, (uint32_t)rows, ratings, sink); \
    else if (mode == 6) e = launch_dsmem_probe<CSV, 6>(sms, ctas_per_sm, (uint32_t)rows, ratings, sink); \
    else e = launch_dsmem_probe<CSV, 7>(sms, ctas_per_sm, (uint32_t)rows, ratings, sink);     \
  }
    BGMF_DS(2) BGMF_DS(4) BGMF_DS(8) BGMF_DS(16)
#undef BGMF_DS
    cudaEventRecord(b);
    if (e == cudaSuccess) e = cudaEventSynchronize(b);
    float ms = 0.f;
    if (e == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaFree(sink);
  if (a) cudaEventDestroy(a);
  if (b) cudaEventDestroy(b);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "bgmf_probe_dsmem");
  *ms_out = best;
  return BGMF_OK;
}

extern "C" int bgmf_probe_l2(int device, int64_t rows, int64_t ratings, int mode,
                             int ctas_per_sm, double* ms_out) {
  if (!ms_out || rows < 1 || rows > 0x7fffffff || ratings < 1 || mode < 0 || mode > 4)
    return fail(nullptr, BGMF_ERR_ARG, "bgmf_probe_l2: bad argument");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* V = nullptr;
  float* sink = nullptr;
  cudaEvent_t a = nullptr, b = nullptr;
  e = cudaMalloc(&V, (size_t)rows * 128 * 4);
  if (e == cudaSuccess) e = cudaMalloc(&sink, 4);
  if (e == cudaSuccess) e = cudaMemset(V, 0, (size_t)rows * 128 * 4);
  if (e == cudaSuccess) e = cudaEventCreate(&a);
  if (e == cudaSuccess) e = cudaEventCreate(&b);
  const dim3 grid(sms * (ctas_per_sm > 0 ? ctas_per_sm : 2));
  float best = 1e30f;
  for (int rep = 0; rep < 4 && e == cudaSuccess; ++rep) {
    cudaEventRecord(a);
    if (mode == 0) l2_probe_kernel<0><<<grid, 256>>>(V, (uint32_t)rows, ratings, sink);
    else if (mode == 1) l2_probe_kernel<1><<<grid, 256>>>(V, (uint32_t)rows, ratings, sink);
    else if (mode == 2) l2_probe_kernel<2><<<grid, 256>>>(V, (uint32_t)rows, ratings, sink);
    else if (mode == 3) l2_probe_kernel<3><<<grid, 256>>>(V, (uint32_t)rows, ratings, sink);
    else l2_probe_kernel<4><<<grid, 256>>>(V, (uint32_t)rows, ratings, sink);
    cudaEventRecord(b);
    e = cudaEventSynchronize(b);
    float ms = 0.f;
    if (e == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;  // rep 0 warms
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaFree(V);
  cudaFree(sink);
  if (a) cudaEventDestroy(a);
  if (b) cudaEventDestroy(b);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "bgmf_probe_l2");
  *ms_out = best;
  return BGMF_OK;
}
