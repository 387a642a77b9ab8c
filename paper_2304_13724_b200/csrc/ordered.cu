// ordered.cu -- order-faithful stratum sweep (fast mode, fp32).
//
// The reference sweeps a block's entries strictly in stored (row-major)
// order (reference pkg/src/blockmf/_kernels.py:42-55, partition.py:124).  An
// update reads and writes exactly one U row and one V row, so ANY execution
// that applies the updates of every U row in stored order and the updates of
// every V row in stored order computes the same values as the sequential
// walk -- bit for bit, given the same arithmetic.  This kernel is such an
// execution ("slab pipeline"):
//   * the block's columns are cut into S slabs; CTA s of the block (a
//     "stage") holds V slab s in shared memory for the whole launch: one TMA
//     bulk copy (cp.async.bulk) in, one bulk copy out;
//   * the stage's groups claim the block's rows in increasing order and
//     apply each row's entries that fall in slab s (ascending columns, u_r
//     in registers);
//   * column order: entry i of column c carries its rank q_i (earlier
//     entries of c in the block, built once per partition by
//     ensure_order_index); it waits until the column's shared-memory counter
//     equals q_i and releases q_i + 1 after its update;
//   * row order: a row visits its slabs in increasing order; each visit waits
//     until the row's flag (global memory, one word per U row) carries the
//     tag of the visit before it (previous slab of the row, or the previous
//     sweep's last slab), reads u_r, and publishes u_r and its own tag.
// Deadlock freedom: the earliest unfinished entry in stored order has all its
// predecessors done, and its row is claimed because every stage claims rows
// in order and all stages of a launch are resident (cooperative launch).
// Groups of one warp run independently (sub-warp masks; independent thread
// scheduling guarantees forward progress while a group spins).
// After the sweeps: a barrier over the block's stages, then the post-sweep
// SSE (_kernels.py:56) with V still in shared memory, summed in a fixed order
// (static row assignment, stages in order): the whole step is deterministic.

#include "bgmf_internal.cuh"
#include "rows.cuh"

namespace bgmf {
namespace {

constexpr int kOrdThreads = 1024;   // fp32 ordered kernel: 32 warps, <= 64 registers
constexpr int kExactThreads = 512;  // exact (fp64) kernel
constexpr int kOrdMaxBlocks = 96;
constexpr int kOrdMaxStages = 255;  // the row tag keeps slab + 1 in 8 bits
constexpr uint32_t kGenLimit = 1u << 24;

struct OrdBlock {
  int64_t begin;      // first entry of the block in the partition arrays
  int64_t rp;         // offset of the block's h + 1 row pointers in d_rowptr
  int64_t row_start;  // U row of local row 0
  int64_t col_start;  // V row (of vb) of local column 0
  float* vb;          // V (or a private copy of it)
  int32_t h, w;       // rows / columns of the block
  int32_t stage0, nstages;
  int32_t slab_w, block_id;
  int32_t pos;
  int32_t qbase;      // 1: column counters start at the unit's smallest rank
};

// Passed by value (kernel parameter space): the host never has to keep a
// table alive for launches still queued on the stream.
struct OrdLaunch {
  int32_t nblocks, pad;
  OrdBlock b[kOrdMaxBlocks];
};

__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
               : "=r"(v)
               : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(p)),
               "r"(v)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned mb, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(mb), "r"(parity)
      : "memory");
  return ok != 0;
}

// Every wait in these kernels is bounded: a schedule bug or a corrupted
// index array must fail the launch (an error the host reports), never hang
// the GPU.  20 s of %globaltimer, checked every 1024 polls.
struct SpinGuard {
  unsigned long long t0 = 0;
  unsigned n = 0;
  __device__ __forceinline__ void tick() {
    if ((++n & 1023u) != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (!t0) t0 = t;
    else if (t - t0 > 20000000000ull) __trap();
  }
};

// First index in [lo, hi) whose column is >= key (columns ascend within a
// row).  L-ary search: every lane probes one split point per round.
template <int L>
__device__ __forceinline__ int group_lower_bound(const int32_t* __restrict__ a, int lo, int hi,
                                                 int key, int gl, unsigned gmask) {
  while (hi - lo > L) {
    const int n = hi - lo;
    const int p = lo + (int)(((int64_t)(gl + 1) * n) / (L + 1));
    const unsigned bl = __ballot_sync(gmask, __ldg(a + p) < key) & gmask;
    const int c = __popc(bl);  // probes below the key: lanes 0 .. c-1
    const int nlo = c == 0 ? lo : lo + (int)(((int64_t)c * n) / (L + 1)) + 1;
    const int nhi = c == L ? hi : lo + (int)(((int64_t)(c + 1) * n) / (L + 1));
    lo = nlo;
    hi = nhi;
  }
  const bool less = lo + gl < hi && __ldg(a + lo + gl) < key;
  return lo + __popc(__ballot_sync(gmask, less) & gmask);
}

template <int V4, class LN>
__device__ __forceinline__ void load_row_l2(float4 (&dst)[V4], const float* row, const LN& ln) {
#pragma unroll
  for (int q = 0; q < V4; ++q)
    dst[q] = ln.on(q) ? __ldcg(reinterpret_cast<const float4*>(row + ln.off(q))) : zero4();
}

template <int V4, class LN>
__device__ __forceinline__ void load_row_smem(float4 (&dst)[V4], const float* row, const LN& ln) {
#pragma unroll
  for (int q = 0; q < V4; ++q)
    dst[q] = ln.on(q) ? *reinterpret_cast<const float4*>(row + ln.off(q)) : zero4();
}

template <int V4, class LN>
__device__ __forceinline__ void store_row_g(float* row, const float4 (&u)[V4], const LN& ln) {
#pragma unroll
  for (int q = 0; q < V4; ++q)
    if (ln.on(q)) *reinterpret_cast<float4*>(row + ln.off(q)) = u[q];
}

// Per-launch constants of a stage (one CTA).
struct Stage {
  const int32_t* rp;    // block row pointers
  const int32_t* bcol;  // block entries: local column, value, column rank
  const float* bval;
  const int32_t* bq;
  float* Ub;            // U rows of the block
  uint32_t* fl;         // row flags of those rows
  float* sv;            // V slab (shared memory)
  int* cnt;             // column counters of the slab (shared memory)
  int h, w, S, st, sw, cs, ce, nc, kp, qbase;
  int e0;               // first entry of the unit (block-relative)
};

// One sweep of this stage's slab (sweep `it` of the launch).
template <int L, int V4, bool kMask>
__device__ __forceinline__ void stage_sweep(const Stage& T, int it, uint32_t gen, float alpha,
                                            float beta, int pos, int* s_next,
                                            unsigned long long* bad, int* divflag) {
  const Lanes<L, V4, kMask> ln(T.kp);
  const unsigned gmask = L == 32 ? kFull : (((1u << L) - 1u) << ln.gbase);
  const float two_a = 2.0f * alpha;
  const float2 nab = make_float2(-alpha * beta, -alpha * beta);
  const int kp = T.kp;
  __syncthreads();  // this stage's previous sweep / SSE is over
  for (int i = threadIdx.x; i < T.nc; i += kOrdThreads) T.cnt[i] = T.qbase ? INT32_MAX : 0;
  if (threadIdx.x == 0) *s_next = 0;
  __syncthreads();
  if (T.qbase) {
    // a row range of a block: a column's first entry here has the rank of
    // the block's entries of that column before the range
    const int e0 = __ldg(T.rp), e1 = __ldg(T.rp + T.h);
    for (int i = e0 + (int)threadIdx.x; i < e1; i += kOrdThreads) {
      const int c = __ldg(T.bcol + i);
      if (c >= T.cs && c < T.ce) atomicMin(T.cnt + (c - T.cs), __ldg(T.bq + i));
    }
    __syncthreads();
  }
  const uint32_t tag_now = ((gen + (uint32_t)it) << 8) | (uint32_t)(T.st + 1);
  while (true) {
    int r = 0;
    if (ln.gl == 0) r = atomicAdd(s_next, 1);
    r = __shfl_sync(gmask, r, ln.gbase);
    if (r >= T.h) break;
    const int rb = __ldg(T.rp + r), re = __ldg(T.rp + r + 1);
    if (rb == re) continue;
    int lo = rb, hi = re;
    if (T.cs > 0) lo = group_lower_bound<L>(T.bcol, rb, re, T.cs, ln.gl, gmask);
    if (T.ce < T.w) hi = group_lower_bound<L>(T.bcol, lo, re, T.ce, ln.gl, gmask);
    if (lo == hi) continue;
    // row order (several stages): the visit before this one published u_r;
    // one stage: earlier sweeps are ordered by the CTA barrier
    uint32_t want = 0;
    if (T.S > 1) {
      if (lo > rb)
        want = ((gen + (uint32_t)it) << 8) | (uint32_t)(__ldg(T.bcol + lo - 1) / T.sw + 1);
      else if (it > 0)
        want = ((gen + (uint32_t)it - 1u) << 8) | (uint32_t)(__ldg(T.bcol + re - 1) / T.sw + 1);
    }
    if (want) {
      SpinGuard sg;
      while (!__all_sync(gmask, ld_acquire_gpu(T.fl + r) == want)) { __nanosleep(20); sg.tick(); }
    }
    float4 u[V4];
    load_row_l2<V4>(u, T.Ub + (int64_t)r * kp, ln);
    for (int t0 = lo; t0 < hi; t0 += L) {
      int cA = 0, qA = 0;
      float xA = 0.f;
      if (t0 + ln.gl < hi) {
        cA = __ldg(T.bcol + t0 + ln.gl);
        xA = __ldg(T.bval + t0 + ln.gl);
        qA = __ldg(T.bq + t0 + ln.gl);
      }
      const int nt = min(L, hi - t0);
      for (int j = 0; j < nt; ++j) {
        const int c = __shfl_sync(gmask, cA, ln.gbase + j) - T.cs;
        const float x = __shfl_sync(gmask, xA, ln.gbase + j);
        const int q = __shfl_sync(gmask, qA, ln.gbase + j);
        int* cp = T.cnt + c;
        // column order: every earlier entry of this column has been applied
        SpinGuard sg;
        while (!__all_sync(gmask, ld_acquire_cta(cp) == q)) sg.tick();
        float* vr = T.sv + (size_t)c * kp;
        float4 v[V4];
        load_row_smem<V4>(v, vr, ln);
        const float dot = group_sum_m<L>(dot_slice<V4>(u, v), gmask);
        const float e = x - dot;
        if (!isfinite(e) && ln.gl == 0) {
          atomicMin(bad, pack_bad(pos, it, t0 + j - T.e0));
          *divflag = 1;
        }
        const float gg = two_a * e;
        const float2 g2 = make_float2(gg, gg);
#pragma unroll
        for (int q4 = 0; q4 < V4; ++q4) {
          const float2 ul = lo2(u[q4]), uh = hi2(u[q4]), vl = lo2(v[q4]), vh = hi2(v[q4]);
          // the chunked kernel's operation shapes: dv = 2ae*u_old - ab*v,
          // du = 2ae*v - ab*u_old, then u + du, v + dv
          const float2 dvl = __ffma2_rn(g2, ul, __fmul2_rn(nab, vl));
          const float2 dvh = __ffma2_rn(g2, uh, __fmul2_rn(nab, vh));
          const float2 dul = __ffma2_rn(g2, vl, __fmul2_rn(nab, ul));
          const float2 duh = __ffma2_rn(g2, vh, __fmul2_rn(nab, uh));
          u[q4] = cat4(__fadd2_rn(ul, dul), __fadd2_rn(uh, duh));
          if (ln.on(q4))
            *reinterpret_cast<float4*>(vr + ln.off(q4)) =
                cat4(__fadd2_rn(vl, dvl), __fadd2_rn(vh, dvh));
        }
        __syncwarp(gmask);
        if (ln.gl == 0) st_release_cta(cp, q + 1);
      }
    }
    store_row_g<V4>(T.Ub + (int64_t)r * kp, u, ln);
    if (T.S > 1) {
      // publish u_r: the group's stores are ordered before lane 0's release by
      // the warp barrier (bar.warp.sync orders memory among its threads) and a
      // release is cumulative over what precedes it -- the pattern of
      // cooperative groups' grid sync (bar.sync, then one thread's fence and
      // flag).  One release per visit, no full fence.sc (and its L1
      // invalidation) on every lane before it.
      __syncwarp(gmask);
      if (ln.gl == 0) st_release_gpu(T.fl + r, tag_now);
    }
  }
}

// This stage's share of the block's post-sweep SSE: rows g, g + NG, ...
// (static assignment), groups of a warp in order, warps in order.  The total
// is valid in thread 0.
template <int L, int V4, bool kMask>
__device__ __forceinline__ double stage_sse(const Stage& T, double* s_red) {
  constexpr int NG = kOrdThreads / L;
  const Lanes<L, V4, kMask> ln(T.kp);
  const unsigned gmask = L == 32 ? kFull : (((1u << L) - 1u) << ln.gbase);
  const int kp = T.kp;
  double acc = 0.0;
  for (int r = (int)threadIdx.x / L; r < T.h; r += NG) {
    const int rb = __ldg(T.rp + r), re = __ldg(T.rp + r + 1);
    if (rb == re) continue;
    int lo = rb, hi = re;
    if (T.cs > 0) lo = group_lower_bound<L>(T.bcol, rb, re, T.cs, ln.gl, gmask);
    if (T.ce < T.w) hi = group_lower_bound<L>(T.bcol, lo, re, T.ce, ln.gl, gmask);
    if (lo == hi) continue;
    float4 u[V4];
    load_row_l2<V4>(u, T.Ub + (int64_t)r * kp, ln);
    for (int t0 = lo; t0 < hi; t0 += L) {
      int cA = 0;
      float xA = 0.f;
      if (t0 + ln.gl < hi) {
        cA = __ldg(T.bcol + t0 + ln.gl);
        xA = __ldg(T.bval + t0 + ln.gl);
      }
      const int nt = min(L, hi - t0);
      for (int j = 0; j < nt; ++j) {
        const int c = __shfl_sync(gmask, cA, ln.gbase + j) - T.cs;
        const float x = __shfl_sync(gmask, xA, ln.gbase + j);
        float4 v[V4];
        load_row_smem<V4>(v, T.sv + (size_t)c * kp, ln);
        const float dot = group_sum_m<L>(dot_slice<V4>(u, v), gmask);
        const double ed = (double)x - (double)dot;
        acc += ed * ed;
      }
    }
  }
  __syncwarp();
  double wsum = 0.0;
#pragma unroll
  for (int j = 0; j < 32 / L; ++j) wsum += __shfl_sync(kFull, acc, j * L);
  __syncthreads();  // s_red may still be read by the previous call's thread 0
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = wsum;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kOrdThreads / 32; ++w) tot += s_red[w];
  return tot;
}

// Barrier over the block's S stages (all co-resident): barrier number k of
// the launch completes when the counter reaches (k + 1) * S.
__device__ __forceinline__ void block_barrier(uint32_t* ctr, int S, uint32_t k) {
  __syncthreads();
  if (S > 1) {
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1u);
      SpinGuard sg;
      while (ld_acquire_gpu(ctr) < (k + 1u) * (uint32_t)S) { __nanosleep(64); sg.tick(); }
    }
    __syncthreads();
  }
}

// The block's SSE: every stage's partial, summed in stage order by every
// stage (the same bits everywhere).  Valid in thread 0.
template <int L, int V4, bool kMask>
__device__ __forceinline__ double block_sse_all(const Stage& T, double* s_red, double* part,
                                                int stage0, uint32_t* ctr, uint32_t& nbar,
                                                double* s_bcast) {
  const double mine = stage_sse<L, V4, kMask>(T, s_red);
  if (T.S == 1) {
    if (threadIdx.x == 0) *s_bcast = mine;
    __syncthreads();
    return *s_bcast;
  }
  if (threadIdx.x == 0) part[stage0 + T.st] = mine;
  block_barrier(ctr, T.S, nbar++);
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int s2 = 0; s2 < T.S; ++s2) sum += __ldcg(part + stage0 + s2);
    *s_bcast = sum;
  }
  __syncthreads();
  return *s_bcast;
}

// conv = 0: `iters` sweeps, then the post-sweep SSE (sgd_sweeps,
// _kernels.py:31-59).  conv = 1: ConvergeEachBlock on the device
// (sgd_converge, _kernels.py:62-100): sse_before, then sweeps until the
// block's RMSE improvement drops below tol or `iters` (the cap) sweeps ran;
// iters_used / capped per block to conv_out[2 * block_id + 0 / 1].
template <int L, int V4, bool kMask>
__global__ void __launch_bounds__(kOrdThreads, 1)
ordered_kernel(const __grid_constant__ OrdLaunch P, const int32_t* __restrict__ lcol,
               const float* __restrict__ val, const int32_t* __restrict__ qrank,
               const int32_t* __restrict__ rowptr, float* __restrict__ U,
               int kp, float alpha, float beta, int iters, uint32_t gen,
               uint32_t* __restrict__ rflag, uint32_t* __restrict__ bar,
               double* __restrict__ part, double* __restrict__ sse,
               unsigned long long* __restrict__ bad, int conv, double tol,
               int64_t* __restrict__ conv_out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_next;
  __shared__ int s_div;
  __shared__ double s_red[kOrdThreads / 32];
  __shared__ double s_bcast;
  __shared__ __align__(8) unsigned long long s_mbar;

  int bi = 0;
  {
    int lo = 0, hi = P.nblocks - 1;  // last block with stage0 <= blockIdx.x
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.b[mid].stage0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    bi = lo;
  }
  const OrdBlock B = P.b[bi];
  Stage T;
  T.S = B.nstages;
  T.st = (int)blockIdx.x - B.stage0;
  T.sw = B.slab_w;
  T.cs = T.st * T.sw;
  T.ce = min(T.cs + T.sw, B.w);
  T.nc = T.ce - T.cs;
  T.h = B.h;
  T.w = B.w;
  T.kp = kp;
  T.rp = rowptr + B.rp;
  T.bcol = lcol + B.begin;
  T.bval = val + B.begin;
  T.bq = qrank + B.begin;
  T.Ub = U + B.row_start * kp;
  T.fl = rflag + B.row_start;
  T.sv = reinterpret_cast<float*>(smem);
  T.cnt = reinterpret_cast<int*>(T.sv + (size_t)T.sw * kp);
  uint32_t* ctr = bar + 3 * bi;      // barrier counter, arrivals at the end, divergence
  const unsigned bytes = (unsigned)T.nc * (unsigned)kp * 4u;
  float* gv = B.vb + (B.col_start + T.cs) * kp;
  T.qbase = B.qbase;
  T.e0 = __ldg(T.rp);
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&s_mbar);
  const unsigned sva = (unsigned)__cvta_generic_to_shared(T.sv);

  // V slab -> shared memory (TMA bulk copy, completion on an mbarrier)
  if (threadIdx.x == 0) {
    s_div = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && bytes > 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sva),
        "l"(gv), "r"(bytes), "r"(mb)
        : "memory");
  }
  if (bytes > 0) {
    SpinGuard sg;
    while (!mbar_try_wait(mb, 0)) sg.tick();
  }

  uint32_t nbar = 0;
  int swept = 0;
  double sse_now = 0.0;
  const double cntd = (double)(__ldg(T.rp + T.h) - __ldg(T.rp));  // entries of the unit
  if (!conv) {
    for (int it = 0; it < iters; ++it)
      stage_sweep<L, V4, kMask>(T, it, gen, alpha, beta, B.pos, &s_next, bad, &s_div);
    swept = iters;
    if (swept > 0) block_barrier(ctr, T.S, nbar++);  // every stage done: U is final
  } else {
    // sse_before, then sweep -> SSE -> improvement test, all on the device
    sse_now = block_sse_all<L, V4, kMask>(T, s_red, part, B.stage0, ctr, nbar, &s_bcast);
    double rmse_prev = sqrt(sse_now / cntd);
    bool capped = true;
    while (swept < iters) {
      stage_sweep<L, V4, kMask>(T, swept, gen, alpha, beta, B.pos, &s_next, bad, &s_div);
      ++swept;
      __syncthreads();
      if (threadIdx.x == 0 && s_div && T.S > 1) atomicOr(ctr + 2, 1u);
      block_barrier(ctr, T.S, nbar++);
      // a non-finite residual anywhere in the block ends its loop
      if (threadIdx.x == 0) s_bcast = (double)(T.S > 1 ? ld_acquire_gpu(ctr + 2) : 0u) + (double)s_div;
      __syncthreads();
      const bool diverged = s_bcast != 0.0;
      __syncthreads();
      if (diverged) { capped = false; break; }
      sse_now = block_sse_all<L, V4, kMask>(T, s_red, part, B.stage0, ctr, nbar, &s_bcast);
      if (!isfinite(sse_now)) {  // _kernels.py:88-89: (count - 1, iters - 1)
        if (threadIdx.x == 0 && T.st == 0)
          atomicMin(bad, pack_bad(B.pos, swept - 1, (int64_t)cntd - 1));
        capped = false;
        break;
      }
      const double rmse_now = sqrt(sse_now / cntd);
      if (rmse_prev - rmse_now < tol) { capped = false; break; }
      rmse_prev = rmse_now;
    }
    if (threadIdx.x == 0 && T.st == 0) {
      conv_out[2 * B.block_id] = swept;
      conv_out[2 * B.block_id + 1] = capped ? 1 : 0;
    }
  }

  // V slab back to global memory (TMA bulk store)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && bytes > 0 && swept > 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gv),
                 "r"(sva), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  if (!conv) sse_now = block_sse_all<L, V4, kMask>(T, s_red, part, B.stage0, ctr, nbar, &s_bcast);
  if (threadIdx.x == 0) {
    if (T.st == 0) sse[B.block_id] = sse_now;
    if (T.S > 1) {
      // the last stage out resets the block's counters for the next launch
      const unsigned done = atomicAdd(ctr + 1, 1u);
      if (done == (unsigned)T.S - 1) {
        ctr[0] = 0u;
        ctr[1] = 0u;
        ctr[2] = 0u;
      }
    }
    if (bytes > 0 && swept > 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// ---- exact mode: the same schedule in fp64, bit-identical ---------------
// The ordered schedule applies the updates of every U and V row in stored
// order, so with the reference's own arithmetic it reproduces the reference
// bit for bit -- in parallel across rows and columns (round 1's exact kernel
// walked each block on one thread).  Per rating, lane 0 of the warp runs the
// residual chain e = x - u0 v0 - u1 v1 - ... with separately rounded fp64
// products and subtractions (numba fastmath=False, _kernels.py:44-48); the
// lanes then update the k elements in parallel in the reference's order of
// operations (u + a(2e v - b u), _kernels.py:51-55).  u_r is staged in the
// warp's shared-memory row for the row's run, V in the stage's slab.  The
// post-sweep SSE (_kernels.py:16-28) is a sequential sum: every entry's
// (x - u.v)^2 is computed in parallel into `esq`, then one thread adds them
// in stored order.
// e = x - u0 v0 - u1 v1 - ... in the reference's order with separately rounded
// products (_kernels.py:44-48).  The products do not depend on the chain, so
// lane g computes u_g v_g for its elements in parallel and every lane runs the
// subtraction chain over them in g order, the operands broadcast by shuffles
// that issue ahead of the chain: the serial part is k dependent DADDs, not k
// shared-memory load pairs + DMUL + DADD on one lane.  Same bits on all lanes.
__device__ __forceinline__ double exact_residual(double x, const double* us, const double* vs,
                                                 int k, int lane) {
  double e = x;
  for (int j = 0; j * 32 < k; ++j) {
    const int g = j * 32 + lane;
    const double p = g < k ? __dmul_rn(us[g], vs[g]) : 0.0;
    if (k - j * 32 >= 32) {
#pragma unroll
      for (int l = 0; l < 32; ++l) e = __dsub_rn(e, __shfl_sync(kFull, p, l));
    } else {
      for (int l = 0; l < k - j * 32; ++l) e = __dsub_rn(e, __shfl_sync(kFull, p, l));
    }
  }
  return e;
}

__device__ __forceinline__ void exact_stage_sweep(const Stage& T, double* sv, double* urow,
                                                  const double* __restrict__ bval,
                                                  double* __restrict__ Ub, int it, uint32_t gen,
                                                  double alpha, double beta, int pos,
                                                  int* s_next, unsigned long long* bad,
                                                  int* divflag) {
  const int lane = threadIdx.x & 31;
  const int k = T.kp;
  double* us = urow + (threadIdx.x >> 5) * k;
  __syncthreads();
  for (int i = threadIdx.x; i < T.nc; i += kExactThreads) T.cnt[i] = T.qbase ? INT32_MAX : 0;
  if (threadIdx.x == 0) *s_next = 0;
  __syncthreads();
  if (T.qbase) {
    const int e0 = __ldg(T.rp), e1 = __ldg(T.rp + T.h);
    for (int i = e0 + (int)threadIdx.x; i < e1; i += kExactThreads) {
      const int c = __ldg(T.bcol + i);
      if (c >= T.cs && c < T.ce) atomicMin(T.cnt + (c - T.cs), __ldg(T.bq + i));
    }
    __syncthreads();
  }
  const uint32_t tag_now = ((gen + (uint32_t)it) << 8) | (uint32_t)(T.st + 1);
  while (true) {
    int r = 0;
    if (lane == 0) r = atomicAdd(s_next, 1);
    r = __shfl_sync(kFull, r, 0);
    if (r >= T.h) break;
    const int rb = __ldg(T.rp + r), re = __ldg(T.rp + r + 1);
    if (rb == re) continue;
    int lo = rb, hi = re;
    if (T.cs > 0) lo = group_lower_bound<32>(T.bcol, rb, re, T.cs, lane, kFull);
    if (T.ce < T.w) hi = group_lower_bound<32>(T.bcol, lo, re, T.ce, lane, kFull);
    if (lo == hi) continue;
    uint32_t want = 0;
    if (T.S > 1) {
      if (lo > rb)
        want = ((gen + (uint32_t)it) << 8) | (uint32_t)(__ldg(T.bcol + lo - 1) / T.sw + 1);
      else if (it > 0)
        want = ((gen + (uint32_t)it - 1u) << 8) | (uint32_t)(__ldg(T.bcol + re - 1) / T.sw + 1);
    }
    if (want) {
      SpinGuard sg;
      while (!__all_sync(kFull, ld_acquire_gpu(T.fl + r) == want)) { __nanosleep(20); sg.tick(); }
    }
    double* ug = Ub + (int64_t)r * k;
    for (int g = lane; g < k; g += 32) us[g] = __ldcg(ug + g);
    __syncwarp();
    for (int t0 = lo; t0 < hi; t0 += 32) {
      int cA = 0, qA = 0;
      double xA = 0.0;
      if (t0 + lane < hi) {
        cA = __ldg(T.bcol + t0 + lane);
        xA = __ldg(bval + t0 + lane);
        qA = __ldg(T.bq + t0 + lane);
      }
      const int nt = min(32, hi - t0);
      for (int j = 0; j < nt; ++j) {
        const int c = __shfl_sync(kFull, cA, j) - T.cs;
        const double x = __shfl_sync(kFull, xA, j);
        const int q = __shfl_sync(kFull, qA, j);
        int* cp = T.cnt + c;
        SpinGuard sg;
        while (!__all_sync(kFull, ld_acquire_cta(cp) == q)) sg.tick();
        double* vs = sv + (size_t)c * k;
        const double e = exact_residual(x, us, vs, k, lane);
        if (!isfinite(e) && lane == 0) {
          atomicMin(bad, pack_bad(pos, it, t0 + j - T.e0));
          *divflag = 1;
        }
        const double e2 = __dmul_rn(2.0, e);
        for (int g = lane; g < k; g += 32) {
          const double u0 = us[g], v0 = vs[g];
          us[g] = __dadd_rn(u0, __dmul_rn(alpha, __dsub_rn(__dmul_rn(e2, v0), __dmul_rn(beta, u0))));
          vs[g] = __dadd_rn(v0, __dmul_rn(alpha, __dsub_rn(__dmul_rn(e2, u0), __dmul_rn(beta, v0))));
        }
        __syncwarp();
        if (lane == 0) st_release_cta(cp, q + 1);
      }
    }
    for (int g = lane; g < k; g += 32) ug[g] = us[g];
    if (T.S > 1) {  // publish u_r (the release pattern of ordered_kernel's row visits)
      __syncwarp();
      if (lane == 0) st_release_gpu(T.fl + r, tag_now);
    }
    __syncwarp();
  }
}

// (x - u.v)^2 of every entry of this stage's slab into esq (entry order is
// irrelevant: the sum below is sequential)
__device__ __forceinline__ void exact_stage_esq(const Stage& T, const double* sv, double* urow,
                                                const double* __restrict__ bval,
                                                const double* __restrict__ Ub,
                                                double* __restrict__ besq) {
  const int lane = threadIdx.x & 31;
  const int k = T.kp;
  for (int r = (int)threadIdx.x / 32; r < T.h; r += kExactThreads / 32) {
    const int rb = __ldg(T.rp + r), re = __ldg(T.rp + r + 1);
    if (rb == re) continue;
    int lo = rb, hi = re;
    if (T.cs > 0) lo = group_lower_bound<32>(T.bcol, rb, re, T.cs, lane, kFull);
    if (T.ce < T.w) hi = group_lower_bound<32>(T.bcol, lo, re, T.ce, lane, kFull);
    if (lo == hi) continue;
    // the row's u into this warp's shared-memory row, so the per-lane chains
    // below read it with LDS (unrolled, issued ahead of the DSUB chain)
    // instead of one dependent L2 load per element
    const double* ug = Ub + (int64_t)r * k;
    double* us = urow + (threadIdx.x >> 5) * k;
    __syncwarp();
    for (int g = lane; g < k; g += 32) us[g] = __ldcg(ug + g);
    __syncwarp();
    for (int i = lo + lane; i < hi; i += 32) {
      const double* vs = sv + (size_t)(__ldg(T.bcol + i) - T.cs) * k;
      double e = __ldg(bval + i);
#pragma unroll 8
      for (int g = 0; g < k; ++g) e = __dsub_rn(e, __dmul_rn(us[g], vs[g]));
      besq[i] = __dmul_rn(e, e);
    }
  }
}

// The block's SSE, summed in stored order by one thread; every stage gets it.
__device__ __forceinline__ double exact_block_sse(const Stage& T, const double* sv, double* urow,
                                                  const double* __restrict__ bval,
                                                  const double* __restrict__ Ub,
                                                  double* __restrict__ besq, double* part,
                                                  int stage0, uint32_t* ctr, uint32_t& nbar,
                                                  double* s_bcast) {
  exact_stage_esq(T, sv, urow, bval, Ub, besq);
  block_barrier(ctr, T.S, nbar++);  // every stage's terms are written
  if (T.st == 0 && threadIdx.x < 32) {
    // the stored-order sum s += esq[i] (_kernels.py:16-28) by one warp: tiles
    // of 32 terms loaded coalesced PF tiles ahead, then added in order from
    // shuffles -- every lane runs the same DADD chain (same bits), which is
    // then the only serial part (one thread with one L2 load per term before)
    const int lane = threadIdx.x;
    const int e0 = __ldg(T.rp), e1 = __ldg(T.rp + T.h);
    constexpr int PF = 8;
    double buf[PF];
#pragma unroll
    for (int p = 0; p < PF; ++p) {
      const int i = e0 + p * 32 + lane;
      buf[p] = i < e1 ? __ldcg(besq + i) : 0.0;
    }
    double s = 0.0;
    for (int t = e0; t < e1; t += 32 * PF) {
#pragma unroll
      for (int p = 0; p < PF; ++p) {
        const int base = t + p * 32;
        const double cur = buf[p];
        const int ni = base + PF * 32 + lane;
        buf[p] = ni < e1 ? __ldcg(besq + ni) : 0.0;
        const int n = min(32, e1 - base);
        if (n == 32) {
#pragma unroll
          for (int l = 0; l < 32; ++l) s = __dadd_rn(s, __shfl_sync(kFull, cur, l));
        } else {
          for (int l = 0; l < n; ++l) s = __dadd_rn(s, __shfl_sync(kFull, cur, l));
        }
      }
    }
    if (lane == 0) {
      part[stage0] = s;
      *s_bcast = s;
    }
  }
  if (T.S > 1) {
    block_barrier(ctr, T.S, nbar++);
    if (threadIdx.x == 0) *s_bcast = __ldcg(part + stage0);
  }
  __syncthreads();
  return *s_bcast;
}

__global__ void __launch_bounds__(kExactThreads, 1)
ordered_exact_kernel(const __grid_constant__ OrdLaunch P, const int32_t* __restrict__ lcol,
                     const double* __restrict__ val, const int32_t* __restrict__ qrank,
                     const int32_t* __restrict__ rowptr, double* __restrict__ U, int k,
                     double alpha, double beta, int iters, uint32_t gen,
                     uint32_t* __restrict__ rflag, uint32_t* __restrict__ bar,
                     double* __restrict__ part, double* __restrict__ esq,
                     double* __restrict__ sse, unsigned long long* __restrict__ bad, int conv,
                     double tol, int64_t* __restrict__ conv_out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_next;
  __shared__ int s_div;
  __shared__ double s_bcast;
  __shared__ __align__(8) unsigned long long s_mbar;
  int bi = 0;
  {
    int lo = 0, hi = P.nblocks - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.b[mid].stage0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    bi = lo;
  }
  const OrdBlock B = P.b[bi];
  Stage T;
  T.S = B.nstages;
  T.st = (int)blockIdx.x - B.stage0;
  T.sw = B.slab_w;
  T.cs = T.st * T.sw;
  T.ce = min(T.cs + T.sw, B.w);
  T.nc = T.ce - T.cs;
  T.h = B.h;
  T.w = B.w;
  T.kp = k;
  T.rp = rowptr + B.rp;
  T.bcol = lcol + B.begin;
  T.bq = qrank + B.begin;
  T.fl = rflag + B.row_start;
  T.qbase = B.qbase;
  T.e0 = __ldg(T.rp);
  double* sv = reinterpret_cast<double*>(smem);
  T.cnt = reinterpret_cast<int*>(sv + (size_t)T.sw * k);
  double* urow = reinterpret_cast<double*>(smem + (((size_t)T.sw * k * 8 + (size_t)T.sw * 4 + 15) & ~(size_t)15));
  const double* bval = val + B.begin;
  double* Ub = U + B.row_start * k;
  double* besq = esq + B.begin;
  uint32_t* ctr = bar + 3 * bi;
  double* gv = reinterpret_cast<double*>(B.vb) + (B.col_start + T.cs) * k;
  // TMA bulk copies need 16-byte aligned addresses and sizes: rows of odd k
  // doubles are not, so those slabs move with plain loads / stores
  const bool bulk = ((reinterpret_cast<uintptr_t>(gv) | ((size_t)T.nc * k * 8)) & 15) == 0;
  const unsigned bytes = bulk ? (unsigned)T.nc * (unsigned)k * 8u : 0u;
  if (!bulk)
    for (int i = threadIdx.x; i < T.nc * k; i += kExactThreads) sv[i] = __ldcg(gv + i);
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&s_mbar);
  const unsigned sva = (unsigned)__cvta_generic_to_shared(sv);
  if (threadIdx.x == 0) {
    s_div = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && bytes > 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sva),
        "l"(gv), "r"(bytes), "r"(mb)
        : "memory");
  }
  if (bytes > 0) {
    SpinGuard sg;
    while (!mbar_try_wait(mb, 0)) sg.tick();
  }
  uint32_t nbar = 0;
  int swept = 0;
  double sse_now = 0.0;
  const double cntd = (double)(__ldg(T.rp + T.h) - __ldg(T.rp));
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  if (!conv) {
    for (int it = 0; it < iters; ++it)
      exact_stage_sweep(T, sv, urow, bval, Ub, it, gen, alpha, beta, B.pos, &s_next, bad, &s_div);
    swept = iters;
    block_barrier(ctr, T.S, nbar++);  // every stage done: U is final
    sse_now = exact_block_sse(T, sv, urow, bval, Ub, besq, part, B.stage0, ctr, nbar, &s_bcast);
    if (!isfinite(sse_now) && threadIdx.x == 0 && T.st == 0)  // _kernels.py:56-58
      atomicMin(bad, pack_bad(B.pos, iters - 1, (int64_t)cntd - 1));
  } else {
    sse_now = exact_block_sse(T, sv, urow, bval, Ub, besq, part, B.stage0, ctr, nbar, &s_bcast);
    double rmse_prev = sqrt(sse_now / cntd);
    bool capped = true;
    while (swept < iters) {
      exact_stage_sweep(T, sv, urow, bval, Ub, swept, gen, alpha, beta, B.pos, &s_next, bad,
                        &s_div);
      ++swept;
      __syncthreads();
      if (threadIdx.x == 0 && s_div && T.S > 1) atomicOr(ctr + 2, 1u);
      block_barrier(ctr, T.S, nbar++);
      if (threadIdx.x == 0) s_bcast = (double)(T.S > 1 ? ld_acquire_gpu(ctr + 2) : 0u) + (double)s_div;
      __syncthreads();
      const bool diverged = s_bcast != 0.0;
      __syncthreads();
      if (diverged) { capped = false; sse_now = nan; break; }
      sse_now = exact_block_sse(T, sv, urow, bval, Ub, besq, part, B.stage0, ctr, nbar, &s_bcast);
      if (!isfinite(sse_now)) {
        if (threadIdx.x == 0 && T.st == 0)
          atomicMin(bad, pack_bad(B.pos, swept - 1, (int64_t)cntd - 1));
        capped = false;
        break;
      }
      const double rmse_now = sqrt(sse_now / cntd);
      if (rmse_prev - rmse_now < tol) { capped = false; break; }
      rmse_prev = rmse_now;
    }
    if (threadIdx.x == 0 && T.st == 0) {
      conv_out[2 * B.block_id] = swept;
      conv_out[2 * B.block_id + 1] = capped ? 1 : 0;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && bytes > 0 && swept > 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gv),
                 "r"(sva), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  if (!bulk && swept > 0)
    for (int i = threadIdx.x; i < T.nc * k; i += kExactThreads) gv[i] = sv[i];
  if (threadIdx.x == 0) {
    if (T.st == 0) sse[B.block_id] = sse_now;
    if (T.S > 1) {
      const unsigned done = atomicAdd(ctr + 1, 1u);
      if (done == (unsigned)T.S - 1) {
        ctr[0] = 0u;
        ctr[1] = 0u;
        ctr[2] = 0u;
      }
    }
    if (bytes > 0 && swept > 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// ---- order index (once per partition) ---------------------------------
__device__ __forceinline__ int block_of(const int64_t* __restrict__ off, int nb, int64_t i) {
  int lo = 0, hi = nb - 1;  // last b with off[b] <= i
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void rank_keys(const int32_t* __restrict__ lcol, const int64_t* __restrict__ off,
                          int nb, int64_t n, int cbits, uint64_t* __restrict__ keys,
                          uint32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = ((uint64_t)block_of(off, nb, i) << cbits) | (uint32_t)lcol[i];
    idx[i] = (uint32_t)i;
  }
}

// keys sorted by (block, column), stable: a run's first position per key
__global__ void rank_heads(const uint64_t* __restrict__ keys, int64_t n,
                           uint32_t* __restrict__ first) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    if (p == 0 || keys[p - 1] != keys[p]) first[keys[p]] = (uint32_t)p;
}

__global__ void rank_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                             const uint32_t* __restrict__ first, int64_t n,
                             int32_t* __restrict__ q) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    q[idx[p]] = (int32_t)((uint32_t)p - first[keys[p]]);
}

// Row pointers of every block (relative to the block's first entry): the
// entry that starts row r (or the first entry after an empty run of rows)
// writes the pointers of the rows it closes.
__global__ void row_pointers(const int32_t* __restrict__ lrow, const int64_t* __restrict__ off,
                             const int64_t* __restrict__ rpo, int nb, int64_t n,
                             int32_t* __restrict__ rowptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = block_of(off, nb, i);
    const int64_t beg = off[b], end = off[b + 1];
    const int r = lrow[i];
    const int prev = i > beg ? lrow[i - 1] : -1;
    int32_t* rp = rowptr + rpo[b];
    for (int rr = prev + 1; rr <= r; ++rr) rp[rr] = (int32_t)(i - beg);
    if (i == end - 1) {
      const int h = (int)(rpo[b + 1] - rpo[b] - 1);
      for (int rr = r + 1; rr <= h; ++rr) rp[rr] = (int32_t)(end - beg);
    }
  }
}

// Shape of the ordered kernel's groups.  warp = 1: one group per warp (L =
// 32, up to 4 float4 per lane), so a group spinning on a column counter or a
// row flag never shares its warp with the group it waits for.
Shape ordered_shape(int kp, int warp) {
  if (!warp) return shape_for(kp);
  const int f4 = kp / 4;
  int v4 = 1;
  while (32 * v4 < f4) ++v4;
  return {32, v4};
}

#define BGMF_ORD_SHAPES(X)                                                              \
  BGMF_SHAPES(X) X(32, 1, true) X(32, 1, false) X(32, 2, true) X(32, 2, false) X(32, 3, true)

#define BGMF_ORD(LL, VV, MM)                                           \
  if (sh.L == LL && sh.V4 == VV && mk == MM)                           \
    return reinterpret_cast<const void*>(&ordered_kernel<LL, VV, MM>);
const void* ordered_kernel_ptr(int kp, int warp) {
  const Shape sh = ordered_shape(kp, warp);
  const bool mk = needs_mask(sh, kp);
  BGMF_ORD_SHAPES(BGMF_ORD)
  return nullptr;
}
#undef BGMF_ORD

// Shared memory of a stage: the V slab and its column counters; exact mode
// (fp64 rows of k) adds one staged u row per warp.
size_t slab_smem(bgmf_ctx* c, int cols) {
  if (!c->exact) return (size_t)cols * ((size_t)c->kp * 4 + 4);
  const size_t slab = ((size_t)cols * ((size_t)c->k * 8 + 4) + 15) & ~(size_t)15;
  return slab + (size_t)(kExactThreads / 32) * c->k * 8;
}
size_t row_bytes(bgmf_ctx* c) { return c->exact ? (size_t)c->k * 8 + 4 : (size_t)c->kp * 4 + 4; }
size_t fixed_smem(bgmf_ctx* c) {
  return c->exact ? 16 + (size_t)(kExactThreads / 32) * c->k * 8 : 0;
}

// Largest dynamic shared memory a CTA may ask for (static smem aside).
size_t smem_budget(bgmf_ctx* c) {
  static int optin = 0;
  if (!optin) cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
  const size_t stat = 1024;  // s_next, s_red, s_mbar + slack
  return optin > (int)stat ? (size_t)optin - stat : 0;
}

const void* stage_kernel_ptr(bgmf_ctx* c) {
  return c->exact ? reinterpret_cast<const void*>(&ordered_exact_kernel)
                  : ordered_kernel_ptr(c->kp, c->ord_warp);
}

// co-resident CTAs of the (fp32 or exact) ordered kernel with `smem` bytes
int ordered_capacity(bgmf_ctx* c, size_t smem) {
  const void* fn = stage_kernel_ptr(c);
  if (!fn) return 0;
  const uint64_t key = ((uint64_t)c->kp << 34) | ((uint64_t)c->exact << 33) |
                       ((uint64_t)c->ord_warp << 32) | (uint64_t)smem;
  auto it = c->ord_cap.find(key);
  if (it != c->ord_cap.end()) return it->second;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_budget(c));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, c->exact ? kExactThreads : kOrdThreads,
                                                smem);
  c->ord_cap[key] = per_sm * c->num_sms;
  return per_sm * c->num_sms;
}

}  // namespace

void order_release(bgmf_ctx* c) {
  dfree(c->d_qrank, c->stream);
  dfree(c->d_rowptr, c->stream);
  dfree(c->d_rflag, c->stream);
  dfree(c->d_obar, c->stream);
  dfree(c->d_conv, c->stream);
  c->d_conv = nullptr;
  dfree(c->d_opart, c->stream);
  dfree(c->d_esq, c->stream);
  c->d_esq = nullptr;
  c->d_qrank = c->d_rowptr = nullptr;
  c->d_rflag = c->d_obar = nullptr;
  c->d_opart = nullptr;
  c->h_rp.clear();
  c->ord_ready = false;
}

int sort_pairs_device(bgmf_ctx* ctx, uint64_t** keys, uint32_t** vals, int64_t n, int bits,
                      int lo_bit = 0);

// Column ranks and row pointers of the resident partition (once per
// partition; ~24 B per rating of temporaries).
int ensure_order_index(bgmf_ctx* c) {
  if (c->ord_ready) return BGMF_OK;
  if (!c->partitioned) return fail(c, BGMF_ERR_STATE, "no partition");
  cudaStream_t s = c->stream;
  const int nb = c->I * c->J;
  const int64_t n = c->nnz;
  c->h_rp.assign(nb + 1, 0);
  for (int b = 0; b < nb; ++b) {
    const int bi = b / c->J;
    c->h_rp[b + 1] = c->h_rp[b] + (c->row_bounds[bi + 1] - c->row_bounds[bi]) + 1;
  }
  int bbits = 0;
  while (bbits < 31 && (1ll << bbits) < nb) ++bbits;
  const int key_bits = bbits + c->cbits;
  int64_t *d_off = nullptr, *d_rpo = nullptr;
  uint64_t* keys = nullptr;
  uint32_t *idx = nullptr, *first = nullptr;
  auto cleanup = [&]() {
    dfree(d_off, s); dfree(d_rpo, s); dfree(keys, s); dfree(idx, s); dfree(first, s);
  };
  const size_t N = (size_t)(n > 0 ? n : 1);
  cudaError_t e = dmalloc(&c->d_qrank, N * 4, s);
  if (e == cudaSuccess) e = dmalloc(&c->d_rowptr, (size_t)c->h_rp[nb] * 4, s);
  if (e == cudaSuccess) e = dmalloc(&c->d_rflag, (size_t)(c->n > 0 ? c->n : 1) * 4, s);
  if (e == cudaSuccess) e = dmalloc(&c->d_obar, (size_t)3 * kOrdMaxBlocks * 4, s);
  if (e == cudaSuccess) e = dmalloc(&c->d_conv, (size_t)2 * (nb > 0 ? nb : 1) * 8, s);
  if (e == cudaSuccess) e = dmalloc(&c->d_opart, (size_t)8192 * 8, s);
  if (e == cudaSuccess) e = dmalloc(&d_off, (size_t)(nb + 1) * 8, s);
  if (e == cudaSuccess) e = dmalloc(&d_rpo, (size_t)(nb + 1) * 8, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_rflag, 0, (size_t)(c->n > 0 ? c->n : 1) * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_obar, 0, (size_t)3 * kOrdMaxBlocks * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_rowptr, 0, (size_t)c->h_rp[nb] * 4, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_off, c->h_offsets.data(), (size_t)(nb + 1) * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_rpo, c->h_rp.data(), (size_t)(nb + 1) * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && n > 0) e = dmalloc(&keys, N * 8, s);
  if (e == cudaSuccess && n > 0) e = dmalloc(&idx, N * 4, s);
  if (e == cudaSuccess && n > 0) e = dmalloc(&first, ((size_t)nb << c->cbits) * 4, s);
  if (e != cudaSuccess) {
    cleanup();
    order_release(c);
    return cuda_fail(c, e, "ensure_order_index");
  }
  const int grid = c->num_sms * 8;
  if (n > 0) {
    rank_keys<<<grid, 256, 0, s>>>(c->d_lcol, d_off, nb, n, c->cbits, keys, idx);
    int rc = sort_pairs_device(c, &keys, &idx, n, key_bits);
    if (rc) { cleanup(); order_release(c); return rc; }
    rank_heads<<<grid, 256, 0, s>>>(keys, n, first);
    rank_scatter<<<grid, 256, 0, s>>>(keys, idx, first, n, c->d_qrank);
    row_pointers<<<grid, 256, 0, s>>>(c->d_lrow, d_off, d_rpo, nb, n, c->d_rowptr);
  }
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cleanup();
  if (e != cudaSuccess) { order_release(c); return cuda_fail(c, e, "ensure_order_index"); }
  c->ord_gen = 1;
  c->ord_ready = true;
  return BGMF_OK;
}

// Can the ordered kernel take block b (its V block in <= kOrdMaxStages
// slabs that each fit a CTA, all of them co-resident, row pointers in int32)?
bool ordered_block_ok(bgmf_ctx* c, int b) {
  if (c->streaming || !stage_kernel_ptr(c)) return false;
  const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
  if (cnt >= INT32_MAX) return false;
  const int64_t w = c->col_bounds[b % c->J + 1] - c->col_bounds[b % c->J];
  const size_t budget = smem_budget(c);
  if (budget <= fixed_smem(c)) return false;
  const int64_t per = (int64_t)((budget - fixed_smem(c)) / row_bytes(c));
  if (per < 1) return false;
  const int64_t smin = (w + per - 1) / per;
  if (smin > kOrdMaxStages) return false;
  const int cap = ordered_capacity(c, slab_smem(c, (int)((w + smin - 1) / smin)));
  return smin <= cap;
}

namespace {

// One unit of the ordered kernel: a block of the partition (or a CPMF row
// shard of the 1 x 1 block with its private V copy).
struct OrdItem {
  OrdBlock ob;
  int64_t cnt;
  size_t smem;
};

// Stage count of an item with w columns and cnt ratings, `items` units in
// the launch: enough slabs for one to fit a CTA; more while the batch leaves
// SMs idle, at ~ord_stage_ratings ratings per stage (a row then visits more
// slabs: each visit moves u_r through L2).
void plan_stages(bgmf_ctx* c, OrdItem& it, int items) {
  const int64_t per = (int64_t)((smem_budget(c) - fixed_smem(c)) / row_bytes(c));
  const int64_t w = it.ob.w;
  const int64_t smin = (w + per - 1) / per;
  int64_t S = (it.cnt + c->ord_stage_ratings - 1) / c->ord_stage_ratings;
  // co-residency allows ord_fill_ctas stages per SM (1024-thread CTAs: at most 2)
  const int64_t fill = (int64_t)c->num_sms * c->ord_fill_ctas / (items > 0 ? items : 1);
  if (S > fill) S = fill;
  if (S < smin) S = smin;
  if (S > w) S = w;
  if (S > kOrdMaxStages) S = kOrdMaxStages;
  if (S < 1) S = 1;
  const int64_t swd = (w + S - 1) / S;
  it.ob.nstages = (int32_t)((w + swd - 1) / swd);  // no empty slab
  it.ob.slab_w = (int32_t)swd;
  it.smem = slab_smem(c, (int)swd);
}

// Launch the items: as few cooperative launches as co-residency allows.
int launch_items(bgmf_ctx* c, std::vector<OrdItem>& items, int iters, float alpha, float beta,
                 bool conv, double tol, double* sse_dev, double alpha64 = 0.0,
                 double beta64 = 0.0) {
  cudaStream_t s = c->stream;
  const void* fn = stage_kernel_ptr(c);
  const size_t budget = smem_budget(c);
  if (c->exact && !c->d_esq) BGMF_CK(c, dmalloc(&c->d_esq, (size_t)(c->nnz > 0 ? c->nnz : 1) * 8, s));
  size_t i = 0;
  while (i < items.size()) {
    // pack units into one launch while every stage stays co-resident
    OrdLaunch L{};
    size_t smem = 0;
    int ctas = 0;
    size_t j = i;
    double ratings = 0;
    while (j < items.size() && L.nblocks < kOrdMaxBlocks) {
      const size_t sm2 = std::max(smem, items[j].smem);
      if (ctas + items[j].ob.nstages > ordered_capacity(c, sm2) && L.nblocks > 0) break;
      OrdBlock& ob = L.b[L.nblocks++];
      ob = items[j].ob;
      ob.stage0 = ctas;
      ctas += ob.nstages;
      ratings += (double)items[j].cnt;
      smem = sm2;
      ++j;
    }
    if (ctas > ordered_capacity(c, smem) || ctas > 8192)
      return fail(c, BGMF_ERR_STATE, "ordered sweep: block does not fit the GPU");
    if (c->ord_gen + (uint32_t)iters + 1u >= kGenLimit) {
      BGMF_CK(c, cudaMemsetAsync(c->d_rflag, 0, (size_t)c->n * 4, s));
      c->ord_gen = 1;
    }
    uint32_t gen = c->ord_gen;
    c->ord_gen += (uint32_t)(iters > 0 ? iters : 1);  // converge: iters = the cap
    const int32_t* lcol = c->d_lcol;
    const float* val = c->d_val;
    const int32_t* qr = c->d_qrank;
    const int32_t* rpp = c->d_rowptr;
    float* U = c->d_u;
    int kp = c->kp, its = iters;
    uint32_t* rfl = c->d_rflag;
    uint32_t* bar = c->d_obar;
    double* part = c->d_opart;
    double* sse = sse_dev;
    unsigned long long* bad = c->d_bad;
    int cv = conv ? 1 : 0;
    int64_t* cout = c->d_conv;
    void* args[] = {&L, &lcol, &val, &qr, &rpp, &U, &kp, &alpha, &beta, &its, &gen,
                    &rfl, &bar, &part, &sse, &bad, &cv, &tol, &cout};
    // exact: fp64 values, U and arithmetic (ordered_exact_kernel)
    const double* val64 = c->d_val64;
    double* U64 = c->d_u64;
    int k = c->k;
    double a64 = alpha64, b64 = beta64;
    double* esq = c->d_esq;
    void* args64[] = {&L, &lcol, &val64, &qr, &rpp, &U64, &k, &a64, &b64, &its, &gen,
                      &rfl, &bar, &part, &esq, &sse, &bad, &cv, &tol, &cout};
    TimedLaunch* slot = nullptr;
    if (c->timing) record_begin(c, 0, ratings * iters * (12.0 + 16.0 * c->k), &slot);
    BGMF_CK(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)budget));
    BGMF_CK(c, cudaLaunchCooperativeKernel(fn, dim3(ctas),
                                           dim3(c->exact ? kExactThreads : kOrdThreads),
                                           c->exact ? args64 : args, smem, s));
    if (slot) record_end(c, slot);
    i = j;
  }
  return BGMF_OK;
}

}  // namespace

// One batch (stratum, or part of one) through the ordered kernel: `iters`
// sweeps (or, conv, the converge loop capped at iters) and the post-sweep
// SSE of every block in plan[q0 .. q1) (plan positions pos_base + q).  The
// caller has checked use_ordered.
int run_batch_ordered(bgmf_ctx* c, const int32_t* plan, int q0, int q1, int pos_base,
                      int iters, float alpha, float beta, bool conv, double tol,
                      double alpha64, double beta64) {
  int rc = ensure_order_index(c);
  if (rc) return rc;
  std::vector<OrdItem> items;
  for (int q = q0; q < q1; ++q) {
    const int b = plan[q];
    const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
    if (cnt == 0) continue;  // its SSE stays 0
    const int bi = b / c->J, bj = b % c->J;
    OrdItem it{};
    it.cnt = cnt;
    it.ob.begin = c->h_offsets[b];
    it.ob.rp = c->h_rp[b];
    it.ob.row_start = c->row_bounds[bi];
    it.ob.col_start = c->col_bounds[bj];
    it.ob.vb = c->exact ? reinterpret_cast<float*>(c->d_v64) : c->d_v;
    it.ob.h = (int32_t)(c->row_bounds[bi + 1] - c->row_bounds[bi]);
    it.ob.w = (int32_t)(c->col_bounds[bj + 1] - c->col_bounds[bj]);
    it.ob.block_id = b;
    it.ob.pos = pos_base + q;
    it.ob.qbase = 0;
    items.push_back(it);
  }
  for (auto& it : items) plan_stages(c, it, (int)items.size());
  return launch_items(c, items, iters, alpha, beta, conv, tol, c->d_sse, alpha64, beta64);
}

// CPMF shards (baselines.py:100-182) through the ordered kernel: shard w =
// rows [r0[w], r1[w]) of the 1 x 1 partition, swept in stored order on the
// shared U and its private V copy vpriv + w * m * kp; SSE to sse_dev[w].
int run_shards_ordered(bgmf_ctx* c, const int32_t* r0, const int32_t* r1, const int64_t* edges,
                       int nshards, float* vpriv, float alpha, float beta, double* sse_dev) {
  int rc = ensure_order_index(c);
  if (rc) return rc;
  std::vector<OrdItem> items;
  for (int w = 0; w < nshards; ++w) {
    if (r1[w] <= r0[w]) continue;
    OrdItem it{};
    it.cnt = edges[w + 1] - edges[w];  // sets the stage count as for a block of that size
    it.ob.begin = 0;
    it.ob.rp = c->h_rp[0] + r0[w];
    it.ob.row_start = r0[w];
    it.ob.col_start = 0;
    it.ob.vb = vpriv ? vpriv + (size_t)w * c->m * c->kp : c->d_v;
    it.ob.h = r1[w] - r0[w];
    it.ob.w = (int32_t)c->m;
    it.ob.block_id = w;
    it.ob.pos = w;
    it.ob.qbase = 1;  // column ranks count the earlier shards' entries too
    items.push_back(it);
  }
  for (auto& it : items) plan_stages(c, it, (int)items.size());
  return launch_items(c, items, 1, alpha, beta, false, 0.0, sse_dev);
}

// Routing of one batch.  ord_mode 1: ordered whenever every block fits;
// 0: never; -1 (auto): ordered when it fits and the chunked sweep would
// distort the reference order -- a dense block (> 1/8 of its cells rated:
// rows share their columns and concurrent chunks collide on every V row),
// chunks shorter than ord_row_split mean rows of a block, or more than
// ord_col_conc concurrent groups per V row (chunked_splits_rows).  Every
// fast-mode drift past 1e-3 in the randomised sweeps
// was in one of these; C1-C5 single-GPU strata are in none.  Ring ranks set
// ord_col_conc = 6 (their 2-block launches of C4 run up to 4.0 groups per V
// row -- block_chunk's (ratings per column - 32) / 80 -- measured within
// 2e-5, and the randomised ring sweeps cover worlds 2-4).  ConvergeEachBlock
// routes the same way; both paths run its per-block loop on the device (the
// ordered kernel in-launch, the chunked one as a CUDA-graph WHILE node).
// Exact mode: always the ordered schedule when it fits (fp64, bit-identical).
//
// The auto rule's risk test alone (no feasibility): would the chunked sweep
// of this batch distort the reference order (a dense block, split rows, or
// too many groups per V row)?
bool order_risky(bgmf_ctx* c, const int32_t* plan, int q0, int q1) {
  int nonempty = 0;
  bool dense = false;
  for (int q = q0; q < q1; ++q) {
    const int b = plan[q];
    const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
    if (cnt == 0) continue;
    ++nonempty;
    const int64_t h = c->row_bounds[b / c->J + 1] - c->row_bounds[b / c->J];
    const int64_t w = c->col_bounds[b % c->J + 1] - c->col_bounds[b % c->J];
    dense |= cnt * 8 > h * w;
  }
  return dense || (nonempty > 0 && chunked_splits_rows(c, plan, q0, q1, c->ord_row_split,
                                                       c->ord_col_conc));
}

bool use_ordered(bgmf_ctx* c, const int32_t* plan, int q0, int q1, bool converge) {
  if (c->ord_mode == 0 || c->streaming) return false;
  if (c->exact) {  // fp64: the ordered schedule is the reference's, bit for bit
    for (int q = q0; q < q1; ++q)
      if (c->h_offsets[plan[q] + 1] > c->h_offsets[plan[q]] && !ordered_block_ok(c, plan[q]))
        return false;
    return true;
  }
  for (int q = q0; q < q1; ++q)
    if (c->h_offsets[plan[q] + 1] > c->h_offsets[plan[q]] && !ordered_block_ok(c, plan[q]))
      return false;
  if (c->ord_mode > 0) return true;
  (void)converge;  // ConvergeEachBlock routes like fixed schedules: both paths loop on the device
  return order_risky(c, plan, q0, q1);
}

}  // namespace bgmf
