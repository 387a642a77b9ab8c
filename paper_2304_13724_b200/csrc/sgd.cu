// sgd.cu -- per-stratum SGD kernels (reference pkg/src/blockmf/_kernels.py).
//
// Fast path (default, fp32):  a "group" of L lanes owns one rating at a time;
// each lane holds V4 float4 of the (padded) latent vector, so kp = 4*L*V4.
// The blocks of one batch (a stratum of plan_step, scheduler.py:45-75) are
// cut into contiguous row-major chunks, one chunk per group:
//   * rating triples are read coalesced, L at a time, and broadcast with shfl;
//   * u_r stays in registers for the whole run of ratings of user r (entries
//     are sorted row-major, partition.py:124), so within a chunk the U updates
//     are exactly sequential; the run is written back with a plain store, or
//     -- when the run crosses a chunk boundary -- with red.add of its delta;
//   * v_c is read with 128-bit loads and its delta alpha*(2e*u - beta*v) is
//     applied with red.global.add.v4.f32 (lossless: no update is ever lost,
//     reads may be stale by the few concurrent groups on the same block);
//   * the dot product is a butterfly xor-shuffle over the L lanes;
//   * factor rows are read with ld.global.cg (L2, never a stale L1 line):
//     V is L2-resident (C4: 9.1 MB of 126 MB) and the reds resolve in L2.
// Update rule per entry (_kernels.py:44-55): e = x - u.v;
//   u <- u + a(2e v - b u);  v <- v + a(2e u_old - b v)  (both pre-update).
// The post-sweep SSE of every block (_kernels.py:56, consumed by the trace,
// trainer.py:149-158) is a second kernel over the same chunks.
//
// Exact path (fp64, opt-in): one thread walks a whole block sequentially
// with explicitly rounded __dmul_rn/__dsub_rn/__dadd_rn in the reference's
// operation order -- bit-identical to numba's fastmath=False loops.  Blocks of
// a batch are independent, so the batch is still parallel across blocks.

#include <cooperative_groups.h>

#include <cmath>
#include <string>
#include <utility>

#include <atomic>

#include "bgmf_internal.cuh"
#include "rows.cuh"

namespace bgmf {
namespace {

namespace cg = cooperative_groups;

__device__ __forceinline__ void red_add_v4(float* p, float4 d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(d.x), "f"(d.y),
               "f"(d.z), "f"(d.w)
               : "memory");
}

// Bulk asynchronous reduction (TMA engine): global[dst .. dst+bytes) +=
// shared[src ..], fp32 adds performed at L2.  Issued by one lane for a whole
// V-row delta, it replaces that group's per-lane REDG traffic through L1TEX.
__device__ __forceinline__ void bulk_red_add(float* gdst, const float* ssrc, unsigned bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                   gdst),
               "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Programmatic dependent launch: a sweep / SSE kernel lets the next one be
// scheduled as soon as SMs free up (trigger), and waits for the previous
// grid's completion and memory before touching factors (wait); the work table
// and ratings it reads first are not written by that grid.  Without the
// launch attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// smem ring of V-row deltas per group for the bulk path
constexpr int kBulkBufs = 4;

__device__ __forceinline__ int find_work(const BlockWork* __restrict__ work, int nwork, int c) {
  int lo = 0, hi = nwork - 1;  // last w with first_chunk <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (work[mid].first_chunk <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}


// Chunk geometry shared by the sweep and SSE kernels.
struct Chunk {
  int64_t begin, end, bbeg, bend;
  int64_t row_start, col_start;
  int block_id, pos;
  int w;     // work item
  int iter;  // the work item's device-side iteration, or -1 (the launch's)
};

__device__ __forceinline__ Chunk locate_chunk(const BlockWork* __restrict__ work, int nwork,
                                              int total_chunks, int chunk) {
  Chunk ch{0, 0, 0, 0, 0, 0, 0, 0, -1, -1};
  if (chunk < total_chunks) {
    const int w = find_work(work, nwork, chunk);
    ch.w = w;
    const BlockWork bw = work[w];
    ch.begin = bw.begin + (int64_t)(chunk - bw.first_chunk) * bw.chunk_len;
    ch.end = min(ch.begin + (int64_t)bw.chunk_len, bw.end);
    ch.bbeg = bw.begin;
    ch.bend = bw.end;
    ch.row_start = bw.row_start;
    ch.col_start = bw.col_start;
    ch.block_id = bw.block_id;
    ch.pos = bw.pos;
    if (bw.active && !*((volatile const int32_t*)bw.active)) ch.end = ch.begin;  // converged
    ch.iter = bw.iter ? *((volatile const int32_t*)bw.iter) : -1;
  }
  return ch;
}


// Dynamic chunking (the sweep's dyn_split option): the static one-wave table
// (chunk_len, first_chunk per work item, T0 chunks) is cut D ways.  Warp slot s
// covers GPW consecutive static chunk indices of phase p = s / ceil(T0 / GPW):
// static chunk j of block w becomes its sub-chunks [p n_w, (p + 1) n_w) of
// length ceil(chunk_len / D), so within a phase each block has as many groups
// on it as in the static wave (the per-block concurrency floors still hold)
// and only the last phase's short chunks form the tail.
__device__ __forceinline__ Chunk locate_dyn(const BlockWork* __restrict__ work, int nwork,
                                            int total_chunks, int dyn_d, int slot, int g,
                                            int gpw) {
  Chunk ch{0, 0, 0, 0, 0, 0, 0, 0, -1, -1};
  const int per_phase = (total_chunks + gpw - 1) / gpw;
  const int p = slot / per_phase;
  const int j = (slot - p * per_phase) * gpw + g;
  if (p < dyn_d && j < total_chunks) {
    const int w = find_work(work, nwork, j);
    ch.w = w;
    const BlockWork bw = work[w];
    const int64_t cnt = bw.end - bw.begin;
    const int64_t n0 = (cnt + bw.chunk_len - 1) / bw.chunk_len;
    const int64_t cl = ((int64_t)bw.chunk_len + dyn_d - 1) / dyn_d;
    const int64_t idx = (int64_t)p * n0 + (j - bw.first_chunk);
    ch.begin = min(bw.begin + idx * cl, bw.end);
    ch.end = min(ch.begin + cl, bw.end);
    ch.bbeg = bw.begin;
    ch.bend = bw.end;
    ch.row_start = bw.row_start;
    ch.col_start = bw.col_start;
    ch.block_id = bw.block_id;
    ch.pos = bw.pos;
    if (bw.active && !*((volatile const int32_t*)bw.active)) ch.end = ch.begin;  // converged
    ch.iter = bw.iter ? *((volatile const int32_t*)bw.iter) : -1;
  }
  return ch;
}

// Rating triple of entry i.  cbits < 0: SoA int32 row / int32 col arrays;
// cbits >= 0: packed 4-byte (row << cbits | col) records in `lrow` (the
// out-of-core stream format, 8 B per rating with the fp32 value), the low 8
// bits the column bits; bit 8: `val` holds 1-byte integer codes (5 B/rating).
__device__ __forceinline__ void load_triple(const int32_t* __restrict__ lrow,
                                            const int32_t* __restrict__ lcol,
                                            const float* __restrict__ val, int cbits, int64_t i,
                                            int& r, int& c, float& x) {
  if (cbits < 0) {
    r = __ldg(lrow + i);
    c = __ldg(lcol + i);
    x = __ldg(val + i);
  } else {
    const int cb = cbits & 0xFF;
    const uint32_t rc = (uint32_t)__ldg(lrow + i);
    r = (int)(rc >> cb);
    c = (int)(rc & ((1u << cb) - 1u));
    x = (cbits & 0x100) ? (float)__ldg(reinterpret_cast<const uint8_t*>(val) + i)
                        : __ldg(val + i);
  }
}

__device__ __forceinline__ int load_rowidx(const int32_t* __restrict__ lrow, int cbits,
                                           int64_t i) {
  return cbits < 0 ? __ldg(lrow + i) : (int)((uint32_t)__ldg(lrow + i) >> (cbits & 0xFF));
}

// Run-aligned chunk edges (the sweep's snap option): a nominal chunk edge P
// inside a user run moves forward to that run's end when it lies within
// `cap` entries, so the run is walked by one group (U stays in registers, no
// per-rating U red.add, no re-reads) instead of being straddled.  A pure
// function of P: the chunk ending at P and the one starting there agree.
// Group-parallel (ballots over L entries); all warp lanes execute it.
template <int L>
__device__ __forceinline__ int64_t snap_edge(const int32_t* __restrict__ lrow, int cbits,
                                             int64_t P, int64_t lo, int64_t hi, int cap) {
  const int lane = threadIdx.x & 31, gl = lane & (L - 1), gbase = lane & ~(L - 1);
  const bool inside = P > lo && P < hi;
  const int prev = inside ? load_rowidx(lrow, cbits, P - 1) : 0;
  bool open = inside && load_rowidx(lrow, cbits, P) == prev;  // P splits a run
  int64_t out = P;
  for (int base = 1; base < cap; base += L) {
    const int64_t i = P + base + gl;
    const bool edge = open && (i >= hi || load_rowidx(lrow, cbits, min(i, hi - 1)) != prev);
    const unsigned m = (__ballot_sync(0xffffffffu, edge) >> gbase) & (L == 32 ? 0xffffffffu : ((1u << L) - 1u));
    if (open && m) {
      out = min(P + base + (int64_t)(__ffs(m) - 1), hi);
      open = false;
    }
  }
  return out;  // still open: the run is longer than cap, keep the straddle
}

// U-row L2 prefetch (upf; routed by u_prefetch): when a triple batch is loaded, each
// lane whose rating starts a user run asks the TMA unit to pull that run's U
// row into L2 (cp.async.bulk.prefetch, no registers, no completion), so the
// register load at the run switch L..2L ratings later hits L2, not DRAM.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int L>
__device__ __forceinline__ void prefetch_runs(const float* Ub, int row, int kp, bool valid) {
  const int gl = (threadIdx.x & 31) & (L - 1);
  const int prev = __shfl_up_sync(0xffffffffu, row, 1);
  if (valid && (gl == 0 || prev != row)) prefetch_l2(Ub + (int64_t)row * kp, (unsigned)kp * 4u);
}

// L2-coherent 128-bit load (the factors are written by other SMs during the
// kernel; ld.global.cg never returns a stale L1 line).
__device__ __forceinline__ float4 ld_cg(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}

template <int V4, class LN>
__device__ __forceinline__ void load_row(float4 (&dst)[V4], const float* row, const LN& ln) {
#pragma unroll
  for (int q = 0; q < V4; ++q) dst[q] = ln.on(q) ? ld_cg(row + ln.off(q)) : zero4();
}

// Read-only rows (no writer during the kernel): ld.global.nc.
template <int V4, class LN>
__device__ __forceinline__ void load_row_ro(float4 (&dst)[V4], const float* row, const LN& ln) {
#pragma unroll
  for (int q = 0; q < V4; ++q)
    dst[q] = ln.on(q) ? __ldg(reinterpret_cast<const float4*>(row + ln.off(q))) : zero4();
}

template <int V4, class LN>
__device__ __forceinline__ void store_row(float* row, const float4 (&u)[V4], const LN& ln) {
#pragma unroll
  for (int q = 0; q < V4; ++q)
    if (ln.on(q)) *reinterpret_cast<float4*>(row + ln.off(q)) = u[q];
}


// Software-pipelined walk over one chunk.  While rating t is computed, the
// triple of t+1 is already in registers (the next L triples are prefetched a
// batch ahead), its V row is in flight, and -- when t+1 starts a new user run
// -- so is its U row.  kSweep: SGD update; else: accumulate (x - u.v)^2.
// A user run that continues into a neighbour chunk ("shared") applies each
// rating's U delta with red.add as it goes; an interior run is stored once.
// The update is the reference's  u += a(2e v - b u),  v += a(2e u_old - b v)
// evaluated as t = 2ae*v - ab*u (FFMA2 of an FMUL2) and u + t, in packed fp32.
// All lanes of the warp execute the same trip count (maxlen) so the shuffles
// stay converged; groups past their chunk end are predicated off.
// MODE 0: plain; 1 (bulk): V deltas through the TMA bulk reduce; 2 (uring):
// the U row of a run starting UD ratings ahead is requested into a per-lane
// shared-memory ring by cp.async (sbuf = this thread's slice), so short user
// runs -- skewed or very sparse blocks, ~1-3 ratings per run -- do not wait a
// DRAM round trip at every run switch (the register prefetch leads by one
// rating only).
template <int L, int V4, bool kMask, bool kSweep, int MODE = 0>
__device__ __forceinline__ double walk_chunk(const Chunk& ch, int maxlen,
                                             const int32_t* __restrict__ lrow,
                                             const int32_t* __restrict__ lcol,
                                             const float* __restrict__ val, float* U, float* V,
                                             int kp, float alpha, float beta, int iter,
                                             unsigned long long* bad, int cbits = -1,
                                             float* sbuf = nullptr, bool upf = false) {
  constexpr bool kBulk = MODE == 1;
  constexpr bool kURing = MODE == 2 && kSweep && L >= 4;
  constexpr int UD = L >= 8 ? 4 : 3;  // ring depth (needs UD < L: rows from batches A, B)
  const Lanes<L, V4, kMask> ln(kp);
  int nbulk = 0;  // bulk ops issued by this group (ring position)
  const int len = (int)(ch.end - ch.begin);
  float* Ub = U + ch.row_start * kp;
  float* Vb = V + ch.col_start * kp;
  int first_row = -1, last_row = -1;
  if (kSweep && len > 0) {
    const int fr = load_rowidx(lrow, cbits, ch.begin);
    const int lr = load_rowidx(lrow, cbits, ch.end - 1);
    if (ch.begin > ch.bbeg && load_rowidx(lrow, cbits, ch.begin - 1) == fr) first_row = fr;
    if (ch.end < ch.bend && load_rowidx(lrow, cbits, ch.end) == lr) last_row = lr;
  }
  // triple batches A (current) and B (next)
  int rA = 0, cA = 0, rB = 0, cB = 0;
  float xA = 0.f, xB = 0.f;
  if (ln.gl < len) load_triple(lrow, lcol, val, cbits, ch.begin + ln.gl, rA, cA, xA);
  if (L + ln.gl < len) load_triple(lrow, lcol, val, cbits, ch.begin + L + ln.gl, rB, cB, xB);
  if (upf) prefetch_runs<L>(Ub, rB, kp, L + ln.gl < len);
  int r = __shfl_sync(kFull, rA, ln.gbase);
  int c = __shfl_sync(kFull, cA, ln.gbase);
  float x = __shfl_sync(kFull, xA, ln.gbase);
  float4 u[V4], v[V4];
  if (len > 0) {
    load_row<V4>(u, Ub + (int64_t)r * kp, ln);
    load_row<V4>(v, Vb + (int64_t)c * kp, ln);
  } else {
#pragma unroll
    for (int q = 0; q < V4; ++q) u[q] = v[q] = zero4();
  }
  bool shared = kSweep && (r == first_row || r == last_row);
  bool dead = false;
  double acc = 0.0;
  const float two_a = 2.0f * alpha;
  const float2 nab = make_float2(-alpha * beta, -alpha * beta);
  float4* uring = reinterpret_cast<float4*>(sbuf);
  // row of rating i of the two triple batches (i < 2L), for the ring
  auto row_at = [&](int i) {
    const int v = __shfl_sync(kFull, i < L ? rA : rB, ln.gbase + (i & (L - 1)));
    return v;
  };
  auto u_issue = [&](int t, int row, bool start) {  // U row of rating t -> slot t % UD
    if (t < len && start) {
      float4* slot = uring + (t % UD) * V4 * 256;
      const float* src = Ub + (int64_t)row * kp;
#pragma unroll
      for (int q = 0; q < V4; ++q)
        if (ln.on(q)) cp_async16(slot + q * 256, src + ln.off(q));
    }
    cp_async_commit();
  };
  if (kURing) {
#pragma unroll
    for (int d = 1; d <= UD; ++d) {
      const int rd = row_at(d), rp = row_at(d - 1);
      u_issue(d, rd, rd != rp);
    }
  }

  for (int t0 = 0; t0 < maxlen; t0 += L) {
#pragma unroll 1
    for (int j = 0; j < L; ++j) {
      const int t = t0 + j;
      // look ahead: triple of t+1 (from batch A, or B at the batch edge)
      const bool last_in_batch = (j + 1 == L);
      const int src = ln.gbase + ((j + 1) & (L - 1));
      const int rn = __shfl_sync(kFull, last_in_batch ? rB : rA, src);
      const int cn = __shfl_sync(kFull, last_in_batch ? cB : cA, src);
      const float xn = __shfl_sync(kFull, last_in_batch ? xB : xA, src);
      const bool valid = t < len && !dead;
      const bool nvalid = t + 1 < len && !dead;
      const bool newrun = nvalid && rn != r;
      float4 vn[V4], un[V4];
      if (nvalid) load_row<V4>(vn, Vb + (int64_t)cn * kp, ln);
      if (kURing) {
        cp_async_wait<UD - 1>();  // rating t+1's U row has landed (when it starts a run)
        if (newrun) {
          const float4* slot = uring + ((t + 1) % UD) * V4 * 256;
#pragma unroll
          for (int q = 0; q < V4; ++q) un[q] = ln.on(q) ? slot[q * 256] : zero4();
        }
        const int ri = row_at(j + 1 + UD), rp = row_at(j + UD);
        u_issue(t + 1 + UD, ri, ri != rp);
      } else if (newrun) {
        load_row<V4>(un, Ub + (int64_t)rn * kp, ln);
      }

      const float dot = group_sum<L>(dot_slice<V4>(u, v));
      const float e = x - dot;
      if (valid) {
        if (!kSweep) {
          const double ed = (double)x - (double)dot;
          acc += ed * ed;
        } else if (!isfinite(e)) {
          if (ln.gl == 0)
            atomicMin(bad, pack_bad(ch.pos, ch.iter >= 0 ? ch.iter : iter, ch.begin + t - ch.bbeg));
          dead = true;
        } else {
          const float g = two_a * e;
          const float2 g2 = make_float2(g, g);
          float* vp = Vb + (int64_t)c * kp;
          float* up = Ub + (int64_t)r * kp;
#pragma unroll
          for (int q = 0; q < V4; ++q) {
            const float2 ul = lo2(u[q]), uh = hi2(u[q]), vl = lo2(v[q]), vh = hi2(v[q]);
            // dv = 2ae*u_old - ab*v ; du = 2ae*v - ab*u_old
            const float2 dvl = __ffma2_rn(g2, ul, __fmul2_rn(nab, vl));
            const float2 dvh = __ffma2_rn(g2, uh, __fmul2_rn(nab, vh));
            const float2 dul = __ffma2_rn(g2, vl, __fmul2_rn(nab, ul));
            const float2 duh = __ffma2_rn(g2, vh, __fmul2_rn(nab, uh));
            u[q] = cat4(__fadd2_rn(ul, dul), __fadd2_rn(uh, duh));
            if (ln.on(q)) {
              if (kBulk)
                *reinterpret_cast<float4*>(sbuf + (nbulk % kBulkBufs) * kp + ln.off(q)) =
                    cat4(dvl, dvh);
              else
                red_add_v4(vp + ln.off(q), cat4(dvl, dvh));
              if (shared) red_add_v4(up + ln.off(q), cat4(dul, duh));
            }
          }
        }
      }
      if (kSweep && kBulk) {
        // the group's V delta is in its smem slot: one lane hands the whole
        // row to the TMA engine (bulk reduce-add at L2)
        const bool issue = valid && !dead;
        fence_async_smem();
        __syncwarp();
        if (issue && ln.gl == 0) {
          bulk_red_add(Vb + (int64_t)c * kp, sbuf + (nbulk % kBulkBufs) * kp, (unsigned)kp * 4u);
          bulk_commit();
        }
        if (issue) ++nbulk;
        // before the next write into the ring, its oldest slot must be read
        if (ln.gl == 0) bulk_wait_read<kBulkBufs - 1>();
        __syncwarp();
      }
      if (kSweep && valid && !dead && !shared && (newrun || !nvalid))
        store_row<V4>(Ub + (int64_t)r * kp, u, ln);
      if (newrun) {
#pragma unroll
        for (int q = 0; q < V4; ++q) u[q] = un[q];
        shared = kSweep && (rn == first_row || rn == last_row);
      }
      if (nvalid) {
#pragma unroll
        for (int q = 0; q < V4; ++q) v[q] = vn[q];
      }
      r = rn;
      c = cn;
      x = xn;
    }
    // a run split across chunks: every group red.adds its u deltas, so the
    // global row holds all of them; re-read it once per triple batch so a long
    // shared run (a heavy user) sees the other groups' updates, not only its
    // own (outside the per-rating loop: interior runs pay nothing)
    if (kSweep && shared && !dead && t0 + L < len) load_row<V4>(u, Ub + (int64_t)r * kp, ln);
    // advance the triple batches
    rA = rB; cA = cB; xA = xB;
    const int nb = t0 + 2 * L + ln.gl;
    if (nb < len) load_triple(lrow, lcol, val, cbits, ch.begin + nb, rB, cB, xB);
    if (upf) prefetch_runs<L>(Ub, rB, kp, nb < len);
  }
  if (kSweep && kBulk && ln.gl == 0) bulk_wait_all();
  if (kURing) cp_async_wait<0>();
  return acc;
}

template <int L, int V4, bool kMask, int MODE>
__global__ void __launch_bounds__(256, 2)
sgd_fast_kernel(const BlockWork* __restrict__ work, int nwork, int total_chunks,
                const int32_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                const float* __restrict__ val, float* __restrict__ U, float* __restrict__ V,
                int kp, float alpha, float beta, int iter, unsigned long long* __restrict__ bad,
                int cbits, int dyn_d, unsigned* __restrict__ dyn, int flags) {
  constexpr int GPW = 32 / L;
  extern __shared__ float4 smem_rows[];
  const int snap = flags & 0xFFFF;     // run-aligned chunk edges (0: off)
  const bool upf = (flags >> 16) & 1;  // U-row L2 prefetch
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  // bulk: this group's delta ring, kBulkBufs rows of kp floats; uring: this
  // thread's slice of the U-row ring ([slot][q][thread] float4)
  float* sbuf = MODE == 2 ? reinterpret_cast<float*>(smem_rows + threadIdx.x)
                          : reinterpret_cast<float*>(smem_rows) +
                                (size_t)((threadIdx.x >> 5) * GPW + lane / L) * kBulkBufs * kp;
  if (dyn_d <= 1) {
    int cidx = warp * GPW + lane / L;
    if ((flags >> 17) & 1) {
      // spread: fewer chunks than the grid's groups (a stratum whose per-block
      // concurrency floors bind), dealt evenly over the CTAs -- a full wave of
      // CTAs, so every SM holds the same number of working groups, instead of
      // the last SMs holding one CTA where the others hold two
      const int nb = (int)gridDim.x, b = (int)blockIdx.x;
      const int q = total_chunks / nb, rem = total_chunks % nb;
      const int lg = (int)(threadIdx.x >> 5) * GPW + lane / L;
      cidx = lg < q + (b < rem) ? b * q + min(b, rem) + lg : total_chunks;
    }
    Chunk ch = locate_chunk(work, nwork, total_chunks, cidx);
    if (snap > 0) {
      const int64_t b = snap_edge<L>(lrow, cbits, ch.begin, ch.bbeg, ch.bend, snap);
      const int64_t e = snap_edge<L>(lrow, cbits, ch.end, ch.bbeg, ch.bend, snap);
      ch.begin = b;
      ch.end = max(b, e);
    }
    const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)(ch.end - ch.begin));
    pdl_trigger();
    if (maxlen == 0) return;
    pdl_wait();
    walk_chunk<L, V4, kMask, true, MODE>(ch, maxlen, lrow, lcol, val, U, V, kp, alpha, beta,
                                         iter, bad, cbits, sbuf, upf);
    return;
  }
  // dynamic: slot = this warp, then nwarps + a ticket from dyn[0] until the
  // D phases are taken; the last warp out (dyn[1]) zeroes both counters for
  // the next launch (stream order / griddepcontrol.wait makes that visible)
  pdl_trigger();
  pdl_wait();
  const int nwarps = (int)(gridDim.x * (blockDim.x >> 5));
  const int slots = dyn_d * ((total_chunks + GPW - 1) / GPW);
  for (int slot = warp; slot < slots;) {
    Chunk ch = locate_dyn(work, nwork, total_chunks, dyn_d, slot, lane / L, GPW);
    if (snap > 0) {
      const int64_t b = snap_edge<L>(lrow, cbits, ch.begin, ch.bbeg, ch.bend, snap);
      const int64_t e = snap_edge<L>(lrow, cbits, ch.end, ch.bbeg, ch.bend, snap);
      ch.begin = b;
      ch.end = max(b, e);
    }
    const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)(ch.end - ch.begin));
    if (maxlen > 0)
      walk_chunk<L, V4, kMask, true, MODE>(ch, maxlen, lrow, lcol, val, U, V, kp, alpha, beta,
                                           iter, bad, cbits, sbuf, upf);
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(dyn, 1u);
    slot = nwarps + (int)__shfl_sync(kFull, t, 0);
  }
  if (lane == 0 && atomicAdd(dyn + 1, 1u) == (unsigned)nwarps - 1u) {
    dyn[0] = 0u;
    dyn[1] = 0u;
  }
}

// Post-sweep SSE of each block: sum over the chunk of (x - u.v)^2 in fp64,
// one atomicAdd per group into sse[block_id].
template <int L, int V4, bool kMask>
__global__ void __launch_bounds__(256, 2)
sse_fast_kernel(const BlockWork* __restrict__ work, int nwork, int total_chunks,
                const int32_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                const float* __restrict__ val, const float* __restrict__ U,
                const float* __restrict__ V, int kp, double* __restrict__ sse, int cbits) {
  constexpr int GPW = 32 / L;
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const Chunk ch = locate_chunk(work, nwork, total_chunks, warp * GPW + lane / L);
  const int len = (int)(ch.end - ch.begin);
  const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)len);
  if (maxlen == 0) return;
  const double acc = walk_chunk<L, V4, kMask, false>(ch, maxlen, lrow, lcol, val,
                                                     const_cast<float*>(U), const_cast<float*>(V),
                                                     kp, 0.f, 0.f, 0, nullptr, cbits);
  if ((lane & (L - 1)) == 0 && len > 0) atomicAdd(sse + ch.block_id, acc);
}

// Post-sweep SSE with the V rows streamed through a per-lane shared-memory
// ring by cp.async (LDGSTS): each lane copies its own 16-byte slices of the
// V row of rating t+D while rating t is computed, so D rows per group are in
// flight with no register cost (the pipelined register walk keeps one; the
// pass is latency-bound on those reads: profiles/r01_ncu_c4.md).  A lane only
// reads back what it copied itself, so cp.async.wait_group is the only
// synchronisation.  U stays in registers for a user's run (next run's row
// prefetched one rating ahead, as in walk_chunk).  Requires D <= L.

// The SSE walk of one chunk per group (all groups of the warp together:
// the trip count is the warp's longest chunk).  Returns the group's sum
// (valid in lane gl == 0).  `ring` = this thread's slice of the cp.async ring.
template <int L, int V4, bool kMask, int D>
__device__ __forceinline__ double sse_async_walk(const Chunk& ch, const int32_t* __restrict__ lrow,
                                                 const int32_t* __restrict__ lcol,
                                                 const float* __restrict__ val,
                                                 const float* __restrict__ U,
                                                 const float* __restrict__ V, int kp, int cbits,
                                                 float4* ring, bool upf = false) {
  static_assert(D <= L, "the look-ahead must fit the two triple batches");
  const int len = (int)(ch.end - ch.begin);
  const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)len);
  if (maxlen == 0) return 0.0;
  const Lanes<L, V4, kMask> ln(kp);
  const float* Ub = U + ch.row_start * kp;
  const float* Vb = V + ch.col_start * kp;
  auto issue = [&](int t, int c) {  // V row of rating t -> slot t % D
    if (t < len) {
      const float* row = Vb + (int64_t)c * kp;
      float4* slot = ring + (t % D) * V4 * 256;
#pragma unroll
      for (int q = 0; q < V4; ++q)
        if (ln.on(q)) cp_async16(slot + q * 256, row + ln.off(q));
    }
    cp_async_commit();
  };
  int rA = 0, cA = 0, rB = 0, cB = 0;
  float xA = 0.f, xB = 0.f;
  if (ln.gl < len) load_triple(lrow, lcol, val, cbits, ch.begin + ln.gl, rA, cA, xA);
  if (L + ln.gl < len) load_triple(lrow, lcol, val, cbits, ch.begin + L + ln.gl, rB, cB, xB);
  if (upf) prefetch_runs<L>(Ub, rB, kp, L + ln.gl < len);
#pragma unroll
  for (int d = 0; d < D; ++d) issue(d, __shfl_sync(kFull, cA, ln.gbase + d));
  int r = __shfl_sync(kFull, rA, ln.gbase);
  float4 u[V4], un[V4];
  if (len > 0) load_row_ro(u, Ub + (int64_t)r * kp, ln);
  else {
#pragma unroll
    for (int q = 0; q < V4; ++q) u[q] = zero4();
  }
  double acc = 0.0;
  if (L >= 4) {
    // two ratings per step: their dot products share one reduce-scatter
    // (level L/2 splits the pair between the half-groups, then the usual
    // butterfly), so the shuffle chain is amortised over both.  The pairs of
    // lanes added are the butterfly's, so every dot is bit-identical to it.
    constexpr int H = L / 2;
    const bool upper = (ln.gl & H) != 0;
    int rcur = len > 0 ? r : -1, rnxt = -1;
    for (int t0 = 0; t0 < maxlen; t0 += L) {
#pragma unroll 1
      for (int j = 0; j < L; j += 2) {
        const int t = t0 + j;
        const float x0 = __shfl_sync(kFull, xA, ln.gbase + j);
        const float x1 = __shfl_sync(kFull, xA, ln.gbase + j + 1);
        const int r0 = __shfl_sync(kFull, rA, ln.gbase + j);
        const int r1 = __shfl_sync(kFull, rA, ln.gbase + j + 1);
        const int r2 = __shfl_sync(kFull, j + 2 < L ? rA : rB, ln.gbase + ((j + 2) & (L - 1)));
        const int r3 = __shfl_sync(kFull, j + 3 < L ? rA : rB, ln.gbase + ((j + 3) & (L - 1)));
        cp_async_wait<D - 2>();  // ratings t, t+1 have landed
        float4 v0[V4], v1[V4];
        const float4* s0 = ring + (t % D) * V4 * 256;
        const float4* s1 = ring + ((t + 1) % D) * V4 * 256;
#pragma unroll
        for (int q = 0; q < V4; ++q) {
          v0[q] = ln.on(q) ? s0[q * 256] : zero4();
          v1[q] = ln.on(q) ? s1[q * 256] : zero4();
        }
        // U of rating t, then of t+1: the current run's row, the prefetched
        // next run's row, or (rarely: two runs starting in one pair) a load now
        if (t < len && r0 != rcur) {
          if (r0 == rnxt) {
#pragma unroll
            for (int q = 0; q < V4; ++q) u[q] = un[q];
          } else {
            load_row_ro(u, Ub + (int64_t)r0 * kp, ln);
          }
          rcur = r0;
          rnxt = -1;
        }
        const float p0 = dot_slice<V4>(u, v0);
        if (t + 1 < len && r1 != rcur) {
          if (r1 == rnxt) {
#pragma unroll
            for (int q = 0; q < V4; ++q) u[q] = un[q];
          } else {
            load_row_ro(u, Ub + (int64_t)r1 * kp, ln);
          }
          rcur = r1;
          rnxt = -1;
        }
        const float p1 = dot_slice<V4>(u, v1);
        // request the next run's U row as soon as its start is in view
        if (rnxt < 0) {
          const int cand = (t + 2 < len && r2 != rcur) ? r2 : ((t + 3 < len && r3 != rcur) ? r3 : -1);
          if (cand >= 0) {
            load_row_ro(un, Ub + (int64_t)cand * kp, ln);
            rnxt = cand;
          }
        }
        float a = upper ? p1 : p0;
        const float b = upper ? p0 : p1;
        a += __shfl_xor_sync(kFull, b, H);
#pragma unroll
        for (int o = H / 2; o > 0; o >>= 1) a += __shfl_xor_sync(kFull, a, o);
        const bool valid = upper ? (t + 1 < len) : (t < len);
        if (valid) {
          const double ed = (double)(upper ? x1 : x0) - (double)a;
          acc += ed * ed;
        }
        // refill both slots with ratings t + D, t + D + 1
        const int cd0 = __shfl_sync(kFull, j + D < L ? cA : cB, ln.gbase + ((j + D) & (L - 1)));
        const int cd1 =
            __shfl_sync(kFull, j + D + 1 < L ? cA : cB, ln.gbase + ((j + D + 1) & (L - 1)));
        issue(t + D, cd0);
        issue(t + D + 1, cd1);
      }
      rA = rB; cA = cB; xA = xB;
      const int nb = t0 + 2 * L + ln.gl;
      if (nb < len) load_triple(lrow, lcol, val, cbits, ch.begin + nb, rB, cB, xB);
      if (upf) prefetch_runs<L>(Ub, rB, kp, nb < len);
    }
    // only lanes gl == 0 (rating t) and gl == H (rating t+1) hold each sum once
    if (ln.gl != 0 && ln.gl != H) acc = 0.0;
    acc += __shfl_xor_sync(kFull, acc, H);
  } else {
  for (int t0 = 0; t0 < maxlen; t0 += L) {
#pragma unroll 1
    for (int j = 0; j < L; ++j) {
      const int t = t0 + j;
      const float x = __shfl_sync(kFull, xA, ln.gbase + j);
      const bool last_in_batch = (j + 1 == L);
      const int src = ln.gbase + ((j + 1) & (L - 1));
      const int rn = __shfl_sync(kFull, last_in_batch ? rB : rA, src);
      const bool newrun = t + 1 < len && rn != r;
      if (newrun) load_row_ro(un, Ub + (int64_t)rn * kp, ln);
      cp_async_wait<D - 1>();  // rating t's slot has landed
      float4 v[V4];
      const float4* slot = ring + (t % D) * V4 * 256;
#pragma unroll
      for (int q = 0; q < V4; ++q) v[q] = ln.on(q) ? slot[q * 256] : zero4();
      const float dot = group_sum<L>(dot_slice<V4>(u, v));
      if (t < len) {
        const double ed = (double)x - (double)dot;
        acc += ed * ed;
      }
      // refill this slot with rating t + D (from batch A, or B past its edge)
      const int srcd = ln.gbase + ((j + D) & (L - 1));
      const int cd = __shfl_sync(kFull, j + D < L ? cA : cB, srcd);
      issue(t + D, cd);
      if (newrun) {
#pragma unroll
        for (int q = 0; q < V4; ++q) u[q] = un[q];
      }
      r = rn;
    }
    rA = rB; cA = cB; xA = xB;
    const int nb = t0 + 2 * L + ln.gl;
    if (nb < len) load_triple(lrow, lcol, val, cbits, ch.begin + nb, rB, cB, xB);
    if (upf) prefetch_runs<L>(Ub, rB, kp, nb < len);
  }
  }
  cp_async_wait<0>();
  return acc;
}

template <int L, int V4, bool kMask, int D>
__global__ void __launch_bounds__(256, 2)
sse_async_kernel(const BlockWork* __restrict__ work, int nwork, int total_chunks,
                 const int32_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                 const float* __restrict__ val, const float* __restrict__ U,
                 const float* __restrict__ V, int kp, double* __restrict__ sse, int cbits,
                 int upf) {
  constexpr int GPW = 32 / L;
  // this lane's D slots of V4 float4, lane-interleaved ([slot][q][thread]) so a
  // warp's 16-byte accesses hit 32 consecutive bank quads
  extern __shared__ float4 ring_all[];
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const Chunk ch = locate_chunk(work, nwork, total_chunks, warp * GPW + lane / L);
  pdl_trigger();
  pdl_wait();
  const double acc = sse_async_walk<L, V4, kMask, D>(ch, lrow, lcol, val, U, V, kp, cbits,
                                                      ring_all + threadIdx.x, upf != 0);
  if ((lane & (L - 1)) == 0 && ch.end > ch.begin) atomicAdd(sse + ch.block_id, acc);
}

// Sweep and post-sweep SSE of a stratum in ONE launch.  Phase 1 is
// sgd_fast_kernel (one chunk per group, one wave); a group that finishes its
// chunk counts it into done[w] (after a fence: its V reductions and U stores
// are visible first).  Phase 2: warps take SSE slots (GPW consecutive SSE
// chunks of one block) of blocks whose sweep is complete (done[w] equals the
// block's sweep chunks), from per-block slot counters -- so the SSE of early
// blocks fills the tail of the sweep of late ones, with no second launch.
// The SSE is an order-free sum (atomicAdd per group), as in sse_async_kernel.
// done / next: 2 * nwork counters, zeroed before the launch.
template <int L, int V4, bool kMask, int D>
__global__ void __launch_bounds__(256, 2)
sweep_sse_kernel(const BlockWork* __restrict__ work, int nwork, int total_chunks,
                 const BlockWork* __restrict__ swork, const int32_t* __restrict__ lrow,
                 const int32_t* __restrict__ lcol, const float* __restrict__ val,
                 float* __restrict__ U, float* __restrict__ V, int kp, float alpha, float beta,
                 int iter, unsigned long long* __restrict__ bad, double* __restrict__ sse,
                 unsigned* __restrict__ done, int cbits) {
  constexpr int GPW = 32 / L;
  extern __shared__ float4 ring_all[];
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  {
    const Chunk ch = locate_chunk(work, nwork, total_chunks, warp * GPW + lane / L);
    const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)(ch.end - ch.begin));
    if (maxlen > 0)
      walk_chunk<L, V4, kMask, true>(ch, maxlen, lrow, lcol, val, U, V, kp, alpha, beta, iter,
                                     bad, cbits);
    if ((lane & (L - 1)) == 0 && ch.w >= 0) {
      __threadfence();
      atomicAdd(done + ch.w, 1u);
    }
  }
  unsigned* next = done + nwork;
  const int gl = lane & (L - 1), g = lane / L;
  unsigned long long t0 = 0;
  for (unsigned poll = 0;; ++poll) {
    // lane 0 picks a swept block with unclaimed SSE slots
    int pick = -1, slot = 0, left = 0;
    if (lane == 0) {
      for (int i = 0; i < nwork; ++i) {
        const int w = (warp + i) % nwork;
        const BlockWork bw = swork[w];
        const int nch = (int)((bw.end - bw.begin + bw.chunk_len - 1) / bw.chunk_len);
        const int slots = (nch + GPW - 1) / GPW;
        if ((int)*((volatile unsigned*)(next + w)) >= slots) continue;
        ++left;
        const BlockWork sw = work[w];
        const unsigned need = (unsigned)((sw.end - sw.begin + sw.chunk_len - 1) / sw.chunk_len);
        unsigned d;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(done + w) : "memory");
        if (d < need) continue;
        const int got = (int)atomicAdd(next + w, 1u);
        if (got < slots) { pick = w; slot = got; break; }
      }
    }
    pick = __shfl_sync(kFull, pick, 0);
    left = __shfl_sync(kFull, left, 0);
    if (pick < 0) {
      if (left == 0) break;  // every SSE slot is taken
      if ((poll & 1023u) == 1023u) {  // bounded: a lost counter must not hang the GPU
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (!t0) t0 = t; else if (t - t0 > 20000000000ull) __trap();
      }
      __nanosleep(128);
      continue;
    }
    slot = __shfl_sync(kFull, slot, 0);
    const BlockWork bw = swork[pick];
    Chunk ch{0, 0, 0, 0, bw.row_start, bw.col_start, bw.block_id, bw.pos, pick, -1};
    const int64_t c0 = (int64_t)(slot * GPW + g) * bw.chunk_len;
    ch.bbeg = bw.begin;
    ch.bend = bw.end;
    ch.begin = min(bw.begin + c0, bw.end);
    ch.end = min(ch.begin + (int64_t)bw.chunk_len, bw.end);
    const double acc = sse_async_walk<L, V4, kMask, D>(ch, lrow, lcol, val, U, V, kp, cbits,
                                                        ring_all + threadIdx.x);
    if (gl == 0 && ch.end > ch.begin) atomicAdd(sse + ch.block_id, acc);
  }
}

// Post-sweep SSE, wide form: no update dependency, so each group keeps D
// ratings' U and V rows in flight at once (D x the memory-level parallelism of
// the sweep walk).  Its own (L, V4) shape: 8 floats per lane.  U and V are
// read-only during this kernel, so both go through the L1 (__ldg): a user's
// run re-reads its U row from L1.  One fp64 atomicAdd per group per block.
template <int L, int V4, bool kMask, int D>
__global__ void __launch_bounds__(256, 2)
sse_wide_kernel(const BlockWork* __restrict__ work, int nwork, int total_chunks,
                const int32_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                const float* __restrict__ val, const float* __restrict__ U,
                const float* __restrict__ V, int kp, double* __restrict__ sse, int cbits) {
  constexpr int GPW = 32 / L;
  static_assert(L % D == 0, "D must divide L");
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const Chunk ch = locate_chunk(work, nwork, total_chunks, warp * GPW + lane / L);
  const int len = (int)(ch.end - ch.begin);
  const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)len);
  if (maxlen == 0) return;
  const Lanes<L, V4, kMask> ln(kp);
  const float* Ub = U + ch.row_start * kp;
  const float* Vb = V + ch.col_start * kp;
  double acc = 0.0;
  for (int t0 = 0; t0 < maxlen; t0 += L) {
    int r_l = 0, c_l = 0;
    float x_l = 0.f;
    if (t0 + ln.gl < len) load_triple(lrow, lcol, val, cbits, ch.begin + t0 + ln.gl, r_l, c_l, x_l);
#pragma unroll 1
    for (int j0 = 0; j0 < L; j0 += D) {
      float4 uu[D][V4], vv[D][V4];
      float x[D];
      bool ok[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int r = __shfl_sync(kFull, r_l, ln.gbase + j0 + d);
        const int c = __shfl_sync(kFull, c_l, ln.gbase + j0 + d);
        x[d] = __shfl_sync(kFull, x_l, ln.gbase + j0 + d);
        ok[d] = t0 + j0 + d < len;
#pragma unroll
        for (int q = 0; q < V4; ++q) {
          const bool on = ok[d] && ln.on(q);
          uu[d][q] = on ? __ldg(reinterpret_cast<const float4*>(Ub + (int64_t)r * kp + ln.off(q)))
                        : zero4();
          vv[d][q] = on ? __ldg(reinterpret_cast<const float4*>(Vb + (int64_t)c * kp + ln.off(q)))
                        : zero4();
        }
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const float dot = group_sum<L>(dot_slice<V4>(uu[d], vv[d]));
        if (ok[d]) {
          const double e = (double)x[d] - (double)dot;
          acc += e * e;
        }
      }
    }
  }
  if (ln.gl == 0 && len > 0) atomicAdd(sse + ch.block_id, acc);
}

// Out-of-line copies of the two walks for the persistent kernel: register
// allocation is then per phase, and the call costs once per chunk.
template <int L, int V4, bool kMask>
__device__ __noinline__ void sweep_chunk(const Chunk& ch, int maxlen,
                                         const int32_t* __restrict__ lrow,
                                         const int32_t* __restrict__ lcol,
                                         const float* __restrict__ val, float* U, float* V,
                                         int kp, float alpha, float beta, int iter,
                                         unsigned long long* bad) {
  walk_chunk<L, V4, kMask, true>(ch, maxlen, lrow, lcol, val, U, V, kp, alpha, beta, iter, bad);
}

template <int L, int V4, bool kMask>
__device__ __noinline__ double sse_chunk(const Chunk& ch, int maxlen,
                                         const int32_t* __restrict__ lrow,
                                         const int32_t* __restrict__ lcol,
                                         const float* __restrict__ val, float* U, float* V,
                                         int kp) {
  return walk_chunk<L, V4, kMask, false>(ch, maxlen, lrow, lcol, val, U, V, kp, 0.f, 0.f, 0,
                                         nullptr);
}

// Whole outer step in one cooperative launch: for every batch, `iters`
// sweeps, then the per-block SSE, separated by grid-wide barriers (a stratum
// must finish before its SSE, and the SSE before the next stratum touches the
// same U/V slices).  Groups loop over the batch's chunks (normally one each).
struct BatchDesc {
  int w0, nw, chunks, pad;
};

template <int L, int V4, bool kMask>
__global__ void __launch_bounds__(256, 2)
epoch_fast_kernel(const BlockWork* __restrict__ work, const BatchDesc* __restrict__ batches,
                  int nbatch, int iters, const int32_t* __restrict__ lrow,
                  const int32_t* __restrict__ lcol, const float* __restrict__ val,
                  float* __restrict__ U, float* __restrict__ V, int kp, float alpha, float beta,
                  double* __restrict__ sse, unsigned long long* __restrict__ bad) {
  constexpr int GPW = 32 / L;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int stride = (int)(gridDim.x * (blockDim.x >> 5)) * GPW;
  for (int t = 0; t < nbatch; ++t) {
    const BatchDesc bd = batches[t];
    const BlockWork* w = work + bd.w0;
    for (int it = 0; it < iters; ++it) {
      for (int base = warp * GPW; base < bd.chunks; base += stride) {
        const Chunk ch = locate_chunk(w, bd.nw, bd.chunks, base + lane / L);
        const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)(ch.end - ch.begin));
        if (maxlen > 0)
          sweep_chunk<L, V4, kMask>(ch, maxlen, lrow, lcol, val, U, V, kp, alpha, beta, it, bad);
      }
      grid.sync();
    }
    for (int base = warp * GPW; base < bd.chunks; base += stride) {
      const Chunk ch = locate_chunk(w, bd.nw, bd.chunks, base + lane / L);
      const int len = (int)(ch.end - ch.begin);
      const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)len);
      if (maxlen == 0) continue;
      const double acc = sse_chunk<L, V4, kMask>(ch, maxlen, lrow, lcol, val, U, V, kp);
      if ((lane & (L - 1)) == 0 && len > 0) atomicAdd(sse + ch.block_id, acc);
    }
    if (t + 1 < nbatch) grid.sync();
  }
}

// ---------------------------------------------------------------- exact
// Sequential fp64 sweep of one block in the reference's operation order.
// Returns the first non-finite entry index or -1 (_kernels.py:43-55).
__device__ int64_t sweep_exact(const int32_t* rows, const int32_t* cols, const double* vals,
                               int64_t count, double* u, double* v, int k, double alpha,
                               double beta) {
  for (int64_t i = 0; i < count; ++i) {
    double* ur = u + (int64_t)rows[i] * k;
    double* vc = v + (int64_t)cols[i] * k;
    double e = vals[i];
    for (int g = 0; g < k; ++g) e = __dsub_rn(e, __dmul_rn(ur[g], vc[g]));
    if (!isfinite(e)) return i;
    const double e2 = __dmul_rn(2.0, e);
    for (int g = 0; g < k; ++g) {
      const double ug = ur[g], vg = vc[g];
      ur[g] = __dadd_rn(ug, __dmul_rn(alpha, __dsub_rn(__dmul_rn(e2, vg), __dmul_rn(beta, ug))));
      vc[g] = __dadd_rn(vg, __dmul_rn(alpha, __dsub_rn(__dmul_rn(e2, ug), __dmul_rn(beta, vg))));
    }
  }
  return -1;
}

__device__ double sse_exact(const int32_t* rows, const int32_t* cols, const double* vals,
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

// mode 0: sweeps (sgd_sweeps), mode 1: converge (sgd_converge).
// out[8*w + 0..5] = sse_before, sse_after, iters_used, capped, bad_entry, bad_iter
__global__ void block_exact_kernel(const BlockWork* __restrict__ work, int nwork,
                                   const int32_t* __restrict__ lrow,
                                   const int32_t* __restrict__ lcol,
                                   const double* __restrict__ val, double* U, double* V, int k,
                                   double alpha, double beta, int mode, int iters, double tol,
                                   int64_t cap, int want_before, double* __restrict__ out) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nwork) return;
  const BlockWork bw = work[w];
  const int32_t* rows = lrow + bw.begin;
  const int32_t* cols = lcol + bw.begin;
  const double* vals = val + bw.begin;
  const int64_t count = bw.end - bw.begin;
  double* u = U + bw.row_start * k;
  double* v = V + bw.col_start * k;
  double* o = out + 8 * w;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  const bool before = want_before || mode == 1;
  const double sb = before ? sse_exact(rows, cols, vals, count, u, v, k) : 0.0;
  o[0] = sb; o[3] = 0.0; o[4] = -1.0; o[5] = -1.0;
  if (mode == 0) {
    for (int it = 0; it < iters; ++it) {
      const int64_t b = sweep_exact(rows, cols, vals, count, u, v, k, alpha, beta);
      if (b >= 0) { o[1] = nan; o[2] = iters; o[4] = (double)b; o[5] = it; return; }
    }
    const double sa = sse_exact(rows, cols, vals, count, u, v, k);
    o[2] = iters;
    if (!isfinite(sa)) { o[1] = nan; o[4] = (double)(count - 1); o[5] = iters - 1; return; }
    o[1] = sa;
    return;
  }
  // converge (_kernels.py:62-100)
  if (count == 0) { o[0] = 0.0; o[1] = 0.0; o[2] = 0.0; return; }
  double prev = sqrt(sb / (double)count);
  double s = sb;
  int64_t it = 0;
  while (it < cap) {
    const int64_t b = sweep_exact(rows, cols, vals, count, u, v, k, alpha, beta);
    if (b >= 0) { o[1] = nan; o[2] = (double)(it + 1); o[4] = (double)b; o[5] = (double)it; return; }
    ++it;
    s = sse_exact(rows, cols, vals, count, u, v, k);
    if (!isfinite(s)) {
      o[1] = nan; o[2] = (double)it; o[4] = (double)(count - 1); o[5] = (double)(it - 1);
      return;
    }
    const double now = sqrt(s / (double)count);
    if (prev - now < tol) { o[1] = s; o[2] = (double)it; return; }
    prev = now;
  }
  o[1] = s; o[2] = (double)it; o[3] = 1.0;
}

// <<<>>> with the programmatic-dependent-launch attribute when pdl is set
template <typename... KArgs, typename... Args>
void launch_k(bool pdl, void (*k)(KArgs...), dim3 grid, int block, size_t smem, cudaStream_t s,
              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// ------------------------------------------------------------ dispatch

// SSE pass shape: 8 floats per lane (V4 = 2) unless the row is wider than
// 32 lanes of that; D = ratings in flight per group.
Shape sse_shape_for(int kp) {
  const int f4 = kp / 4;
  int v4 = 2;
  while (v4 * 32 < f4) v4 <<= 1;
  if (f4 < v4) v4 = f4 < 1 ? 1 : (f4 >= 2 ? 2 : 1);
  int L = 1;
  while (L * v4 < f4) L <<= 1;
  return {L, v4};
}

#define BGMF_SSE_SHAPES(X)                                                              \
  X(1, 1, 1) X(1, 2, 1) X(2, 2, 2) X(4, 2, 4) X(8, 2, 4) X(16, 2, 4) X(32, 2, 4)        \
  X(32, 4, 4)

void launch_sse_wide(cudaStream_t s, const BlockWork* w, int nwork, int total,
                     const int32_t* lrow, const int32_t* lcol, const float* val, bgmf_ctx* c,
                     int cbits) {
  const Shape sh = sse_shape_for(c->kp);
  const bool mk = 4 * sh.L * sh.V4 != c->kp;
  const int gpw = 32 / sh.L;
  const int warps = (total + gpw - 1) / gpw;
  const dim3 grid((warps + 7) / 8);
#define BGMF_SSE(LL, VV, DD)                                                                  \
  if (sh.L == LL && sh.V4 == VV) {                                                            \
    if (mk)                                                                                   \
      sse_wide_kernel<LL, VV, true, DD><<<grid, 256, 0, s>>>(w, nwork, total, lrow, lcol, val, \
                                                             c->d_u, c->d_v, c->kp, c->d_sse, \
                                                             cbits);                          \
    else                                                                                      \
      sse_wide_kernel<LL, VV, false, DD><<<grid, 256, 0, s>>>(w, nwork, total, lrow, lcol,    \
                                                              val, c->d_u, c->d_v, c->kp,     \
                                                              c->d_sse, cbits);               \
    return;                                                                                   \
  }
  BGMF_SSE_SHAPES(BGMF_SSE)
#undef BGMF_SSE
}

bool upf_route(bgmf_ctx* c);

template <int LL, int VV, bool MM>
void launch_sse_async(dim3 grid, cudaStream_t s, const BlockWork* w, int nwork, int total,
                      const int32_t* lrow, const int32_t* lcol, const float* val, bgmf_ctx* c,
                      int cbits) {
  constexpr int D = LL < 4 ? LL : 4;
  const int smem = 256 * D * VV * 16;
  static std::atomic<uint64_t> attr_set{0};  // one bit per device: attributes are per context
  const uint64_t bit = 1ull << (c->device & 63);
  if (!(attr_set.load() & bit)) {
    cudaFuncSetAttribute(&sse_async_kernel<LL, VV, MM, D>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set.fetch_or(bit);
  }
  launch_k(c->pdl, &sse_async_kernel<LL, VV, MM, D>, grid, 256, smem, s, w, nwork, total, lrow,
           lcol, val, (const float*)c->d_u, (const float*)c->d_v, c->kp, c->d_sse, cbits,
           upf_route(c) ? 1 : 0);
}

// dynamic smem of the bulk sweep: kBulkBufs delta rows per group
size_t bulk_smem(bgmf_ctx* c, const Shape& sh) {
  return (size_t)(256 / sh.L) * kBulkBufs * c->kp * sizeof(float);
}

// u_prefetch routing: the L2 prefetch of the next runs' U rows pays only when
// nearly every rating starts a user run (C5 shape with 600 M ratings, 0.94
// ratings per (row, block): sweep 0.268 -> 0.248 ms, +11%) and costs issue
// slots and L2 bandwidth otherwise (C5 2 B, 3.1: 0.416 -> 0.437 ms; C4, 13:
// -3%; C3, 18: -5%).  Mean run length = ratings / rows of the non-empty
// blocks (a ring rank's partition holds only its row blocks).
constexpr double kUpfMaxRun = 1.5;

int64_t sweep_groups(bgmf_ctx* c, const Shape& sh);

// u_ring routing: the cp.async ring of upcoming runs' U rows measured +6% on
// the Zipf-skewed C4Z and -11% on uniform C4, -15% on C5 (DESIGN 3.10c); the
// partition's ratings-per-user CV separates them (uniform ~0.1, C4Z >> 1).
// Device-resident partitions only (the out-of-core one computes no CV).
constexpr double kURingMinCV = 1.0;

bool uring_route(bgmf_ctx* c) {
  return c->u_ring > 0 || (c->u_ring < 0 && !c->streaming && c->row_cv > kURingMinCV);
}

bool upf_route(bgmf_ctx* c) {
  const int64_t key = c->nnz * 8191 + (int64_t)c->I * c->J;
  if (c->upf_key != key) {
    double rows = 0.0;
    for (int b = 0; b < c->I * c->J && b + 1 < (int)c->h_offsets.size(); ++b)
      if (c->h_offsets[b + 1] > c->h_offsets[b])
        rows += (double)(c->row_bounds[b / c->J + 1] - c->row_bounds[b / c->J]);
    const double run = rows > 0.0 ? (double)c->nnz / rows : 0.0;
    c->upf_on = c->u_prefetch > 0 || (c->u_prefetch < 0 && rows > 0.0 && run < kUpfMaxRun);
    c->upf_key = key;
  }
  return c->upf_on;
}

void launch_fast_ptr(bool sweep, const Shape& sh, dim3 grid, cudaStream_t s, const BlockWork* w,
                     int nwork, int total, const int32_t* lrow, const int32_t* lcol,
                     const float* val, bgmf_ctx* c, float a, float b, int it, int cbits = -1) {
  const bool mk = needs_mask(sh, c->kp);
  const int dd = sweep && c->d_dyn ? c->dyn_split : 1;
  int sn = c->snap_cap | (upf_route(c) ? 1 << 16 : 0);
  const bool uring = sweep && uring_route(c);
  if (sweep && c->spread && dd <= 1 && !c->bulk_red && !uring) {
    // a partial wave that would leave some SMs with fewer CTAs than others:
    // launch the full wave and deal the chunks evenly (sgd_fast_kernel)
    const int64_t cap = sweep_groups(c, sh) / (8 * (32 / sh.L));
    if ((int64_t)grid.x > c->num_sms && (int64_t)grid.x * 20 < cap * 19) {
      grid.x = (unsigned)cap;
      sn |= 1 << 17;
    }
  }
#define BGMF_CASE(LL, VV, MM)                                                                 \
  if (sh.L == LL && sh.V4 == VV && mk == MM) {                                                \
    if (sweep && c->bulk_red) {                                                               \
      cudaFuncSetAttribute(&sgd_fast_kernel<LL, VV, MM, 1>,                                  \
                           cudaFuncAttributeMaxDynamicSharedMemorySize,                       \
                           (int)bulk_smem(c, sh));                                            \
      sgd_fast_kernel<LL, VV, MM, 1><<<grid, 256, bulk_smem(c, sh), s>>>(                     \
          w, nwork, total, lrow, lcol, val, c->d_u, c->d_v, c->kp, a, b, it, c->d_bad, cbits, dd,    \
          c->d_dyn, sn);                                                                          \
    } else if (uring && LL >= 4) {                                                            \
      constexpr int UD = LL >= 8 ? 4 : 3;                                                     \
      const int sm = 256 * UD * VV * 16;                                                      \
      cudaFuncSetAttribute(&sgd_fast_kernel<LL, VV, MM, 2>,                                  \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                  \
      sgd_fast_kernel<LL, VV, MM, 2><<<grid, 256, sm, s>>>(                                   \
          w, nwork, total, lrow, lcol, val, c->d_u, c->d_v, c->kp, a, b, it, c->d_bad, cbits, dd,    \
          c->d_dyn, sn);                                                                          \
    } else if (sweep)                                                                         \
      launch_k(c->pdl, &sgd_fast_kernel<LL, VV, MM, 0>, grid, 256, 0, s, w, nwork, total, lrow,   \
               lcol, val, c->d_u, c->d_v, c->kp, a, b, it, c->d_bad, cbits, dd, c->d_dyn, sn); \
    else if (c->sse_wide)                                                                     \
      launch_sse_wide(s, w, nwork, total, lrow, lcol, val, c, cbits);                          \
    else if (c->sse_async > 0)                                                                \
      launch_sse_async<LL, VV, MM>(grid, s, w, nwork, total, lrow, lcol, val, c, cbits);      \
    else                                                                                      \
      sse_fast_kernel<LL, VV, MM><<<grid, 256, 0, s>>>(w, nwork, total, lrow, lcol, val,      \
                                                       c->d_u, c->d_v, c->kp, c->d_sse, cbits);      \
    return;                                                                                   \
  }
  BGMF_SHAPES(BGMF_CASE)
#undef BGMF_CASE
}

void launch_fast(bool sweep, const Shape& sh, dim3 grid, cudaStream_t s, const BlockWork* w,
                 int nwork, int total, bgmf_ctx* c, float a, float b, int it) {
  launch_fast_ptr(sweep, sh, grid, s, w, nwork, total, c->d_lrow, c->d_lcol, c->d_val, c, a, b,
                  it);
}

// One stratum's last sweep + its SSE as ONE launch (sweep_sse_kernel), on the
// sweep's grid; its completion counters (2 per work item) are zeroed first.
// Returns false when the shape has no fused instance (the caller launches the
// two kernels).
bool launch_sweep_sse(const Shape& sh, dim3 grid, cudaStream_t s, const BlockWork* w,
                      const BlockWork* sw, int nwork, int total, bgmf_ctx* c, float a, float b,
                      int it) {
  const bool mk = needs_mask(sh, c->kp);
  if (cudaMemsetAsync(c->d_fuse, 0, sizeof(unsigned) * 2 * nwork, s) != cudaSuccess) return false;
#define BGMF_FUSED(LL, VV, MM)                                                                \
  if (sh.L == LL && sh.V4 == VV && mk == MM) {                                                \
    constexpr int D = LL < 4 ? LL : 4;                                                        \
    const int smem = 256 * D * VV * 16;                                                       \
    cudaFuncSetAttribute(&sweep_sse_kernel<LL, VV, MM, D>,                                    \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                   \
    sweep_sse_kernel<LL, VV, MM, D><<<grid, 256, smem, s>>>(                                  \
        w, nwork, total, sw, c->d_lrow, c->d_lcol, c->d_val, c->d_u, c->d_v, c->kp, a, b, it,  \
        c->d_bad, c->d_sse, c->d_fuse, -1);                                                   \
    return true;                                                                              \
  }
  BGMF_SHAPES(BGMF_FUSED)
#undef BGMF_FUSED
  return false;
}

const void* epoch_kernel_ptr(const Shape& sh, int kp) {
  const bool mk = needs_mask(sh, kp);
#define BGMF_EP(LL, VV, MM)                            \
  if (sh.L == LL && sh.V4 == VV && mk == MM)           \
    return reinterpret_cast<const void*>(&epoch_fast_kernel<LL, VV, MM>);
  BGMF_SHAPES(BGMF_EP)
#undef BGMF_EP
  return nullptr;
}

const void* sweep_kernel_ptr(const Shape& sh, int kp, bool bulk) {
  const bool mk = needs_mask(sh, kp);
#define BGMF_SW(LL, VV, MM)                                                             \
  if (sh.L == LL && sh.V4 == VV && mk == MM)                                            \
    return bulk ? reinterpret_cast<const void*>(&sgd_fast_kernel<LL, VV, MM, 1>)        \
                : reinterpret_cast<const void*>(&sgd_fast_kernel<LL, VV, MM, 0>);
  BGMF_SHAPES(BGMF_SW)
#undef BGMF_SW
  return nullptr;
}

// Resident 256-thread CTAs per SM of a kernel (the one-wave capacity).
int resident_ctas(bgmf_ctx* c, const void* fn, size_t smem = 0) {
  if (c->warps_per_sm > 0) return (c->warps_per_sm + 7) / 8;
  if (smem > 0) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int blocks = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, 256, smem);
  return blocks > 0 ? blocks : 1;
}

// Fill h_work for every batch; returns per-batch (work offset, total chunks).
struct BatchRange {
  int w0, nw, chunks;
};

// L2-resident waves.  A stratum's blocks are independent, so running it as
// several sequential sub-batches is the same algorithm.  The sweep's V traffic
// is L2 traffic only while the V blocks being swept at once fit in L2 (C4:
// 16 x 570 KB); when a stratum's V set is larger (C5: 64 x 8 MB = 512 MB) every
// V row read and reduce-add goes to HBM.  Cut each batch into waves whose
// V blocks total <= l2_wave_bytes (each wave re-chunked to fill the GPU).
// Returns the refined batch offsets over the same plan array.
std::vector<int32_t> l2_waves(const bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off,
                              int nbatch) {
  std::vector<int32_t> off;
  off.push_back(batch_off[0]);
  for (int t = 0; t < nbatch; ++t) {
    double bytes = 0;
    for (int q = batch_off[t]; q < batch_off[t + 1]; ++q) {
      const int bj = plan[q] % c->J;
      const double vb = (double)(c->col_bounds[bj + 1] - c->col_bounds[bj]) * c->kp * 4.0;
      if (c->l2_wave_bytes > 0 && bytes > 0 && bytes + vb > (double)c->l2_wave_bytes) {
        off.push_back(q);
        bytes = 0;
      }
      bytes += vb;
    }
    off.push_back(batch_off[t + 1]);
  }
  return off;
}

// Per-block chunk length of the fast paths.  cl = the batch's one-wave
// length (ceil(batch nnz / free groups)); the floor bounds how many groups
// sweep one block at once (lossless Hogwild: a V-row read is stale by the
// other groups' in-flight updates to that row).  Measured on B200 (fast-mode
// drift vs the reference order, tests/ + DESIGN.md §3.1):
//   * sparse blocks (density <= 1/8): at most cols * max(col_ratio,
//     (ratings per column - 32) / 80) groups, floor sparse_min_chunk.  The
//     first term keeps ~one concurrent update per two V rows on blocks with
//     few ratings per column (C1 1x1, 59 per column: 1.9 concurrent updates
//     per row drifted 1.3e-3 in 5 epochs); the second lets blocks with
//     hundreds of ratings per column use the whole GPU when a launch holds few
//     of them (C4, 351 per column, with 2 blocks per launch as each rank of the
//     8-GPU ring runs: ~4 concurrent updates per row, drift 2e-5);
//   * dense blocks: the conservative min_chunk floor (dense rows share their
//     column order, so concurrent groups collide far more often).
// Then stagger_chunk.
int64_t block_chunk(bgmf_ctx* c, int b, int64_t cnt, int64_t cl) {
  const int bi = b / c->J, bj = b % c->J;
  const int64_t rows = c->row_bounds[bi + 1] - c->row_bounds[bi];
  const int64_t cols = c->col_bounds[bj + 1] - c->col_bounds[bj];
  int64_t floor_len = c->min_chunk;
  if (c->sparse_min_chunk > 0 && cnt * 8 <= rows * cols) {
    // max concurrent groups: col_ratio per column, more when the block has many
    // ratings per column (each stale V read is then a smaller perturbation)
    const double per_col = (double)cnt / (double)(cols > 0 ? cols : 1);
    double ratio = (per_col - 32.0) / 80.0;
    if (ratio < c->col_ratio) ratio = c->col_ratio;
    const double cap = ratio * (double)cols;
    floor_len = (int64_t)std::ceil((double)cnt / (cap > 1.0 ? cap : 1.0));
    if (floor_len < c->sparse_min_chunk) floor_len = c->sparse_min_chunk;
  }
  int64_t bl = cl > floor_len ? cl : floor_len;
  bl = stagger_chunk(bl, c->stagger);
  return bl < cnt ? bl : cnt;
}

// Chunking: each batch's ratings are cut into equal chunks, at most `groups`
// of them (groups = worker groups resident in one wave; 0 = one chunk per
// block, the exact path).  chunk = ceil(batch_nnz / (groups - B)) so the
// per-block rounding can never spill into a second wave.
// sse = true: chunks for the post-sweep SSE, an order-free sum -- one-wave
// length only, none of block_chunk's concurrency floors (on small strata the
// sweep's floors leave most of the GPU idle; C1's sweep chunks are ~25
// ratings long, the SSE's ~3).
constexpr int64_t kSseMinChunk = 8;

int build_work(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off, int nbatch,
               int64_t groups, std::vector<BatchRange>& ranges,
               const std::vector<char>* active = nullptr, int w_base = 0, int pos_base = 0,
               bool sse = false) {
  const int total = batch_off[nbatch];
  if (!c->in_step) drain_async_steps(c);  // synchronous callers rewrite the table from 0
  int rc = ensure_step_scratch(c, (size_t)(w_base + total));
  if (rc) return rc;
  ranges.assign(nbatch, BatchRange{0, 0, 0});
  int w = w_base;
  for (int t = 0; t < nbatch; ++t) {
    int64_t batch_nnz = 0;
    int nonempty = 0;
    for (int q = batch_off[t]; q < batch_off[t + 1]; ++q) {
      const int b = plan[q];
      if (b < 0 || b >= c->I * c->J) return fail(c, BGMF_ERR_ARG, "plan block id out of range");
      if (active && !(*active)[q]) continue;
      const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
      batch_nnz += cnt;
      nonempty += cnt > 0;
    }
    int64_t cl = INT32_MAX;
    if (groups > 0) {
      const int64_t slots = groups - nonempty > 0 ? groups - nonempty : 1;
      cl = (batch_nnz + slots - 1) / slots;
    }
    ranges[t].w0 = w;
    int chunks = 0;
    // a batch the ordered kernel cannot take although the chunked sweep would
    // distort the reference order: one chunk (one group, stored order) per block
    const bool seq = groups > 0 && !sse && !active && c->ord_mode != 0 &&
                     order_risky(c, plan, batch_off[t], batch_off[t + 1]) &&
                     !use_ordered(c, plan, batch_off[t], batch_off[t + 1]);
    for (int q = batch_off[t]; q < batch_off[t + 1]; ++q) {
      const int b = plan[q];
      if (active && !(*active)[q]) continue;
      const int64_t beg = c->h_offsets[b], end = c->h_offsets[b + 1];
      const int64_t cnt = end - beg;
      if (cnt == 0) continue;
      int64_t bl = cnt;
      if (groups > 0 && !sse && !seq) bl = block_chunk(c, b, cnt, cl);
      else if (groups > 0) bl = std::min(cnt, std::max(cl, kSseMinChunk));
      BlockWork& bw = c->h_work[w++];
      bw.begin = beg;
      bw.end = end;
      bw.row_start = c->row_bounds[b / c->J];
      bw.col_start = c->col_bounds[b % c->J];
      bw.chunk_len = (int32_t)bl;
      bw.first_chunk = chunks;
      bw.block_id = b;
      bw.pos = pos_base + q;
      bw.active = nullptr;
      bw.iter = nullptr;
      chunks += (int)((cnt + bl - 1) / bl);
    }
    ranges[t].nw = w - ranges[t].w0;
    ranges[t].chunks = chunks;
  }
  return BGMF_OK;
}

// One-wave capacity of the sweep kernel in worker groups (cached: the
// occupancy query and the smem attribute are host calls that must stay out of
// the per-piece path so the copy stream can run ahead).
int64_t sweep_groups(bgmf_ctx* c, const Shape& sh) {
  const int key = (c->warps_per_sm * 4096 + c->kp) * 2 + (c->bulk_red ? 1 : 0);
  if (c->groups_key != key) {
    const size_t smem = c->bulk_red ? bulk_smem(c, sh) : 0;
    const int ctas = resident_ctas(c, sweep_kernel_ptr(sh, c->kp, c->bulk_red), smem);
    c->groups_cache = (int64_t)c->num_sms * ctas * 8 * (32 / sh.L);
    c->groups_key = key;
  }
  return c->groups_cache;
}

// CPMF merge (baselines.py:170-175): v = v_start + sum_w (v_w - v_start),
// the delta accumulated over shards in shard order from zero, per element.
template <typename T>
__global__ void merge_private_v(T* __restrict__ V, const T* __restrict__ priv, int64_t elems,
                                int nshards) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < elems;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T s = V[i];
    T delta = 0;
    for (int w = 0; w < nshards; ++w) delta = delta + (priv[(int64_t)w * elems + i] - s);
    V[i] = s + delta;
  }
}

template <typename T>
__global__ void broadcast_v(const T* __restrict__ V, T* __restrict__ priv, int64_t elems,
                            int nshards) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < elems * nshards;
       i += (int64_t)gridDim.x * blockDim.x)
    priv[i] = V[i % elems];
}

}  // namespace

int ensure_step_scratch(bgmf_ctx* c, size_t nwork) {
  const int nb = c->I * c->J;
  if (!c->d_fuse) BGMF_CK(c, dmalloc(&c->d_fuse, sizeof(unsigned) * 2 * (nb > 64 ? nb : 64), c->stream));
  if (!c->d_sse) {
    BGMF_CK(c, dmalloc(&c->d_sse, sizeof(double) * (nb > 0 ? nb : 1), c->stream));
    BGMF_CK(c, pinned_alloc((void**)&c->h_sse, sizeof(double) * (nb > 0 ? nb : 1)));
    BGMF_CK(c, dmalloc(&c->d_bad, 8, c->stream));
    BGMF_CK(c, pinned_alloc((void**)&c->h_bad, 8));
  }
  if (nwork > c->work_cap) {
    if (c->d_work) dfree(c->d_work, c->stream);
    pinned_free(c->h_work);
    c->d_work = nullptr;
    c->h_work = nullptr;
    size_t cap = nwork < 64 ? 64 : nwork;
    // device: work table, then exact-mode output slots / batch descriptors
    BGMF_CK(c, dmalloc(&c->d_work, sizeof(BlockWork) * cap * 8, c->stream));
    BGMF_CK(c, pinned_alloc((void**)&c->h_work, sizeof(BlockWork) * cap));
    c->work_cap = cap;
  }
  return BGMF_OK;
}

// One outer step, fast path.  Default: per stratum (wave), `iters` sweep
// launches + one SSE launch, all enqueued without a host sync; one D2H of the
// per-block SSEs at the end.  fused=1: ONE cooperative launch of
// epoch_fast_kernel for the whole step (grid barriers between strata;
// measured slower on B200 at every config, kept as an option).
int run_step_fast(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off_in, int nbatch_in,
                  int iters, float alpha, float beta) {
  cudaStream_t s = c->stream;
  const std::vector<int32_t> waves = l2_waves(c, plan, batch_off_in, nbatch_in);
  const bool split = (int)waves.size() - 1 != nbatch_in && c->fused <= 0;
  const int32_t* batch_off = split ? waves.data() : batch_off_in;
  const int nbatch = split ? (int)waves.size() - 1 : nbatch_in;
  const Shape sh = shape_for(c->kp);
  const int gpw = 32 / sh.L;
  const int nb = c->I * c->J;
  const void* ep = epoch_kernel_ptr(sh, c->kp);
  // fused = -1 (auto): the persistent kernel pays off when launches dominate
  // (small strata); big strata run faster as separate sweep / SSE launches.
  const int64_t per_batch = nbatch > 0 ? c->nnz / nbatch : c->nnz;
  const bool fused = c->fused > 0 || (c->fused < 0 && per_batch <= c->fused_max_batch);
  const int ctas_per_sm = fused ? resident_ctas(c, ep) : 0;
  const int64_t groups =
      fused ? (int64_t)c->num_sms * ctas_per_sm * 8 * gpw : sweep_groups(c, sh);
  std::vector<BatchRange> ranges, sranges;
  int rc = ensure_step_scratch(c, 2 * (size_t)batch_off[nbatch]);  // sweep + SSE tables
  if (rc) return rc;
  rc = build_work(c, plan, batch_off, nbatch, groups, ranges);
  if (rc) return rc;
  const int nw = ranges.empty() ? 0 : ranges.back().w0 + ranges.back().nw;
  if (!fused) {
    rc = build_work(c, plan, batch_off, nbatch, groups, sranges, nullptr, nw, 0, true);
    if (rc) return rc;
  }
  const int nw_all = sranges.empty() ? nw : sranges.back().w0 + sranges.back().nw;
  BatchDesc* bdesc = reinterpret_cast<BatchDesc*>(c->d_work + c->work_cap);
  std::vector<BatchDesc> hb(nbatch > 0 ? nbatch : 1);
  int max_chunks = 0;
  double ratings = 0;
  for (int t = 0; t < nbatch; ++t) {
    hb[t] = BatchDesc{ranges[t].w0, ranges[t].nw, ranges[t].chunks, 0};
    if (ranges[t].chunks > max_chunks) max_chunks = ranges[t].chunks;
  }
  for (int q = 0; q < nw; ++q) ratings += (double)(c->h_work[q].end - c->h_work[q].begin);
  if (nw_all > 0)
    BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * nw_all,
                               cudaMemcpyHostToDevice, s));
  BGMF_CK(c, cudaMemsetAsync(c->d_sse, 0, sizeof(double) * nb, s));
  BGMF_CK(c, cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  if (fused && max_chunks > 0) {
    BGMF_CK(c, cudaMemcpyAsync(bdesc, hb.data(), sizeof(BatchDesc) * nbatch,
                               cudaMemcpyHostToDevice, s));
    const int need = (max_chunks + gpw * 8 - 1) / (gpw * 8);
    const int cap = c->num_sms * ctas_per_sm;
    const dim3 grid(need < cap ? need : cap);
    const BlockWork* dw = c->d_work;
    const BatchDesc* db = bdesc;
    int nbt = nbatch, its = iters, kp = c->kp;
    const int32_t* lr = c->d_lrow;
    const int32_t* lc = c->d_lcol;
    const float* vv = c->d_val;
    float* U = c->d_u;
    float* V = c->d_v;
    double* sse = c->d_sse;
    unsigned long long* bad = c->d_bad;
    void* args[] = {&dw, &db, &nbt, &its, &lr, &lc, &vv, &U, &V, &kp, &alpha, &beta, &sse, &bad};
    TimedLaunch* slot = nullptr;
    if (c->timing) record_begin(c, 0, ratings * iters * (12.0 + 16.0 * c->k), &slot);
    BGMF_CK(c, cudaLaunchCooperativeKernel(ep, grid, dim3(256), args, 0, s));
    if (slot) record_end(c, slot);
  } else {
    for (int t = 0; t < nbatch; ++t) {
      const BatchRange& r = ranges[t];
      if (r.chunks == 0) continue;
      if (use_ordered(c, plan, batch_off[t], batch_off[t + 1])) {
        rc = run_batch_ordered(c, plan, batch_off[t], batch_off[t + 1], 0, iters, alpha, beta);
        if (rc) return rc;
        continue;
      }
      const int warps = (r.chunks + gpw - 1) / gpw;
      const dim3 grid((warps + 7) / 8);
      const BlockWork* w = c->d_work + r.w0;
      double br = 0;
      for (int q = 0; q < r.nw; ++q)
        br += (double)(c->h_work[r.w0 + q].end - c->h_work[r.w0 + q].begin);
      const BatchRange& sr = sranges[t];
      const bool fuse = c->fuse_sse && sr.nw == r.nw && c->sse_async > 0 && !c->sse_wide &&
                        !c->bulk_red;
      bool fused_done = false;
      for (int it = 0; it < iters; ++it) {
        TimedLaunch* slot = nullptr;
        if (c->timing) record_begin(c, 0, br * (12.0 + 16.0 * c->k), &slot);
        if (fuse && it == iters - 1)  // the last sweep and the SSE: one launch
          fused_done = launch_sweep_sse(sh, grid, s, w, c->d_work + sr.w0, r.nw, r.chunks, c,
                                        alpha, beta, it);
        if (!fused_done) launch_fast(true, sh, grid, s, w, r.nw, r.chunks, c, alpha, beta, it);
        if (slot) record_end(c, slot);
      }
      if (fused_done) continue;
      const dim3 sgrid(((sr.chunks + gpw - 1) / gpw + 7) / 8);
      TimedLaunch* slot = nullptr;
      if (c->timing) record_begin(c, 1, 0.0, &slot);
      launch_fast(false, sh, sgrid, s, c->d_work + sr.w0, sr.nw, sr.chunks, c, alpha, beta, 0);
      if (slot) record_end(c, slot);
    }
  }
  BGMF_CK(c, cudaGetLastError());
  BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb, cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaStreamSynchronize(s));
  if (c->timing) harvest_timing(c);
  return BGMF_OK;
}

int64_t fast_groups(bgmf_ctx* c) { return sweep_groups(c, shape_for(c->kp)); }

// Would the chunked sweep of batch plan[q0 .. q1) distort the reference
// order beyond what the randomised sweeps showed to be safe?  From the chunk
// length the sweep would use (build_work / block_chunk), per block: fewer
// than `factor` mean rows per chunk (groups sweep pieces of the same rows at
// once, each with a stale copy of u_r merged by red.add), or more than
// `max_col_conc` concurrent groups per V row.  Every fast-mode drift past
// 1e-3 the sweeps found was in one of the two.
bool chunked_splits_rows(bgmf_ctx* c, const int32_t* plan, int q0, int q1, double factor,
                         double max_col_conc) {
  const int64_t groups = sweep_groups(c, shape_for(c->kp));
  int64_t batch_nnz = 0;
  int nonempty = 0;
  for (int q = q0; q < q1; ++q) {
    const int64_t cnt = c->h_offsets[plan[q] + 1] - c->h_offsets[plan[q]];
    batch_nnz += cnt;
    nonempty += cnt > 0;
  }
  const int64_t slots = groups - nonempty > 0 ? groups - nonempty : 1;
  const int64_t cl = (batch_nnz + slots - 1) / slots;
  for (int q = q0; q < q1; ++q) {
    const int b = plan[q];
    const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
    if (cnt == 0) continue;
    const int64_t bl = block_chunk(c, b, cnt, cl);
    if (bl >= cnt) continue;  // one chunk: the block is swept sequentially
    const int64_t h = c->row_bounds[b / c->J + 1] - c->row_bounds[b / c->J];
    if ((double)bl < factor * (double)cnt / (double)(h > 0 ? h : 1)) return true;
    // concurrent groups per V row of the block (block_chunk lets blocks with
    // hundreds of ratings per column run several; max_col_conc <= 0: no cap)
    const int64_t w = c->col_bounds[b % c->J + 1] - c->col_bounds[b % c->J];
    const double conc = (double)((cnt + bl - 1) / bl) / (double)(w > 0 ? w : 1);
    if (max_col_conc > 0 && conc > max_col_conc) return true;
  }
  return false;
}

// ---- asynchronous steps (multi-GPU ring): begin, batches, end ----------
// The distributed trainer interleaves NCCL V-block moves with the strata of a
// step; each stratum's kernels are enqueued on the engine stream without a
// host sync, per-block SSEs accumulate in HBM, and step_end reads them once.
// Work-table slots are reserved for the whole step at begin (no reallocation
// while copies are in flight); plan positions are step-global so divergence
// keeps the reference's "first in plan order" rule.
int step_begin(bgmf_ctx* c, int max_blocks) {
  if (c->exact) return fail(c, BGMF_ERR_STATE, "asynchronous steps are fast-mode only");
  // each submitted block takes a sweep and an SSE work entry; the table is
  // split in two halves used by alternate steps (see ws_done)
  const size_t need = 2 * (size_t)(max_blocks > 0 ? max_blocks : 1);
  if (2 * need > c->work_cap) drain_async_steps(c);  // about to reallocate the table
  int rc = ensure_step_scratch(c, 2 * need);
  if (rc) return rc;
  const int h = c->ws_half ^= 1;
  if (c->ws_pending[h]) {
    BGMF_CK(c, cudaEventSynchronize(c->ws_done[h]));
    c->ws_pending[h] = false;
  }
  const int half = (int)(c->work_cap / 2);
  const int nb = c->I * c->J;
  BGMF_CK(c, cudaMemsetAsync(c->d_sse, 0, sizeof(double) * nb, c->stream));
  BGMF_CK(c, cudaMemsetAsync(c->d_bad, 0xFF, 8, c->stream));
  c->in_step = true;
  c->w_cursor = h * half;
  c->w_limit = h * half + half;
  c->submitted.clear();
  c->step_pos0 = 0;
  return BGMF_OK;
}

void drain_async_steps(bgmf_ctx* c) {
  for (int h = 0; h < 2; ++h)
    if (c->ws_pending[h]) {
      cudaEventSynchronize(c->ws_done[h]);
      c->ws_pending[h] = false;
    }
}

// End of a step's use of its work-table half (stream-ordered marker).
static int mark_half_done(bgmf_ctx* c) {
  const int h = c->ws_half;
  if (!c->ws_done[h]) BGMF_CK(c, cudaEventCreateWithFlags(&c->ws_done[h], cudaEventDisableTiming));
  BGMF_CK(c, cudaEventRecord(c->ws_done[h], c->stream));
  c->ws_pending[h] = true;
  return BGMF_OK;
}

int step_batch(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off_in, int nbatch_in,
               int iters, float alpha, float beta) {
  if (!c->in_step) return fail(c, BGMF_ERR_STATE, "bgmf_step_begin has not been called");
  if (c->streaming) {  // out-of-core rank: the batch's pieces through the slot ring
    const int pos0s = (int)c->submitted.size() - c->step_pos0;
    int rc = stream_batch(c, plan, batch_off_in, nbatch_in, iters, alpha, beta, pos0s);
    if (rc) return rc;
    for (int q = 0; q < batch_off_in[nbatch_in]; ++q) c->submitted.push_back(plan[q]);
    return BGMF_OK;
  }
  const std::vector<int32_t> waves = l2_waves(c, plan, batch_off_in, nbatch_in);
  const int32_t* batch_off = waves.data();
  const int nbatch = (int)waves.size() - 1;
  const int total = batch_off[nbatch];
  if (c->w_cursor + 2 * total > c->w_limit)
    return fail(c, BGMF_ERR_ARG, "more blocks than reserved by bgmf_step_begin");
  const Shape sh = shape_for(c->kp);
  const int gpw = 32 / sh.L;
  std::vector<BatchRange> ranges, sranges;
  // plan positions count from the start of the step (run_steps queues many
  // steps; pack_bad keeps 16 bits of position, and a step has <= 65535 blocks)
  const int pos0 = (int)c->submitted.size() - c->step_pos0;
  int rc = build_work(c, plan, batch_off, nbatch, sweep_groups(c, sh), ranges, nullptr,
                      c->w_cursor, pos0);
  if (rc) return rc;
  const int w_mid = ranges.empty() ? c->w_cursor : ranges.back().w0 + ranges.back().nw;
  rc = build_work(c, plan, batch_off, nbatch, sweep_groups(c, sh), sranges, nullptr, w_mid,
                  pos0, true);
  if (rc) return rc;
  const int w_end = sranges.empty() ? w_mid : sranges.back().w0 + sranges.back().nw;
  if (w_end > c->w_cursor)
    BGMF_CK(c, cudaMemcpyAsync(c->d_work + c->w_cursor, c->h_work + c->w_cursor,
                               sizeof(BlockWork) * (w_end - c->w_cursor), cudaMemcpyHostToDevice,
                               c->stream));
  for (int q = 0; q < total; ++q) c->submitted.push_back(plan[q]);
  for (int t = 0; t < nbatch; ++t) {
    const BatchRange& r = ranges[t];
    if (r.chunks == 0) continue;
    if (use_ordered(c, plan, batch_off[t], batch_off[t + 1])) {
      rc = run_batch_ordered(c, plan, batch_off[t], batch_off[t + 1], pos0, iters, alpha, beta);
      if (rc) return rc;
      continue;
    }
    const int warps = (r.chunks + gpw - 1) / gpw;
    const dim3 grid((warps + 7) / 8);
    double br = 0;
    for (int q = 0; q < r.nw; ++q)
      br += (double)(c->h_work[r.w0 + q].end - c->h_work[r.w0 + q].begin);
    const BatchRange& sr = sranges[t];
    const bool fuse = c->fuse_sse && sr.nw == r.nw && c->sse_async > 0 && !c->sse_wide &&
                      !c->bulk_red;
    bool fused_done = false;
    for (int it = 0; it < iters; ++it) {
      TimedLaunch* slot = nullptr;
      if (c->timing) record_begin(c, 0, br * (12.0 + 16.0 * c->k), &slot);
      if (fuse && it == iters - 1)  // the last sweep and the SSE: one launch
        fused_done = launch_sweep_sse(sh, grid, c->stream, c->d_work + r.w0, c->d_work + sr.w0,
                                      r.nw, r.chunks, c, alpha, beta, it);
      if (!fused_done)
        launch_fast(true, sh, grid, c->stream, c->d_work + r.w0, r.nw, r.chunks, c, alpha, beta,
                    it);
      if (slot) record_end(c, slot);
    }
    if (fused_done) continue;
    const dim3 sgrid(((sr.chunks + gpw - 1) / gpw + 7) / 8);
    TimedLaunch* slot = nullptr;
    if (c->timing) record_begin(c, 1, 0.0, &slot);
    launch_fast(false, sh, sgrid, c->stream, c->d_work + sr.w0, sr.nw, sr.chunks, c, alpha,
                beta, 0);
    if (slot) record_end(c, slot);
  }
  BGMF_CK(c, cudaGetLastError());
  c->w_cursor = w_end;
  return BGMF_OK;
}

// Several outer steps in one call (fixed inner iterations, nothing decided on
// the host between them -- train_blocked without early stopping): every
// step's strata are enqueued back to back on the stream, each step writing
// its own per-block SSE row and divergence word, so the GPU never idles on a
// host round trip between epochs.  ms_out[s] (optional): CUDA-event time of
// step s.  bad_out = {step, block id, entry, iteration} of the first diverged
// step, or -1s.
int run_steps(bgmf_ctx* c, int nsteps, const int32_t* plans, const int32_t* offs,
              const int32_t* nbatch, const int32_t* iters, float alpha, float beta,
              double* sse_out, int64_t* bad_out, float* ms_out) {
  if (c->exact) return fail(c, BGMF_ERR_STATE, "bgmf_run_steps is fast-mode only");
  if (c->streaming) return fail(c, BGMF_ERR_STATE, "bgmf_run_steps does not stream");
  drain_async_steps(c);
  const int nb = c->I * c->J;
  cudaStream_t s = c->stream;
  int64_t total = 0, plan_pos = 0, off_pos = 0;
  for (int k = 0; k < nsteps; ++k) {
    if (nbatch[k] < 0 || iters[k] < 1 || iters[k] > 65535)
      return fail(c, BGMF_ERR_ARG, "bad step description");
    const int32_t* off = offs + off_pos;
    for (int q = 0; q < off[nbatch[k]]; ++q)
      if (plans[plan_pos + q] < 0 || plans[plan_pos + q] >= nb)
        return fail(c, BGMF_ERR_ARG, "plan block id out of range");
    total += off[nbatch[k]];
    plan_pos += off[nbatch[k]];
    off_pos += nbatch[k] + 1;
  }
  int rc = ensure_step_scratch(c, 2 * (size_t)(total > 0 ? total : 1));  // sweep + SSE tables
  if (rc) return rc;
  double* d_sse = nullptr;
  unsigned long long* d_bad = nullptr;
  std::vector<cudaEvent_t> ev(ms_out ? (size_t)nsteps + 1 : 0, nullptr);
  auto cleanup = [&]() {
    dfree(d_sse, s);
    dfree(d_bad, s);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  };
  cudaError_t e = dmalloc(&d_sse, sizeof(double) * (size_t)nb * (nsteps > 0 ? nsteps : 1), s);
  if (e == cudaSuccess) e = dmalloc(&d_bad, 8 * (size_t)(nsteps > 0 ? nsteps : 1), s);
  for (size_t i = 0; i < ev.size() && e == cudaSuccess; ++i) e = cudaEventCreate(&ev[i]);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_sse, 0, sizeof(double) * (size_t)nb * nsteps, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_bad, 0xFF, 8 * (size_t)nsteps, s);
  if (e != cudaSuccess) { cleanup(); return cuda_fail(c, e, "run_steps setup"); }
  double* keep_sse = c->d_sse;
  unsigned long long* keep_bad = c->d_bad;
  c->in_step = true;
  c->w_cursor = 0;
  c->w_limit = (int)c->work_cap;
  c->submitted.clear();
  std::vector<int64_t> pos_start(nsteps);
  plan_pos = off_pos = 0;
  if (!ev.empty()) cudaEventRecord(ev[0], s);
  for (int k = 0; k < nsteps && !rc; ++k) {
    c->d_sse = d_sse + (size_t)k * nb;  // the stratum kernels address these through c
    c->d_bad = d_bad + k;
    const int32_t* off = offs + off_pos;
    pos_start[k] = (int64_t)c->submitted.size();
    c->step_pos0 = (int)pos_start[k];
    rc = step_batch(c, plans + plan_pos, off, nbatch[k], iters[k], alpha, beta);
    if (!ev.empty()) cudaEventRecord(ev[k + 1], s);
    plan_pos += off[nbatch[k]];
    off_pos += nbatch[k] + 1;
  }
  c->d_sse = keep_sse;
  c->d_bad = keep_bad;
  c->in_step = false;
  c->step_pos0 = 0;
  if (rc) { cudaStreamSynchronize(s); cleanup(); return rc; }
  std::vector<unsigned long long> hb((size_t)nsteps);
  e = cudaMemcpyAsync(sse_out, d_sse, sizeof(double) * (size_t)nb * nsteps, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(hb.data(), d_bad, 8 * (size_t)nsteps, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { cleanup(); return cuda_fail(c, e, "run_steps"); }
  for (int k = 0; k < nsteps && ms_out; ++k) cudaEventElapsedTime(&ms_out[k], ev[k], ev[k + 1]);
  if (c->timing) harvest_timing(c);
  bad_out[0] = bad_out[1] = bad_out[2] = bad_out[3] = -1;
  for (int k = 0; k < nsteps; ++k) {
    if (hb[k] == kNoBad) continue;
    const int64_t pos = pos_start[k] + (int64_t)(hb[k] >> 48);
    bad_out[0] = k;
    bad_out[1] = pos < (int64_t)c->submitted.size() ? c->submitted[pos] : -1;
    bad_out[2] = (int64_t)(hb[k] & 0xFFFFFFFFull);
    bad_out[3] = (int64_t)((hb[k] >> 32) & 0xFFFF);
    break;
  }
  cleanup();
  return BGMF_OK;
}

int step_end(bgmf_ctx* c, double* sse_out, int64_t* bad_out) {
  if (!c->in_step) return fail(c, BGMF_ERR_STATE, "bgmf_step_begin has not been called");
  c->in_step = false;
  if (int rc = mark_half_done(c)) return rc;
  const int nb = c->I * c->J;
  BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb, cudaMemcpyDeviceToHost,
                             c->stream));
  BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, c->stream));
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  if (c->timing) harvest_timing(c);
  for (int b = 0; b < nb; ++b) sse_out[b] = c->h_sse[b];
  const unsigned long long bad = *c->h_bad;
  if (bad == kNoBad) {
    bad_out[0] = bad_out[1] = bad_out[2] = -1;
  } else {
    const int64_t pos = (int64_t)(bad >> 48);
    bad_out[0] = pos < (int64_t)c->submitted.size() ? c->submitted[pos] : -1;
    bad_out[1] = (int64_t)(bad & 0xFFFFFFFFull);
    bad_out[2] = (int64_t)((bad >> 32) & 0xFFFF);
  }
  return BGMF_OK;
}


// step_end without a host round trip: the per-block SSEs and the raw
// divergence word are copied (stream-ordered) into caller device memory, so a
// caller can keep enqueueing steps and collectives and read every step's
// results once.  The word is pack_bad(plan position in submission order,
// iteration, entry) or kNoBad; the caller maps positions to blocks.
int step_end_async(bgmf_ctx* c, double* d_sse_out, unsigned long long* d_bad_out) {
  if (!c->in_step) return fail(c, BGMF_ERR_STATE, "bgmf_step_begin has not been called");
  c->in_step = false;
  if (int rc = mark_half_done(c)) return rc;
  const int nb = c->I * c->J;
  BGMF_CK(c, cudaMemcpyAsync(d_sse_out, c->d_sse, sizeof(double) * nb, cudaMemcpyDeviceToDevice,
                             c->stream));
  BGMF_CK(c, cudaMemcpyAsync(d_bad_out, c->d_bad, 8, cudaMemcpyDeviceToDevice, c->stream));
  return BGMF_OK;
}

// Sweeps (`iters` launches) + SSE launch for one piece of a batch whose
// ratings live at (lrow, lcol, val) -- the streaming path's unit of work.
int launch_piece(bgmf_ctx* c, const BlockWork* d_work, int nwork, int chunks,
                 const int32_t* lrow, const int32_t* lcol, const float* val, int iters,
                 float alpha, float beta, double ratings, int cbits) {
  if (chunks == 0) return BGMF_OK;
  const Shape sh = shape_for(c->kp);
  const int gpw = 32 / sh.L;
  const int warps = (chunks + gpw - 1) / gpw;
  const dim3 grid((warps + 7) / 8);
  for (int it = 0; it < iters; ++it) {
    TimedLaunch* slot = nullptr;
    if (c->timing) record_begin(c, 0, ratings * (12.0 + 16.0 * c->k), &slot);
    launch_fast_ptr(true, sh, grid, c->stream, d_work, nwork, chunks, lrow, lcol, val, c, alpha,
                    beta, it, cbits);
    if (slot) record_end(c, slot);
  }
  TimedLaunch* slot = nullptr;
  if (c->timing) record_begin(c, 1, 0.0, &slot);
  launch_fast_ptr(false, sh, grid, c->stream, d_work, nwork, chunks, lrow, lcol, val, c, alpha,
                  beta, 0, cbits);
  if (slot) record_end(c, slot);
  BGMF_CK(c, cudaGetLastError());
  return BGMF_OK;
}

// One sweep launch (inner iteration `it`) of a piece -- the streaming
// converge loop's unit (its SSE measurements use launch_piece with iters 0).
int launch_piece_sweep(bgmf_ctx* c, const BlockWork* d_work, int nwork, int chunks,
                       const int32_t* lrow, const int32_t* lcol, const float* val, float alpha,
                       float beta, int it, int cbits) {
  if (chunks == 0) return BGMF_OK;
  const Shape sh = shape_for(c->kp);
  const int gpw = 32 / sh.L;
  const dim3 grid(((chunks + gpw - 1) / gpw + 7) / 8);
  launch_fast_ptr(true, sh, grid, c->stream, d_work, nwork, chunks, lrow, lcol, val, c, alpha,
                  beta, it, cbits);
  BGMF_CK(c, cudaGetLastError());
  return BGMF_OK;
}

// Exact mode through the ordered schedule (ordered_exact_kernel): every batch
// whose blocks fit, bit-identical to the reference and parallel within the
// block.  Returns 1 (nothing run) when some batch cannot take it.
static int run_exact_ordered(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off,
                             int nbatch, int iters, double alpha, double beta, bool conv,
                             double tol, int64_t cap, int64_t* iters_out, int32_t* capped_out) {
  for (int t = 0; t < nbatch; ++t)
    if (!use_ordered(c, plan, batch_off[t], batch_off[t + 1])) return 1;
  cudaStream_t s = c->stream;
  const int nb = c->I * c->J;
  int rc = ensure_step_scratch(c, 1);
  if (rc) return rc;
  BGMF_CK(c, cudaMemsetAsync(c->d_sse, 0, sizeof(double) * nb, s));
  BGMF_CK(c, cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  const int n_it = conv ? (int)(cap > INT32_MAX ? INT32_MAX : cap) : iters;
  for (int t = 0; t < nbatch && !rc; ++t)
    rc = run_batch_ordered(c, plan, batch_off[t], batch_off[t + 1], 0, n_it, (float)alpha,
                           (float)beta, conv, tol, alpha, beta);
  if (rc) return rc;
  std::vector<int64_t> cv(conv ? (size_t)2 * nb : 0);
  BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb, cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
  if (conv && c->d_conv)
    BGMF_CK(c, cudaMemcpyAsync(cv.data(), c->d_conv, sizeof(int64_t) * 2 * nb,
                               cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaStreamSynchronize(s));
  if (conv)
    for (int b = 0; b < nb; ++b) {
      const bool ne = c->h_offsets[b + 1] > c->h_offsets[b];
      iters_out[b] = ne ? cv[2 * b] : 0;
      capped_out[b] = ne ? (int32_t)cv[2 * b + 1] : 0;
    }
  return BGMF_OK;
}

int run_step_exact(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off, int nbatch,
                   int iters, double alpha, double beta) {
  {
    const int rc = run_exact_ordered(c, plan, batch_off, nbatch, iters, alpha, beta, false, 0.0,
                                     0, nullptr, nullptr);
    if (rc != 1) return rc;
  }
  cudaStream_t s = c->stream;
  std::vector<BatchRange> ranges;
  int rc = build_work(c, plan, batch_off, nbatch, 0, ranges);
  if (rc) return rc;
  const int nw = ranges.empty() ? 0 : ranges.back().w0 + ranges.back().nw;
  const int nb = c->I * c->J;
  double* d_out = reinterpret_cast<double*>(c->d_work + c->work_cap);  // scratch after work
  if (nw > 0)
    BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * nw,
                               cudaMemcpyHostToDevice, s));
  for (int t = 0; t < nbatch; ++t) {
    const BatchRange& r = ranges[t];
    if (r.nw == 0) continue;
    block_exact_kernel<<<(r.nw + 31) / 32, 32, 0, s>>>(
        c->d_work + r.w0, r.nw, c->d_lrow, c->d_lcol, c->d_val64, c->d_u64, c->d_v64, c->k,
        alpha, beta, 0, iters, 0.0, 0, 0, d_out + 8 * r.w0);
  }
  BGMF_CK(c, cudaGetLastError());
  std::vector<double> out((size_t)8 * (nw > 0 ? nw : 1));
  if (nw > 0)
    BGMF_CK(c, cudaMemcpyAsync(out.data(), d_out, sizeof(double) * 8 * nw,
                               cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaStreamSynchronize(s));
  for (int b = 0; b < nb; ++b) c->h_sse[b] = 0.0;
  unsigned long long best = kNoBad;
  for (int q = 0; q < nw; ++q) {
    const BlockWork& bw = c->h_work[q];
    const double* o = &out[8 * q];
    c->h_sse[bw.block_id] = o[1];
    if (o[4] >= 0) {
      const unsigned long long key = pack_bad(bw.pos, (int64_t)o[5], (int64_t)o[4]);
      if (key < best) best = key;
    }
  }
  *c->h_bad = best;
  return BGMF_OK;
}

// One outer step of the synchronized row-sharded trainer (CPMF,
// baselines.py:100-182) on a 1x1 partition: shard w owns entries
// [edges[w], edges[w+1]) (whole rows), updates U in place and a private copy of
// V; the copies' deltas are merged in shard order.  A single shard works on V
// directly.  Exact mode: one fp64 thread per shard in the reference's order
// (bit-identical); fast mode: each shard is chunked over worker groups like a
// block of the stratum kernel, V copies in fp32.  sse_out[w] = the shard's
// post-sweep SSE; bad_out = {shard, entry, iteration} of the first diverged
// shard in shard order, or -1s.
int run_sync_parallel_step(bgmf_ctx* c, const int64_t* edges, int nshards, double alpha,
                           double beta, double* sse_out, int64_t* bad_out) {
  if (c->I != 1 || c->J != 1) return fail(c, BGMF_ERR_STATE, "sync-parallel needs a 1x1 partition");
  if (nshards < 1 || !edges || !sse_out || !bad_out) return fail(c, BGMF_ERR_ARG, "bad shards");
  for (int w = 0; w < nshards; ++w)
    if (edges[w] < 0 || edges[w] > edges[w + 1] || edges[w + 1] > c->nnz)
      return fail(c, BGMF_ERR_ARG, "shard edges must be non-decreasing within [0, nnz]");
  cudaStream_t s = c->stream;
  int rc = ensure_step_scratch(c, (size_t)nshards);
  if (rc) return rc;
  const bool priv = nshards > 1;
  const int64_t elems = c->m * (c->exact ? c->k : c->kp);
  const size_t esz = c->exact ? 8 : 4;
  if (priv) {
    const size_t need = (size_t)nshards * elems * esz;
    if (need > c->priv_bytes) {
      dfree(c->d_priv, s);
      c->d_priv = nullptr;
      c->priv_bytes = 0;
      BGMF_CK(c, dmalloc(&c->d_priv, need, s));
      c->priv_bytes = need;
    }
  }
  const int grid = c->num_sms * 4;
  if (c->exact) {
    double* V = c->d_v64;
    double* P = reinterpret_cast<double*>(c->d_priv);
    for (int w = 0; w < nshards; ++w) {
      BlockWork& bw = c->h_work[w];
      bw = BlockWork{edges[w], edges[w + 1], 0, priv ? (int64_t)w * c->m : 0, 0, 0, w, w};
    }
    BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * nshards,
                               cudaMemcpyHostToDevice, s));
    if (priv) broadcast_v<double><<<grid, 256, 0, s>>>(V, P, elems, nshards);
    double* d_out = reinterpret_cast<double*>(c->d_work + c->work_cap);
    block_exact_kernel<<<(nshards + 31) / 32, 32, 0, s>>>(
        c->d_work, nshards, c->d_lrow, c->d_lcol, c->d_val64, c->d_u64, priv ? P : V, c->k,
        alpha, beta, 0, 1, 0.0, 0, 0, d_out);
    if (priv) merge_private_v<double><<<grid, 256, 0, s>>>(V, P, elems, nshards);
    BGMF_CK(c, cudaGetLastError());
    std::vector<double> out((size_t)8 * nshards);
    BGMF_CK(c, cudaMemcpyAsync(out.data(), d_out, sizeof(double) * 8 * nshards,
                               cudaMemcpyDeviceToHost, s));
    BGMF_CK(c, cudaStreamSynchronize(s));
    bad_out[0] = bad_out[1] = bad_out[2] = -1;
    for (int w = 0; w < nshards; ++w) {
      sse_out[w] = out[8 * w + 1];
      if (bad_out[0] < 0 && out[8 * w + 4] >= 0) {
        bad_out[0] = w;
        bad_out[1] = (int64_t)out[8 * w + 4];
        bad_out[2] = (int64_t)out[8 * w + 5];
      }
    }
    return BGMF_OK;
  }
  if (c->ord_mode != 0 && ordered_block_ok(c, 0)) {
    // fast mode, ordered: each shard's rows in the reference's stored order
    // (ordered.cu), so the only difference from the reference is fp32
    std::vector<int32_t> lr(2 * (size_t)nshards, 0), r0(nshards), r1(nshards);
    for (int w = 0; w < nshards; ++w) {
      if (edges[w + 1] == edges[w]) continue;
      BGMF_CK(c, cudaMemcpyAsync(&lr[2 * w], c->d_lrow + edges[w], 4, cudaMemcpyDeviceToHost, s));
      BGMF_CK(c, cudaMemcpyAsync(&lr[2 * w + 1], c->d_lrow + edges[w + 1] - 1, 4,
                                 cudaMemcpyDeviceToHost, s));
    }
    BGMF_CK(c, cudaStreamSynchronize(s));
    for (int w = 0; w < nshards; ++w) {
      r0[w] = lr[2 * w];
      r1[w] = edges[w + 1] > edges[w] ? lr[2 * w + 1] + 1 : r0[w];
    }
    double* sse_dev = reinterpret_cast<double*>(c->d_work + c->work_cap);
    BGMF_CK(c, cudaMemsetAsync(sse_dev, 0, sizeof(double) * nshards, s));
    BGMF_CK(c, cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
    float* P = reinterpret_cast<float*>(c->d_priv);
    if (priv) broadcast_v<float><<<grid, 256, 0, s>>>(c->d_v, P, elems, nshards);
    rc = run_shards_ordered(c, r0.data(), r1.data(), edges, nshards, priv ? P : nullptr,
                            (float)alpha, (float)beta, sse_dev);
    if (rc) return rc;
    if (priv) merge_private_v<float><<<grid, 256, 0, s>>>(c->d_v, P, elems, nshards);
    BGMF_CK(c, cudaGetLastError());
    std::vector<double> out((size_t)nshards);
    BGMF_CK(c, cudaMemcpyAsync(out.data(), sse_dev, sizeof(double) * nshards,
                               cudaMemcpyDeviceToHost, s));
    BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
    BGMF_CK(c, cudaStreamSynchronize(s));
    if (c->timing) harvest_timing(c);
    for (int w = 0; w < nshards; ++w) sse_out[w] = out[w];
    const unsigned long long b = *c->h_bad;
    bad_out[0] = bad_out[1] = bad_out[2] = -1;
    if (b != kNoBad) {  // pos = shard
      bad_out[0] = (int64_t)(b >> 48);
      bad_out[1] = (int64_t)(b & 0xFFFFFFFFull);
      bad_out[2] = (int64_t)((b >> 32) & 0xFFFF);
    }
    return BGMF_OK;
  }
  // fast mode: shards as the "blocks" of one chunked launch
  const int64_t groups = fast_groups(c);
  int64_t total = 0;
  int nonempty = 0;
  for (int w = 0; w < nshards; ++w) {
    total += edges[w + 1] - edges[w];
    nonempty += edges[w + 1] > edges[w];
  }
  const int64_t slots = groups - nonempty > 0 ? groups - nonempty : 1;
  int64_t cl = (total + slots - 1) / slots;
  if (cl < c->min_chunk) cl = c->min_chunk;
      cl = stagger_chunk(cl, c->stagger);
  int nw = 0, chunks = 0;
  for (int w = 0; w < nshards; ++w) {
    const int64_t cnt = edges[w + 1] - edges[w];
    if (cnt == 0) continue;
    const int64_t bl = cl < cnt ? cl : cnt;
    c->h_work[nw++] = BlockWork{edges[w], edges[w + 1], 0, priv ? (int64_t)w * c->m : 0,
                                (int32_t)bl, chunks, w, w};
    chunks += (int)((cnt + bl - 1) / bl);
  }
  if (nw > 0)
    BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * nw,
                               cudaMemcpyHostToDevice, s));
  double* sse_dev = reinterpret_cast<double*>(c->d_work + c->work_cap);
  BGMF_CK(c, cudaMemsetAsync(sse_dev, 0, sizeof(double) * nshards, s));
  BGMF_CK(c, cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  float* V = c->d_v;
  float* P = reinterpret_cast<float*>(c->d_priv);
  if (priv) broadcast_v<float><<<grid, 256, 0, s>>>(V, P, elems, nshards);
  // the stratum kernels address V / the SSE array through the context
  double* keep_sse = c->d_sse;
  c->d_sse = sse_dev;
  if (priv) c->d_v = P;
  rc = launch_piece(c, c->d_work, nw, chunks, c->d_lrow, c->d_lcol, c->d_val, 1, (float)alpha,
                    (float)beta, (double)total, -1);
  c->d_v = V;
  c->d_sse = keep_sse;
  if (rc) return rc;
  if (priv) merge_private_v<float><<<grid, 256, 0, s>>>(V, P, elems, nshards);
  BGMF_CK(c, cudaGetLastError());
  std::vector<double> out((size_t)nshards);
  BGMF_CK(c, cudaMemcpyAsync(out.data(), sse_dev, sizeof(double) * nshards,
                             cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaStreamSynchronize(s));
  if (c->timing) harvest_timing(c);
  for (int w = 0; w < nshards; ++w) sse_out[w] = out[w];
  const unsigned long long b = *c->h_bad;
  if (b == kNoBad) {
    bad_out[0] = bad_out[1] = bad_out[2] = -1;
  } else {  // pos = shard
    bad_out[0] = (int64_t)(b >> 48);
    bad_out[1] = (int64_t)(b & 0xFFFFFFFFull);
    bad_out[2] = (int64_t)((b >> 32) & 0xFFFF);
  }
  return BGMF_OK;
}

int run_step_converge_exact(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off,
                            int nbatch, double tol, int64_t cap, double alpha, double beta,
                            int64_t* iters_out, int32_t* capped_out) {
  {
    const int rc = run_exact_ordered(c, plan, batch_off, nbatch, 0, alpha, beta, true, tol, cap,
                                     iters_out, capped_out);
    if (rc != 1) return rc;
  }
  cudaStream_t s = c->stream;
  std::vector<BatchRange> ranges;
  int rc = build_work(c, plan, batch_off, nbatch, 0, ranges);
  if (rc) return rc;
  const int nw = ranges.empty() ? 0 : ranges.back().w0 + ranges.back().nw;
  const int nb = c->I * c->J;
  double* d_out = reinterpret_cast<double*>(c->d_work + c->work_cap);
  if (nw > 0)
    BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * nw,
                               cudaMemcpyHostToDevice, s));
  for (int t = 0; t < nbatch; ++t) {
    const BatchRange& r = ranges[t];
    if (r.nw == 0) continue;
    block_exact_kernel<<<(r.nw + 31) / 32, 32, 0, s>>>(
        c->d_work + r.w0, r.nw, c->d_lrow, c->d_lcol, c->d_val64, c->d_u64, c->d_v64, c->k,
        alpha, beta, 1, 0, tol, cap, 1, d_out + 8 * r.w0);
  }
  BGMF_CK(c, cudaGetLastError());
  std::vector<double> out((size_t)8 * (nw > 0 ? nw : 1));
  if (nw > 0)
    BGMF_CK(c, cudaMemcpyAsync(out.data(), d_out, sizeof(double) * 8 * nw,
                               cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaStreamSynchronize(s));
  for (int b = 0; b < nb; ++b) { c->h_sse[b] = 0.0; iters_out[b] = 0; capped_out[b] = 0; }
  unsigned long long best = kNoBad;
  for (int q = 0; q < nw; ++q) {
    const BlockWork& bw = c->h_work[q];
    const double* o = &out[8 * q];
    c->h_sse[bw.block_id] = o[1];
    iters_out[bw.block_id] = (int64_t)o[2];
    capped_out[bw.block_id] = (int32_t)o[3];
    if (o[4] >= 0) {
      const unsigned long long key = pack_bad(bw.pos, (int64_t)o[5], (int64_t)o[4]);
      if (key < best) best = key;
    }
  }
  *c->h_bad = best;
  return BGMF_OK;
}

// Fast converge mode: per batch, sweep the still-active blocks, measure each
// block's post-sweep SSE, deactivate blocks whose RMSE improvement < tol.
// ---- ConvergeEachBlock on the device, chunked kernel -------------------
// sgd_converge (_kernels.py:62-100) for every block of a batch at once, with
// no host round trip per sweep: one CUDA graph per batch whose WHILE node
// repeats [sweep of the active blocks -> their post-sweep SSE -> conv_decide]
// while any block is active; conv_decide sets the node's condition
// (cudaGraphSetConditional).  A block's chunks in the work tables point at its
// active flag (BlockWork::active) and skip themselves once it is 0.
struct ConvState {
  double prev;     // RMSE of the last measurement
  int64_t iters;   // sweeps done
  int32_t capped;
  int32_t pad;
};

namespace {

__global__ void conv_prep(const BlockWork* __restrict__ w, int nw, int32_t* __restrict__ act) {
  for (int i = threadIdx.x; i < nw; i += blockDim.x) act[i] = w[i].end > w[i].begin ? 1 : 0;
}

// after the sse_before measurement
__global__ void conv_init(const BlockWork* __restrict__ w, int nw, double* __restrict__ sse,
                          ConvState* __restrict__ st, int32_t* __restrict__ act,
                          int32_t* __restrict__ iter, int64_t cap,
                          cudaGraphConditionalHandle h) {
  int any = 0;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) {
    const double cnt = (double)(w[i].end - w[i].begin);
    ConvState z{0.0, 0, 0, 0};
    if (cnt > 0) {
      z.prev = sqrt(sse[w[i].block_id] / cnt);
      if (cap > 0) {
        sse[w[i].block_id] = 0.0;  // the next measurement accumulates here
        any = 1;
      } else {
        z.capped = 1;  // no sweep allowed: sse_after = sse_before, capped
        act[i] = 0;
      }
    }
    st[i] = z;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    *iter = 0;
    cudaGraphSetConditional(h, any ? 1u : 0u);
  }
}

// after each sweep + SSE of the active blocks: the reference's stopping rule
__global__ void conv_decide(const BlockWork* __restrict__ w, int nw, double* __restrict__ sse,
                            ConvState* __restrict__ st, int32_t* __restrict__ act,
                            int32_t* __restrict__ iter, int64_t cap, double tol,
                            unsigned long long* __restrict__ bad,
                            cudaGraphConditionalHandle h) {
  int any = 0;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) {
    if (!act[i]) continue;
    ConvState z = st[i];
    const int64_t cnt = w[i].end - w[i].begin;
    const int b = w[i].block_id;
    ++z.iters;
    const double s2 = sse[b];
    if (!isfinite(s2)) {  // _kernels.py:88-89: (count - 1, iters - 1)
      atomicMin(bad, pack_bad(w[i].pos, z.iters - 1, cnt - 1));
      act[i] = 0;
    } else {
      const double now = sqrt(s2 / (double)cnt);
      if (z.prev - now < tol) {
        act[i] = 0;  // converged: sse_after stays
      } else {
        z.prev = now;
        if (z.iters >= cap) {
          act[i] = 0;
          z.capped = 1;
        } else {
          sse[b] = 0.0;
          any = 1;
        }
      }
    }
    st[i] = z;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    ++*iter;
    // a divergence anywhere ends the step (the trainer raises)
    cudaGraphSetConditional(h, (any && *bad == kNoBad) ? 1u : 0u);
  }
}

}  // namespace

// ConvergeEachBlock for the batches `ts` of a step through the chunked
// kernels, the loops on the device: ONE graph per step -- for each batch in
// plan order: prep -> sse_before -> init -> WHILE { sweep, SSE, decide } --
// launched once and read back once (per-block SSE in d_sse, iterations and
// capped flags in h_conv, batch-major).  Blocks of different batches are
// disjoint, so d_sse is zeroed once.
static int converge_step_graph(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off,
                               int nbatch, const std::vector<int>& ts, double tol, int64_t cap,
                               float alpha, float beta, std::vector<ConvState>& h_conv,
                               std::vector<BlockWork>& items) {
  cudaStream_t s = c->stream;
  const Shape sh = shape_for(c->kp);
  const int gpw = 32 / sh.L;
  std::vector<BatchRange> rg, srg;
  // both tables at once: growing the table between the two builds would drop the first
  int rc = ensure_step_scratch(c, 2 * (size_t)batch_off[nbatch]);
  if (rc) return rc;
  rc = build_work(c, plan, batch_off, nbatch, sweep_groups(c, sh), rg);
  if (rc) return rc;
  const int nw_all = rg.empty() ? 0 : rg.back().w0 + rg.back().nw;
  rc = build_work(c, plan, batch_off, nbatch, sweep_groups(c, sh), srg, nullptr, nw_all, 0, true);
  if (rc) return rc;
  // device state: per work item (all batches) flags + state, one iteration word per batch
  const int cap_items = nw_all > 64 ? nw_all : 64;
  if (!c->d_cstate || c->cstate_cap < cap_items) {
    dfree(c->d_cstate, s);
    c->cstate_cap = cap_items;
    BGMF_CK(c, dmalloc(reinterpret_cast<char**>(&c->d_cstate),
                       (size_t)c->cstate_cap * (sizeof(ConvState) + 8) + 16, s));
  }
  ConvState* st = reinterpret_cast<ConvState*>(c->d_cstate);
  int32_t* act = reinterpret_cast<int32_t*>(st + c->cstate_cap);
  int32_t* iters = act + c->cstate_cap;  // [batch]
  items.clear();
  for (int t : ts) {
    const BatchRange& r = rg[t];
    const BatchRange& sr = srg[t];
    if (sr.nw != r.nw) return fail(c, BGMF_ERR_STATE, "converge: work tables disagree");
    for (int q = 0; q < r.nw; ++q) {
      c->h_work[r.w0 + q].active = act + r.w0 + q;
      c->h_work[r.w0 + q].iter = iters + t;
      c->h_work[sr.w0 + q].active = act + r.w0 + q;
      c->h_work[sr.w0 + q].iter = nullptr;
      items.push_back(c->h_work[r.w0 + q]);
    }
  }
  if (items.empty()) return BGMF_OK;
  const int w_end = srg.back().w0 + srg.back().nw;
  BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * w_end,
                             cudaMemcpyHostToDevice, s));
  // instantiated graphs are cached per step plan, layout and hyper-parameters:
  // a run of steps cycles through P plans
  std::string key((const char*)plan, sizeof(int32_t) * batch_off[nbatch]);
  key.append((const char*)ts.data(), sizeof(int) * ts.size());
  {
    const double kv[4] = {(double)alpha, (double)beta, tol, (double)cap};
    const int64_t lv[9] = {(int64_t)(uintptr_t)c->d_sse, (int64_t)(uintptr_t)c->d_bad,
                           (int64_t)(uintptr_t)c->d_u,   (int64_t)(uintptr_t)c->d_v,
                           (int64_t)(uintptr_t)c->d_lrow, (int64_t)(uintptr_t)c->d_val,
                           (int64_t)(uintptr_t)c->d_work, (int64_t)(uintptr_t)c->d_cstate,
                           (int64_t)w_end};
    key.append((const char*)kv, sizeof kv).append((const char*)lv, sizeof lv);
  }
  cudaGraphExec_t ge = nullptr;
  auto hit = c->conv_graphs.find(key);
  if (hit != c->conv_graphs.end()) {
    ge = hit->second;
  } else {
    cudaStream_t cs = nullptr, cs2 = nullptr;
    cudaGraph_t g = nullptr;
    const bool pdl = c->pdl;
    c->pdl = false;  // plain serialised edges inside the graph
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_sse, 0, sizeof(double) * (size_t)c->I * c->J, cs);
    for (int t : ts) {
      const BatchRange& r = rg[t];
      const BatchRange& sr = srg[t];
      if (e != cudaSuccess || r.nw == 0) continue;
      cudaStreamCaptureStatus stt;
      cudaGraph_t cg = nullptr;
      cudaGraphConditionalHandle h = 0;
      e = cudaStreamGetCaptureInfo(cs, &stt, nullptr, &cg, nullptr, nullptr);
      if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault);
      const dim3 grid(((r.chunks + gpw - 1) / gpw + 7) / 8);
      const dim3 sgrid(((sr.chunks + gpw - 1) / gpw + 7) / 8);
      if (e == cudaSuccess) {
        conv_prep<<<1, 256, 0, cs>>>(c->d_work + r.w0, r.nw, act + r.w0);
        launch_fast(false, sh, sgrid, cs, c->d_work + sr.w0, sr.nw, sr.chunks, c, alpha, beta, 0);
        conv_init<<<1, 256, 0, cs>>>(c->d_work + r.w0, r.nw, c->d_sse, st + r.w0, act + r.w0,
                                     iters + t, cap, h);
        e = cudaGetLastError();
      }
      const cudaGraphNode_t* deps = nullptr;
      size_t ndeps = 0;
      if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(cs, &stt, nullptr, &cg, &deps, &ndeps);
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t cond = nullptr;
      if (e == cudaSuccess) e = cudaGraphAddNode(&cond, cg, deps, ndeps, &cp);
      if (e == cudaSuccess)
        e = cudaStreamUpdateCaptureDependencies(cs, &cond, 1, cudaStreamSetCaptureDependencies);
      if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(cs2, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed);
      if (e == cudaSuccess) {
        launch_fast(true, sh, grid, cs2, c->d_work + r.w0, r.nw, r.chunks, c, alpha, beta, 0);
        launch_fast(false, sh, sgrid, cs2, c->d_work + sr.w0, sr.nw, sr.chunks, c, alpha, beta,
                    0);
        conv_decide<<<1, 256, 0, cs2>>>(c->d_work + r.w0, r.nw, c->d_sse, st + r.w0, act + r.w0,
                                        iters + t, cap, tol, c->d_bad, h);
        e = cudaGetLastError();
        cudaGraph_t bg = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(cs2, &bg);
        if (e == cudaSuccess) e = e2;
      }
    }
    {
      cudaGraph_t gg = nullptr;
      const cudaError_t e3 = cudaStreamEndCapture(cs, &gg);
      g = gg;
      if (e == cudaSuccess) e = e3;
    }
    c->pdl = pdl;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
    if (g) cudaGraphDestroy(g);
    if (cs) cudaStreamDestroy(cs);
    if (cs2) cudaStreamDestroy(cs2);
    if (e != cudaSuccess) {
      if (ge) cudaGraphExecDestroy(ge);
      return cuda_fail(c, e, "device-side converge graph");
    }
    c->conv_graphs[key] = ge;
  }
  BGMF_CK(c, cudaGraphLaunch(ge, s));
  h_conv.resize(items.size());
  // state of the step's items, gathered in batch order
  std::vector<ConvState> all((size_t)(nw_all > 0 ? nw_all : 1));
  BGMF_CK(c, cudaMemcpyAsync(all.data(), st, sizeof(ConvState) * nw_all, cudaMemcpyDeviceToHost,
                             s));
  BGMF_CK(c, cudaStreamSynchronize(s));
  size_t o = 0;
  for (int t : ts)
    for (int q = 0; q < rg[t].nw; ++q) h_conv[o++] = all[rg[t].w0 + q];
  return BGMF_OK;
}

void conv_graphs_release(bgmf_ctx* c) {
  for (auto& kv : c->conv_graphs) cudaGraphExecDestroy(kv.second);
  c->conv_graphs.clear();
}

int run_step_converge_fast(bgmf_ctx* c, const int32_t* plan, const int32_t* batch_off,
                           int nbatch, double tol, int64_t cap, double alpha, double beta,
                           int64_t* iters_out, int32_t* capped_out) {
  cudaStream_t s = c->stream;
  const Shape sh = shape_for(c->kp);
  const int nb = c->I * c->J;
  const int64_t cl = sweep_groups(c, sh);
  std::vector<double> sse_final(nb, 0.0);
  for (int b = 0; b < nb; ++b) { iters_out[b] = 0; capped_out[b] = 0; }
  unsigned long long best = kNoBad;
  int rc0 = ensure_step_scratch(c, (size_t)batch_off[nbatch]);
  if (rc0) return rc0;
  BGMF_CK(c, cudaMemsetAsync(c->d_bad, 0xFF, 8, s));
  const int gpw = 32 / sh.L;
  std::vector<int64_t> conv((size_t)2 * nb);
  for (int t = 0; t < nbatch; ++t) {
    const int q0 = batch_off[t], q1 = batch_off[t + 1];
    if (use_ordered(c, plan, q0, q1)) {
      // the whole per-block converge loop on the device, in stored order (ordered.cu)
      const int capi = cap > INT32_MAX ? INT32_MAX : (int)cap;
      int rc = run_batch_ordered(c, plan, q0, q1, 0, capi, (float)alpha, (float)beta, true, tol);
      if (rc) return rc;
      BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb, cudaMemcpyDeviceToHost,
                                 s));
      BGMF_CK(c, cudaMemcpyAsync(conv.data(), c->d_conv, sizeof(int64_t) * 2 * nb,
                                 cudaMemcpyDeviceToHost, s));
      BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
      BGMF_CK(c, cudaStreamSynchronize(s));
      for (int q = q0; q < q1; ++q) {
        const int b = plan[q];
        if (c->h_offsets[b + 1] == c->h_offsets[b]) continue;
        sse_final[b] = c->h_sse[b];
        iters_out[b] = conv[2 * b];
        capped_out[b] = (int32_t)conv[2 * b + 1];
      }
      if (*c->h_bad != kNoBad) break;
      continue;
    }
    if (c->conv_graph && !c->streaming) {  // the loop on the device (converge_step_graph)
      std::vector<ConvState> hc;
      std::vector<BlockWork> items;
      // every remaining batch that also takes the chunked path joins this graph
      std::vector<int> ts;
      for (int t2 = t; t2 < nbatch; ++t2) {
        if (t2 > t && use_ordered(c, plan, batch_off[t2], batch_off[t2 + 1])) break;
        ts.push_back(t2);
      }
      int rc = converge_step_graph(c, plan, batch_off, nbatch, ts, tol, cap, (float)alpha,
                                   (float)beta, hc, items);
      if (rc) return rc;
      t = ts.back();  // the loop's ++t moves past the batches just run
      BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb, cudaMemcpyDeviceToHost,
                                 s));
      BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
      BGMF_CK(c, cudaStreamSynchronize(s));
      for (size_t q = 0; q < items.size(); ++q) {
        const int b = items[q].block_id;
        sse_final[b] = c->h_sse[b];
        iters_out[b] = hc[q].iters;
        capped_out[b] = hc[q].capped;
      }
      if (*c->h_bad != kNoBad) break;
      continue;
    }
    std::vector<char> active(batch_off[nbatch], 0);
    std::vector<double> prev(nb, 0.0);
    int n_active = 0;
    for (int q = q0; q < q1; ++q) {
      const int b = plan[q];
      if (c->h_offsets[b + 1] > c->h_offsets[b]) { active[q] = 1; ++n_active; }
    }
    // sse_before of the active blocks
    auto measure = [&](std::vector<double>& out) -> int {
      std::vector<BatchRange> rg;
      int rc = build_work(c, plan + 0, batch_off, nbatch, cl, rg, &active);
      if (rc) return rc;
      const BatchRange& r = rg[t];
      BGMF_CK(c, cudaMemsetAsync(c->d_sse, 0, sizeof(double) * nb, s));
      if (r.chunks > 0) {
        BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work + r.w0, sizeof(BlockWork) * r.nw,
                                   cudaMemcpyHostToDevice, s));
        const int warps = (r.chunks + gpw - 1) / gpw;
        launch_fast(false, sh, dim3((warps + 7) / 8), s, c->d_work, r.nw, r.chunks, c,
                    (float)alpha, (float)beta, 0);
      }
      BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb,
                                 cudaMemcpyDeviceToHost, s));
      BGMF_CK(c, cudaStreamSynchronize(s));
      for (int b = 0; b < nb; ++b) out[b] = c->h_sse[b];
      return BGMF_OK;
    };
    std::vector<double> cur(nb, 0.0);
    int rc = measure(cur);
    if (rc) return rc;
    for (int q = q0; q < q1; ++q) {
      const int b = plan[q];
      const double cnt = (double)(c->h_offsets[b + 1] - c->h_offsets[b]);
      if (active[q]) prev[b] = std::sqrt(cur[b] / cnt);
    }
    int64_t it = 0;
    while (n_active > 0 && it < cap) {
      std::vector<BatchRange> rg;
      rc = build_work(c, plan, batch_off, nbatch, cl, rg, &active);
      if (rc) return rc;
      const BatchRange& r = rg[t];
      if (r.chunks > 0) {
        BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work + r.w0, sizeof(BlockWork) * r.nw,
                                   cudaMemcpyHostToDevice, s));
        const int warps = (r.chunks + gpw - 1) / gpw;
        launch_fast(true, sh, dim3((warps + 7) / 8), s, c->d_work, r.nw, r.chunks, c,
                    (float)alpha, (float)beta, (int)(it & 0xFFFF));
      }
      BGMF_CK(c, cudaGetLastError());
      ++it;
      rc = measure(cur);
      if (rc) return rc;
      BGMF_CK(c, cudaMemcpyAsync(c->h_bad, c->d_bad, 8, cudaMemcpyDeviceToHost, s));
      BGMF_CK(c, cudaStreamSynchronize(s));
      for (int q = q0; q < q1; ++q) {
        if (!active[q]) continue;
        const int b = plan[q];
        const int64_t cnt = c->h_offsets[b + 1] - c->h_offsets[b];
        iters_out[b] = it;
        sse_final[b] = cur[b];
        const double now = std::sqrt(cur[b] / (double)cnt);
        if (!std::isfinite(cur[b])) {
          const unsigned long long key = pack_bad(q, it - 1, cnt - 1);
          if (key < best) best = key;
          active[q] = 0; --n_active;
        } else if (prev[b] - now < tol) {
          active[q] = 0; --n_active;
        } else {
          prev[b] = now;
        }
      }
      if (*c->h_bad != kNoBad) break;
    }
    for (int q = q0; q < q1; ++q)
      if (active[q]) capped_out[plan[q]] = 1;
    if (*c->h_bad != kNoBad) break;
  }
  for (int b = 0; b < nb; ++b) c->h_sse[b] = sse_final[b];
  if (*c->h_bad < best) best = *c->h_bad;
  *c->h_bad = best;
  return BGMF_OK;
}

int train_sse_fast(bgmf_ctx* c, double* out) {
  const int nb = c->I * c->J;
  std::vector<int32_t> plan(nb), off{0, nb};
  for (int b = 0; b < nb; ++b) plan[b] = b;
  const Shape sh = shape_for(c->kp);
  std::vector<BatchRange> ranges;
  int rc = build_work(c, plan.data(), off.data(), 1, sweep_groups(c, sh), ranges);
  if (rc) return rc;
  cudaStream_t s = c->stream;
  BGMF_CK(c, cudaMemsetAsync(c->d_sse, 0, sizeof(double) * nb, s));
  const BatchRange& r = ranges[0];
  if (r.chunks > 0) {
    BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * r.nw,
                               cudaMemcpyHostToDevice, s));
    const int gpw = 32 / sh.L;
    const int warps = (r.chunks + gpw - 1) / gpw;
    launch_fast(false, sh, dim3((warps + 7) / 8), s, c->d_work, r.nw, r.chunks, c, 0.f, 0.f, 0);
  }
  BGMF_CK(c, cudaGetLastError());
  BGMF_CK(c, cudaMemcpyAsync(c->h_sse, c->d_sse, sizeof(double) * nb, cudaMemcpyDeviceToHost, s));
  BGMF_CK(c, cudaStreamSynchronize(s));
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) acc += c->h_sse[b];
  *out = acc;
  return BGMF_OK;
}

int train_sse_exact(bgmf_ctx* c, double* out) {
  const int nb = c->I * c->J;
  std::vector<int32_t> plan(nb), off{0, nb};
  for (int b = 0; b < nb; ++b) plan[b] = b;
  std::vector<BatchRange> ranges;
  int rc = build_work(c, plan.data(), off.data(), 1, 0, ranges);
  if (rc) return rc;
  cudaStream_t s = c->stream;
  const int nw = ranges[0].nw;
  double* d_out = reinterpret_cast<double*>(c->d_work + c->work_cap);
  double acc = 0.0;
  if (nw > 0) {
    BGMF_CK(c, cudaMemcpyAsync(c->d_work, c->h_work, sizeof(BlockWork) * nw,
                               cudaMemcpyHostToDevice, s));
    // iters = 0 sweeps: o[1] = post-"sweep" SSE of the untouched block
    block_exact_kernel<<<(nw + 31) / 32, 32, 0, s>>>(c->d_work, nw, c->d_lrow, c->d_lcol,
                                                     c->d_val64, c->d_u64, c->d_v64, c->k, 0.0,
                                                     0.0, 0, 0, 0.0, 0, 0, d_out);
    BGMF_CK(c, cudaGetLastError());
    std::vector<double> o((size_t)8 * nw);
    BGMF_CK(c, cudaMemcpyAsync(o.data(), d_out, sizeof(double) * 8 * nw, cudaMemcpyDeviceToHost, s));
    BGMF_CK(c, cudaStreamSynchronize(s));
    for (int q = 0; q < nw; ++q) acc += o[8 * q + 1];
  }
  *out = acc;
  return BGMF_OK;
}

int block_exact(bgmf_ctx* c, const int64_t* rows, const int64_t* cols, const double* vals,
                int64_t count, double* u, int64_t u_rows, double* v, int64_t v_rows, int k,
                double alpha, double beta, int mode, int iters, double tol, int64_t cap,
                double* out6) {
  if (k < 1 || count < 0 || u_rows < 0 || v_rows < 0)
    return fail(c, BGMF_ERR_ARG, "bad block shape");
  for (int64_t i = 0; i < count; ++i) {
    if (rows[i] < 0 || rows[i] >= u_rows || cols[i] < 0 || cols[i] >= v_rows)
      return fail(c, BGMF_ERR_ARG, "block entry index outside its factor slice");
  }
  cudaStream_t s = c->stream;
  const size_t N = (size_t)(count > 0 ? count : 1);
  std::vector<int32_t> r32(N), c32(N);
  for (int64_t i = 0; i < count; ++i) { r32[i] = (int32_t)rows[i]; c32[i] = (int32_t)cols[i]; }
  int32_t *dr = nullptr, *dc = nullptr;
  double *dv = nullptr, *du = nullptr, *dV = nullptr, *dout = nullptr;
  BlockWork* dw = nullptr;
  int rc = BGMF_OK;
  auto cleanup = [&]() {
    dfree(dr, c->stream); dfree(dc, c->stream); dfree(dv, c->stream); dfree(du, c->stream); dfree(dV, c->stream); dfree(dout, c->stream);
    dfree(dw, c->stream);
  };
#define XCK(call)                                                                       \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) { rc = cuda_fail(c, _e, #call); cleanup(); return rc; }      \
  } while (0)
  XCK(dmalloc(&dr, N * 4, c->stream));
  XCK(dmalloc(&dc, N * 4, c->stream));
  XCK(dmalloc(&dv, N * 8, c->stream));
  XCK(dmalloc(&du, (size_t)(u_rows > 0 ? u_rows : 1) * k * 8, c->stream));
  XCK(dmalloc(&dV, (size_t)(v_rows > 0 ? v_rows : 1) * k * 8, c->stream));
  XCK(dmalloc(&dout, 8 * 8, c->stream));
  XCK(dmalloc(&dw, sizeof(BlockWork), c->stream));
  BlockWork w{0, count, 0, 0, 0, 0, 0, 0};
  XCK(cudaMemcpyAsync(dw, &w, sizeof w, cudaMemcpyHostToDevice, s));
  if (count > 0) {
    XCK(cudaMemcpyAsync(dr, r32.data(), count * 4, cudaMemcpyHostToDevice, s));
    XCK(cudaMemcpyAsync(dc, c32.data(), count * 4, cudaMemcpyHostToDevice, s));
    XCK(cudaMemcpyAsync(dv, vals, count * 8, cudaMemcpyHostToDevice, s));
  }
  if (u_rows > 0) XCK(cudaMemcpyAsync(du, u, (size_t)u_rows * k * 8, cudaMemcpyHostToDevice, s));
  if (v_rows > 0) XCK(cudaMemcpyAsync(dV, v, (size_t)v_rows * k * 8, cudaMemcpyHostToDevice, s));
  block_exact_kernel<<<1, 32, 0, s>>>(dw, 1, dr, dc, dv, du, dV, k, alpha, beta,
                                      mode == 1 ? 1 : 0, iters, tol, cap, 1, dout);
  XCK(cudaGetLastError());
  double o[8];
  XCK(cudaMemcpyAsync(o, dout, 8 * 8, cudaMemcpyDeviceToHost, s));
  if (mode != 2) {  // mode 2: block_sse, factors untouched
    if (u_rows > 0) XCK(cudaMemcpyAsync(u, du, (size_t)u_rows * k * 8, cudaMemcpyDeviceToHost, s));
    if (v_rows > 0) XCK(cudaMemcpyAsync(v, dV, (size_t)v_rows * k * 8, cudaMemcpyDeviceToHost, s));
  }
  XCK(cudaStreamSynchronize(s));
#undef XCK
  for (int i = 0; i < 6; ++i) out6[i] = o[i];
  cleanup();
  return BGMF_OK;
}

}  // namespace bgmf
