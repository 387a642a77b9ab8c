// partition.cu -- GPU block partitioner, bit-exact with the reference
// BlockedDataset (reference pkg/src/blockmf/partition.py:112-136).
//
// The reference computes block ids with searchsorted over balanced slab
// bounds (partition.py:18-37,120-122) and orders entries with
// np.lexsort((cols, rows, block_id)) -- (block, row, col), ties in input
// order.  Here:
//   1. make_keys: closed-form slab index (first n % P slabs are one longer),
//      one 64-bit key per rating = block | local row | local col.  Within a
//      block, (local row, local col) orders exactly like (row, col).  When the
//      source index fits in the key's spare low bits (fast mode: C1-C4) it is
//      appended there and the fp32 value rides along as the payload, so the
//      sort needs no gather afterwards; otherwise the payload is the index.
//   2. LSD radix sort over the key bits, 8- or 9-bit digits, stable: tile
//      histogram (shared-memory atomics) -> per-digit tile scan -> scatter.
//      The scatter ranks a tile's items per warp (__match_any_sync, in
//      order), lays the tile out digit-major in shared memory and writes each
//      digit's run contiguously, so global stores are coalesced runs instead
//      of one scattered 8 B store per lane.  Duplicate cells keep input order
//      like lexsort.
//   3. decode: local coords from the key (and the source index from its low
//      bits, or the fp64/fp32 value gathered by source index when it is the
//      payload), block offsets by binary search.
// HBM-bound integer work: every pass streams key+payload (12 B/rating) in and
// out; grid sized to tiles of 4096 ratings.

#include <omp.h>

#include <algorithm>
#include <cmath>

#include <thread>

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
constexpr int RS_WARPS = RS_THREADS / 32;

__device__ __forceinline__ int64_t slab_index(int64_t x, int64_t base, int64_t extra) {
  const int64_t big = extra * (base + 1);
  if (x < (int64_t)UINT32_MAX && base < (int64_t)UINT32_MAX)  // 32-bit divides
    return x < big ? (uint32_t)x / (uint32_t)(base + 1)
                   : extra + (uint32_t)(x - big) / (uint32_t)base;
  return x < big ? x / (base + 1) : extra + (x - big) / base;
}
__device__ __forceinline__ int64_t slab_start(int64_t s, int64_t base, int64_t extra) {
  return s * base + (s < extra ? s : extra);
}

// payload: the source index, or (embed) the fp32 value's bits with the index
// in the key's low ibits.
template <typename IT>
__global__ void make_keys(const IT* __restrict__ rows, const IT* __restrict__ cols,
                          int64_t nnz, int64_t n, int64_t m, int64_t rbase, int64_t rextra,
                          int64_t cbase, int64_t cextra, int J, int rbits, int cbits, int ibits,
                          const float* __restrict__ vals32, uint64_t* __restrict__ keys,
                          uint32_t* __restrict__ payload, unsigned long long* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (int64_t)rows[i], c = (int64_t)cols[i];
    payload[i] = vals32 ? __float_as_uint(vals32[i]) : (uint32_t)i;
    if (r < 0 || r >= n || c < 0 || c >= m) {
      atomicMin(bad, (unsigned long long)i);
      keys[i] = 0;
      continue;
    }
    const int64_t bi = slab_index(r, rbase, rextra);
    const int64_t bj = slab_index(c, cbase, cextra);
    const uint64_t lr = (uint64_t)(r - slab_start(bi, rbase, rextra));
    const uint64_t lc = (uint64_t)(c - slab_start(bj, cbase, cextra));
    const uint64_t key = ((uint64_t)(bi * J + bj) << (rbits + cbits)) | (lr << cbits) | lc;
    keys[i] = (key << ibits) | (ibits ? (uint64_t)i : 0ull);
  }
}

// Per-tile digit histogram, written digit-major: hist[d * ntiles + tile].
// RD = buckets per pass (256: 8-bit digits, 512: 9-bit digits).
template <int RD>
__global__ void __launch_bounds__(RS_THREADS)
radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift, int64_t ntiles,
           uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[RD];
  for (int d = threadIdx.x; d < RD; d += RS_THREADS) h[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
  uint64_t k[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    const int64_t i = base + (int64_t)j * RS_THREADS + threadIdx.x;
    k[j] = i < n ? __ldcs(keys + i) : ~0ull;
  }
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j)
    if (base + (int64_t)j * RS_THREADS + threadIdx.x < n)
      atomicAdd(&h[(unsigned)(k[j] >> shift) & (RD - 1u)], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < RD; d += RS_THREADS) hist[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

// One CTA per digit: exclusive scan of hist[d * ntiles + 0 .. ntiles) in
// place; digit total to totals[d].
__global__ void __launch_bounds__(1024)
radix_scan_tiles(uint32_t* __restrict__ hist, int64_t ntiles, uint32_t* __restrict__ totals) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t chunk_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* row = hist + (int64_t)blockIdx.x * ntiles;
  uint32_t carry = 0;
  for (int64_t t0 = 0; t0 < ntiles; t0 += 1024) {
    const int64_t t = t0 + threadIdx.x;
    const uint32_t x = t < ntiles ? row[t] : 0u;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t s = wsum[lane];
      uint32_t si = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, si, o);
        if (lane >= o) si += y;
      }
      wsum[lane] = si - s;
      if (lane == 31) chunk_total = si;
    }
    __syncthreads();
    if (t < ntiles) row[t] = carry + wsum[warp] + incl - x;
    carry += chunk_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

// Stable scatter of one tile.  Warp w owns tile items [w*512, (w+1)*512),
// walked 32 at a time in order; an item's rank among its warp's equal digits
// comes from __match_any_sync plus a per-(warp, digit) counter.  A CTA scan
// over (digit, warp) turns those into tile positions (digit-major, stable);
// the tile is laid out there in shared memory and thread t then writes items
// t, t+256, ... to global[digit base + tile digit offset + (i - tile digit
// start)], so each digit's run is stored contiguously.
template <int RD>
constexpr size_t scatter_smem() {
  return (size_t)RS_TILE * 12 + (size_t)RS_WARPS * RD * 4 + (size_t)RD * 4;
}

template <int RD>
__global__ void __launch_bounds__(RS_THREADS)
radix_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
              uint64_t* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n, int shift,
              const uint32_t* __restrict__ hist, int64_t ntiles,
              const uint32_t* __restrict__ totals) {
  constexpr int DPT = RD / RS_THREADS;  // digits per thread
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* skey = reinterpret_cast<uint64_t*>(smem);
  uint32_t* sval = reinterpret_cast<uint32_t*>(skey + RS_TILE);
  uint32_t* woff = sval + RS_TILE;          // [RS_WARPS][RD]
  uint32_t* gdst = woff + RS_WARPS * RD;  // [RD], mod 2^32
  __shared__ uint32_t wsum[2][RS_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  const int64_t tbase = (int64_t)blockIdx.x * RS_TILE;

#pragma unroll
  for (int w = 0; w < RS_WARPS; ++w)
#pragma unroll
    for (int q = 0; q < DPT; ++q) woff[w * RD + tid * DPT + q] = 0;

  const int64_t wbase = tbase + (int64_t)warp * (32 * RS_ITEMS);
  uint64_t key[RS_ITEMS];
  uint32_t val[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    const int64_t i = wbase + j * 32 + lane;
    key[j] = i < n ? __ldcs(kin + i) : 0ull;
    val[j] = i < n ? __ldcs(vin + i) : 0u;
  }
  __syncthreads();
  // rank within the warp (in item order)
  const unsigned lt = (1u << lane) - 1u;
  uint32_t* my = woff + warp * RD;
  uint32_t rank[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    const bool valid = wbase + j * 32 + lane < n;
    const unsigned vm = __ballot_sync(kFull, valid);
    const unsigned d = (unsigned)(key[j] >> shift) & (RD - 1u);
    unsigned peers = 0;
    uint32_t before = 0;
    if (valid) {
      peers = __match_any_sync(vm, d);
      before = my[d];
    }
    rank[j] = before + (uint32_t)__popc(peers & lt);
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) my[d] = before + (uint32_t)__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // tile positions: exclusive scan over digits (thread tid owns digits
  // [tid*DPT, tid*DPT+DPT)), then over warps inside each digit; and the global
  // digit bases (scan of totals + this tile's offset within each digit)
  {
    uint32_t cnt[DPT], tot[DPT], mine = 0, gmine = 0;
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
      cnt[q] = 0;
#pragma unroll
      for (int w = 0; w < RS_WARPS; ++w) cnt[q] += woff[w * RD + tid * DPT + q];
      mine += cnt[q];
      tot[q] = totals[tid * DPT + q];
      gmine += tot[q];
    }
    uint32_t incl = mine, gincl = gmine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      const uint32_t gy = __shfl_up_sync(kFull, gincl, o);
      if (lane >= o) { incl += y; gincl += gy; }
    }
    if (lane == 31) { wsum[0][warp] = incl; wsum[1][warp] = gincl; }
    __syncthreads();
    uint32_t run = incl - mine, grun = gincl - gmine;
    for (int w = 0; w < warp; ++w) { run += wsum[0][w]; grun += wsum[1][w]; }
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
      const int d = tid * DPT + q;
      gdst[d] = grun + hist[(int64_t)d * ntiles + blockIdx.x] - run;
      uint32_t r = run;
#pragma unroll
      for (int w = 0; w < RS_WARPS; ++w) {
        const uint32_t c = woff[w * RD + d];
        woff[w * RD + d] = r;
        r += c;
      }
      run += cnt[q];
      grun += tot[q];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    if (wbase + j * 32 + lane < n) {
      const unsigned d = (unsigned)(key[j] >> shift) & (RD - 1u);
      const uint32_t p = my[d] + rank[j];
      skey[p] = key[j];
      sval[p] = val[j];
    }
  }
  __syncthreads();
  const int64_t valid_n = n - tbase < RS_TILE ? n - tbase : RS_TILE;
#pragma unroll 4
  for (int j = 0; j < RS_ITEMS; ++j) {
    const int i = j * RS_THREADS + tid;
    if (i < valid_n) {
      const uint64_t k = skey[i];
      const unsigned d = (unsigned)(k >> shift) & (RD - 1u);
      const uint32_t p = gdst[d] + (uint32_t)i;  // < nnz < 2^32
      __stcs(kout + p, k);
      __stcs(vout + p, sval[i]);
    }
  }
}

__global__ void block_offsets(const uint64_t* __restrict__ keys, int64_t n, int nblocks,
                              int shift, int64_t* __restrict__ off) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nblocks) return;
  if (b == nblocks) {
    off[b] = n;
    return;
  }
  const uint64_t target = (uint64_t)b << shift;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < target) lo = mid + 1; else hi = mid;
  }
  off[b] = lo;
}

template <typename VT>
__global__ void decode(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                       const VT* __restrict__ vin, int64_t n, int cbits, uint64_t rmask,
                       uint64_t cmask, int32_t* __restrict__ lrow, int32_t* __restrict__ lcol,
                       float* __restrict__ val, double* __restrict__ val64,
                       uint32_t* __restrict__ order) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const uint32_t o = idx[i];
    lrow[i] = (int32_t)((k >> cbits) & rmask);
    lcol[i] = (int32_t)(k & cmask);
    order[i] = o;
    const VT x = vin[o];
    val[i] = (float)x;
    if (val64) val64[i] = (double)x;
  }
}

// Embedded layout: source index in the key's low ibits, fp32 value bits as
// the payload -- no gather.
__global__ void decode_embedded(const uint64_t* __restrict__ keys,
                                const uint32_t* __restrict__ vbits, int64_t n, int ibits,
                                int cbits, uint64_t rmask, uint64_t cmask,
                                int32_t* __restrict__ lrow, int32_t* __restrict__ lcol,
                                float* __restrict__ val, uint32_t* __restrict__ order) {
  const uint64_t imask = (1ull << ibits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = __ldcs(keys + i);
    order[i] = (uint32_t)(k & imask);
    const uint64_t kk = k >> ibits;
    lrow[i] = (int32_t)((kk >> cbits) & rmask);
    lcol[i] = (int32_t)(kk & cmask);
    val[i] = __uint_as_float(__ldcs(vbits + i));
  }
}

// out-of-core chunks: packed (row << cbits | col) records and the input index
// of every partitioned entry (gidx = the chunk's input indices)
__global__ void pack_and_order(const int32_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                               const uint32_t* __restrict__ order,
                               const uint32_t* __restrict__ gidx, int64_t n, int cbits,
                               int32_t* __restrict__ rec, uint32_t* __restrict__ gorder) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (rec) rec[i] = (int32_t)(((uint32_t)lrow[i] << cbits) | (uint32_t)lcol[i]);
    gorder[i] = gidx[order[i]];
  }
}

int bits_for(uint64_t maxval) {  // bits to represent 0..maxval
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

template <typename T>
void free_dev(T*& p, cudaStream_t s) {
  if (p) dfree(p, s);
  p = nullptr;
}

}  // namespace

// Stable LSD radix sort of (key, payload) pairs over key bits [lo_bit, lo_bit + bits), with
// the partitioner's kernels.  *keys / *vals are swapped with the sorted
// buffers (the caller frees whatever they point to afterwards).  Used by the
// ordered sweep's column-rank index (ordered.cu).
int sort_pairs_device(bgmf_ctx* ctx, uint64_t** keys, uint32_t** vals, int64_t n, int bits,
                      int lo_bit) {
  if (n <= 1 || bits <= 0) return BGMF_OK;
  cudaStream_t s = ctx->stream;
  const bool wide = (bits + 8) / 9 < (bits + 7) / 8;
  const int dbits = wide ? 9 : 8, RD = 1 << dbits;
  const int passes = (bits + dbits - 1) / dbits;
  const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  uint64_t* kb = nullptr;
  uint32_t *ib = nullptr, *hist = nullptr, *tot = nullptr;
  auto cleanup = [&]() { free_dev(kb, s); free_dev(ib, s); free_dev(hist, s); free_dev(tot, s); };
  cudaError_t e = dmalloc(&kb, (size_t)n * 8, s);
  if (e == cudaSuccess) e = dmalloc(&ib, (size_t)n * 4, s);
  if (e == cudaSuccess) e = dmalloc(&hist, (size_t)RD * ntiles * 4, s);
  if (e == cudaSuccess) e = dmalloc(&tot, (size_t)RD * 4, s);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(&radix_scatter<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)scatter_smem<512>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(&radix_scatter<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)scatter_smem<256>());
  if (e != cudaSuccess) { cleanup(); return cuda_fail(ctx, e, "sort_pairs_device"); }
  uint64_t* ka = *keys;
  uint32_t* ia = *vals;
  for (int p = 0; p < passes; ++p) {
    const int shift = lo_bit + dbits * p;
    if (wide) {
      radix_hist<512><<<(unsigned)ntiles, RS_THREADS, 0, s>>>(ka, n, shift, ntiles, hist);
      radix_scan_tiles<<<512, 1024, 0, s>>>(hist, ntiles, tot);
      radix_scatter<512><<<(unsigned)ntiles, RS_THREADS, scatter_smem<512>(), s>>>(
          ka, ia, kb, ib, n, shift, hist, ntiles, tot);
    } else {
      radix_hist<256><<<(unsigned)ntiles, RS_THREADS, 0, s>>>(ka, n, shift, ntiles, hist);
      radix_scan_tiles<<<256, 1024, 0, s>>>(hist, ntiles, tot);
      radix_scatter<256><<<(unsigned)ntiles, RS_THREADS, scatter_smem<256>(), s>>>(
          ka, ia, kb, ib, n, shift, hist, ntiles, tot);
    }
    uint64_t* tk = ka; ka = kb; kb = tk;
    uint32_t* ti = ia; ia = ib; ib = ti;
  }
  e = cudaGetLastError();
  *keys = ka;
  *vals = ia;
  cleanup();  // the spare buffers (kb/ib now hold the other halves)
  return e == cudaSuccess ? BGMF_OK : cuda_fail(ctx, e, "sort_pairs_device");
}

// dev_in: rows/cols/vals are device buffers whose ownership passes to this
// call (freed as soon as they are consumed); otherwise host arrays.
// Skew statistic of a partition (routes the sweep's u_ring, sgd.cu): the
// coefficient of variation of the ratings per user.  Entries are sorted by
// (block, row), so a warp's equal rows are neighbours: one atomic per distinct
// (block, row) run per warp (__match_any_sync), then sum of squares.
__global__ void row_hist(const int32_t* __restrict__ lrow, const int64_t* __restrict__ off,
                         int nb, int J, int64_t rbase, int64_t rextra, int64_t nnz,
                         unsigned* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
       base < nnz; base += warps * 32) {
    const int64_t i = base + lane;
    long long grow = -1;
    if (i < nnz) {
      int lo = 0, hi = nb - 1;  // last block b with off[b] <= i
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= i) lo = mid; else hi = mid - 1;
      }
      const int64_t bi = lo / J;
      grow = bi * rbase + min(bi, rextra) + __ldg(lrow + i);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, grow);
    if (grow >= 0 && lane == __ffs(peers) - 1) atomicAdd(cnt + grow, (unsigned)__popc(peers));
  }
}

__global__ void sum_squares(const unsigned* __restrict__ cnt, int64_t n,
                            unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = cnt[i];
    acc += c * c;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

int partition_device(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols,
                     const double* vals, int64_t nnz, int64_t n, int64_t m, int I, int J,
                     bool dev_in, int64_t row_lo, int64_t row_hi) {
  if (row_hi < 0) row_hi = n;
  if (row_lo < 0 || row_lo > row_hi || row_hi > n)
    return fail(ctx, BGMF_ERR_ARG, "row range must satisfy 0 <= row_lo <= row_hi <= n");
  const bool filter = row_lo > 0 || row_hi < n;
  if (n < 1 || m < 1) return fail(ctx, BGMF_ERR_ARG, "n and m must be >= 1");
  if (I < 1 || I > n) return fail(ctx, BGMF_ERR_ARG, "grid_i must be in [1, n]");
  if (J < 1 || J > m) return fail(ctx, BGMF_ERR_ARG, "grid_j must be in [1, m]");
  if (nnz < 0 || nnz >= (int64_t)0xFFFFFFFFll)
    return fail(ctx, BGMF_ERR_ARG, "nnz must be in [0, 2^32-1)");
  if ((int64_t)I * J > 65535) return fail(ctx, BGMF_ERR_ARG, "grid_i*grid_j must be <= 65535");
  if (nnz > 0 && (!rows || !cols || !vals)) return fail(ctx, BGMF_ERR_ARG, "NULL input");

  const int64_t rbase = n / I, rextra = n % I, cbase = m / J, cextra = m % J;
  const int rbits = bits_for((uint64_t)(rbase + (rextra ? 1 : 0)) - 1);
  const int cbits = bits_for((uint64_t)(cbase + (cextra ? 1 : 0)) - 1);
  const int bbits = bits_for((uint64_t)I * J - 1);
  if (rbits + cbits + bbits > 64) return fail(ctx, BGMF_ERR_ARG, "grid too large for 64-bit keys");
  if (rbits > 31 || cbits > 31) return fail(ctx, BGMF_ERR_ARG, "block slab wider than 2^31");

  // release any previous partition (and its order index)
  order_release(ctx);
  free_dev(ctx->d_lrow, ctx->stream); free_dev(ctx->d_lcol, ctx->stream); free_dev(ctx->d_val, ctx->stream);
  free_dev(ctx->d_val64, ctx->stream); free_dev(ctx->d_order, ctx->stream);
  ctx->partitioned = false;

  cudaStream_t s = ctx->stream;
  ctx->n = n; ctx->m = m; ctx->I = I; ctx->J = J; ctx->nnz = nnz;
  ctx->rbits = rbits; ctx->cbits = cbits;
  ctx->row_bounds.assign(I + 1, 0);
  ctx->col_bounds.assign(J + 1, 0);
  for (int p = 0; p < I; ++p) ctx->row_bounds[p + 1] = ctx->row_bounds[p] + rbase + (p < rextra);
  for (int p = 0; p < J; ++p) ctx->col_bounds[p + 1] = ctx->col_bounds[p] + cbase + (p < cextra);
  const int nb = I * J;
  ctx->h_offsets.assign(nb + 1, 0);

  const size_t N = (size_t)(nnz > 0 ? nnz : 1);
  int64_t *d_rows = nullptr, *d_cols = nullptr, *d_off = nullptr;
  double* d_vin = nullptr;
  uint64_t *ka = nullptr, *kb = nullptr;
  uint32_t *ia = nullptr, *ib = nullptr, *hist = nullptr, *tot = nullptr;
  unsigned long long* d_bad = nullptr;
  int rc = BGMF_OK;
  auto cleanup = [&]() {
    free_dev(d_rows, ctx->stream); free_dev(d_cols, ctx->stream); free_dev(d_vin, ctx->stream); free_dev(ka, ctx->stream); free_dev(kb, ctx->stream);
    free_dev(ia, ctx->stream); free_dev(ib, ctx->stream); free_dev(hist, ctx->stream); free_dev(tot, ctx->stream); free_dev(d_bad, ctx->stream); free_dev(d_off, ctx->stream);
  };
#define PCK(call)                                           \
  do {                                                      \
    cudaError_t _e = (call);                                \
    if (_e != cudaSuccess) { rc = cuda_fail(ctx, _e, #call); cleanup(); return rc; } \
  } while (0)

  prof_mark(ctx, nullptr);
  // host input with 32-bit dimensions: narrowed staged upload (int32 indices,
  // fp32 values unless exact mode needs the fp64 ones)
  const bool narrow = !dev_in && n <= INT32_MAX && m <= INT32_MAX;
  if (filter && !narrow)
    return fail(ctx, BGMF_ERR_ARG, "row ranges need host input with 32-bit dimensions");
  const bool v32 = narrow && !ctx->exact;
  if (dev_in) {
    d_rows = const_cast<int64_t*>(rows);
    d_cols = const_cast<int64_t*>(cols);
    d_vin = const_cast<double*>(vals);
  } else {
    PCK(dmalloc(&d_rows, N * (narrow ? 4 : 8), ctx->stream));
    PCK(dmalloc(&d_cols, N * (narrow ? 4 : 8), ctx->stream));
    PCK(dmalloc(&d_vin, N * (v32 ? 4 : 8), ctx->stream));
  }
  PCK(dmalloc(&ka, N * 8, ctx->stream));
  PCK(dmalloc(&ia, N * 4, ctx->stream));
  PCK(dmalloc(&d_bad, 8, ctx->stream));
  PCK(dmalloc(&d_off, (nb + 1) * 8, ctx->stream));
  int64_t host_bad = -1;
  if (nnz > 0 && narrow) {
    int urc = BGMF_OK;
    int64_t kept = nnz;
    host_bad = staged_upload(ctx, rows, cols, vals, nnz, n, m,
                             reinterpret_cast<int32_t*>(d_rows),
                             reinterpret_cast<int32_t*>(d_cols), d_vin, !v32, &urc, row_lo,
                             row_hi, &kept);
    if (urc) { cleanup(); return urc; }
    if (host_bad < 0) nnz = kept;  // the partition holds only the kept rows
    ctx->nnz = nnz;
  } else if (nnz > 0 && !dev_in) {
    PCK(cudaMemcpyAsync(d_rows, rows, nnz * 8, cudaMemcpyHostToDevice, s));
    PCK(cudaMemcpyAsync(d_cols, cols, nnz * 8, cudaMemcpyHostToDevice, s));
    PCK(cudaMemcpyAsync(d_vin, vals, nnz * 8, cudaMemcpyHostToDevice, s));
  }
  prof_mark(ctx, "partition: alloc + upload");
  PCK(cudaMemsetAsync(d_bad, 0xFF, 8, s));
  const int grid = ctx->num_sms * 8;
  // source index in the key's spare low bits, fp32 value as the payload
  const int ibits = nnz > 1 ? bits_for((uint64_t)nnz - 1) : 0;
  const bool embed = v32 && nnz > 1 && rbits + cbits + bbits + ibits <= 64;
  const float* v32in = embed ? reinterpret_cast<const float*>(d_vin) : nullptr;
  if (nnz > 0 && host_bad < 0) {
    if (narrow)
      make_keys<int32_t><<<grid, 256, 0, s>>>(reinterpret_cast<const int32_t*>(d_rows),
                                              reinterpret_cast<const int32_t*>(d_cols), nnz, n,
                                              m, rbase, rextra, cbase, cextra, J, rbits, cbits,
                                              embed ? ibits : 0, v32in, ka, ia, d_bad);
    else
      make_keys<int64_t><<<grid, 256, 0, s>>>(d_rows, d_cols, nnz, n, m, rbase, rextra, cbase,
                                              cextra, J, rbits, cbits, 0, nullptr, ka, ia,
                                              d_bad);
  }
  PCK(cudaGetLastError());
  unsigned long long hbad = 0;
  PCK(cudaMemcpyAsync(&hbad, d_bad, 8, cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  if (host_bad >= 0) hbad = (unsigned long long)host_bad;
  if (hbad != ~0ull) {
    int64_t br = 0, bc = 0;
    if (dev_in) {
      cudaMemcpy(&br, d_rows + hbad, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&bc, d_cols + hbad, 8, cudaMemcpyDeviceToHost);
    } else {
      br = rows[hbad];
      bc = cols[hbad];
    }
    char buf[160];
    snprintf(buf, sizeof buf, "entry %lld: index (%lld, %lld) outside %lldx%lld matrix",
             (long long)hbad, (long long)br, (long long)bc, (long long)n, (long long)m);
    cleanup();
    return fail(ctx, BGMF_ERR_DATA, buf);
  }
  free_dev(d_rows, ctx->stream);
  free_dev(d_cols, ctx->stream);
  if (embed) free_dev(d_vin, ctx->stream);
  prof_mark(ctx, "partition: keys + check");

  // LSD passes: 9-bit digits (512 buckets) when that saves a pass over 8-bit
  // ones (C4: 34 key bits -> 4 passes instead of 5)
  const int total_bits = rbits + cbits + bbits;
  const bool wide = (total_bits + 8) / 9 < (total_bits + 7) / 8;
  const int dbits = wide ? 9 : 8, RD = 1 << dbits;
  const int passes = (total_bits + dbits - 1) / dbits;
  const size_t NK = (size_t)(nnz > 0 ? nnz : 1);  // kept entries
  const int64_t ntiles = (nnz + RS_TILE - 1) / RS_TILE;
  if (passes > 0 && nnz > 1) {
    PCK(dmalloc(&kb, NK * 8, ctx->stream));
    PCK(dmalloc(&ib, NK * 4, ctx->stream));
    PCK(dmalloc(&hist, (size_t)RD * ntiles * 4, ctx->stream));
    PCK(dmalloc(&tot, RD * 4, ctx->stream));
    // > 48 KB of dynamic shared memory
    PCK(cudaFuncSetAttribute(&radix_scatter<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)scatter_smem<512>()));
    PCK(cudaFuncSetAttribute(&radix_scatter<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)scatter_smem<256>()));
    for (int p = 0; p < passes; ++p) {
      const int shift = (embed ? ibits : 0) + dbits * p;
      if (wide) {
        radix_hist<512><<<(unsigned)ntiles, RS_THREADS, 0, s>>>(ka, nnz, shift, ntiles, hist);
        radix_scan_tiles<<<512, 1024, 0, s>>>(hist, ntiles, tot);
        radix_scatter<512><<<(unsigned)ntiles, RS_THREADS, scatter_smem<512>(), s>>>(
            ka, ia, kb, ib, nnz, shift, hist, ntiles, tot);
      } else {
        radix_hist<256><<<(unsigned)ntiles, RS_THREADS, 0, s>>>(ka, nnz, shift, ntiles, hist);
        radix_scan_tiles<<<256, 1024, 0, s>>>(hist, ntiles, tot);
        radix_scatter<256><<<(unsigned)ntiles, RS_THREADS, scatter_smem<256>(), s>>>(
            ka, ia, kb, ib, nnz, shift, hist, ntiles, tot);
      }
      PCK(cudaGetLastError());
      uint64_t* tk = ka; ka = kb; kb = tk;
      uint32_t* ti = ia; ia = ib; ib = ti;
    }
    free_dev(kb, ctx->stream); free_dev(ib, ctx->stream); free_dev(hist, ctx->stream); free_dev(tot, ctx->stream);
  }
  prof_mark(ctx, "partition: radix sort");

  PCK(dmalloc(&ctx->d_lrow, NK * 4, ctx->stream));
  PCK(dmalloc(&ctx->d_lcol, NK * 4, ctx->stream));
  PCK(dmalloc(&ctx->d_val, NK * 4, ctx->stream));
  PCK(dmalloc(&ctx->d_order, NK * 4, ctx->stream));
  if (ctx->exact) PCK(dmalloc(&ctx->d_val64, NK * 8, ctx->stream));
  if (nnz > 0 && embed) {
    decode_embedded<<<grid, 256, 0, s>>>(ka, ia, nnz, ibits, cbits, (1ull << rbits) - 1,
                                         (1ull << cbits) - 1, ctx->d_lrow, ctx->d_lcol,
                                         ctx->d_val, ctx->d_order);
  } else if (nnz > 0) {
    if (v32)
      decode<float><<<grid, 256, 0, s>>>(ka, ia, reinterpret_cast<const float*>(d_vin), nnz,
                                         cbits, (1ull << rbits) - 1, (1ull << cbits) - 1,
                                         ctx->d_lrow, ctx->d_lcol, ctx->d_val, ctx->d_val64,
                                         ctx->d_order);
    else
    decode<double><<<grid, 256, 0, s>>>(ka, ia, d_vin, nnz, cbits, (1ull << rbits) - 1,
                                (1ull << cbits) - 1, ctx->d_lrow, ctx->d_lcol, ctx->d_val,
                                ctx->d_val64, ctx->d_order);
  }
  block_offsets<<<(nb + 1 + 255) / 256, 256, 0, s>>>(ka, nnz, nb,
                                                    rbits + cbits + (embed ? ibits : 0), d_off);
  PCK(cudaGetLastError());
  PCK(cudaMemcpyAsync(ctx->h_offsets.data(), d_off, (nb + 1) * 8, cudaMemcpyDeviceToHost, s));
  // ratings-per-user skew (ctx->row_cv), reusing the sort's scratch (ia: nnz
  // x 4 B >= n x 4 B is not guaranteed, so its own n counters)
  ctx->row_cv = 0.0;
  if (nnz > 0 && ctx->u_ring < 0) {
    unsigned* cnt = nullptr;
    unsigned long long* sq = nullptr;
    PCK(dmalloc(&cnt, (size_t)n * 4, s));
    PCK(dmalloc(&sq, 8, s));
    PCK(cudaMemsetAsync(cnt, 0, (size_t)n * 4, s));
    PCK(cudaMemsetAsync(sq, 0, 8, s));
    row_hist<<<grid, 256, 0, s>>>(ctx->d_lrow, d_off, nb, J, rbase, rextra, nnz, cnt);
    sum_squares<<<grid, 256, 0, s>>>(cnt, n, sq);
    unsigned long long h_sq = 0;
    cudaError_t e = cudaMemcpyAsync(&h_sq, sq, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    free_dev(cnt, s);
    free_dev(sq, s);
    PCK(e);
    // over the kept rows (a ring rank's shard; the others count 0 and add
    // nothing to the sum of squares)
    const double rows_kept = (double)std::max<int64_t>(1, row_hi - row_lo);
    const double mean = (double)nnz / rows_kept;
    const double var = (double)h_sq / rows_kept - mean * mean;
    ctx->row_cv = var > 0.0 ? std::sqrt(var) / mean : 0.0;
  }
  PCK(cudaStreamSynchronize(s));
  prof_mark(ctx, "partition: decode + offsets");
  cleanup();
  prof_mark(ctx, "partition: free temporaries");
#undef PCK
  ctx->partitioned = true;
  return BGMF_OK;
}


// ---- out-of-core partition -------------------------------------------
// A dataset whose partition does not fit the device (the paper's motivating
// case: BGMF needs only the blocks being computed) enters
// here instead of partition_device:
//   1. host pass (OpenMP over input ranges): range checks, per-block counts;
//   2. row blocks grouped into chunks whose partition temporaries
//      (kChunkBytes per rating) fit `budget`;
//   3. host pass: each entry narrowed (int32 row/col, fp32 value) into its
//      chunk's bucket with its input index, input order kept per chunk;
//   4. per chunk: upload, device keys + radix sort + decode (the in-core
//      kernels, so the block order and in-block order are the reference's
//      lexsort order, bit for bit), packed records, then D2H of every block
//      straight into the pinned diagonal layout of the streaming path.
// Peak device memory: one chunk's temporaries, then the slot ring.
namespace {
constexpr int64_t kChunkBytes = 64;  // device bytes per rating while a chunk is partitioned
}

int partition_ooc(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols, const double* vals,
                  int64_t nnz, int64_t n, int64_t m, int I, int J, int64_t budget,
                  int64_t slot_ratings, int nslots, int64_t row_lo, int64_t row_hi) {
  if (row_hi < 0) row_hi = n;
  if (row_lo < 0 || row_lo > row_hi || row_hi > n)
    return fail(ctx, BGMF_ERR_ARG, "row range must satisfy 0 <= row_lo <= row_hi <= n");
  if (n < 1 || m < 1 || n > INT32_MAX || m > INT32_MAX)
    return fail(ctx, BGMF_ERR_ARG, "n and m must be in [1, 2^31)");
  if (I < 1 || I > n) return fail(ctx, BGMF_ERR_ARG, "grid_i must be in [1, n]");
  if (J < 1 || J > m) return fail(ctx, BGMF_ERR_ARG, "grid_j must be in [1, m]");
  if ((int64_t)I * J > 65535) return fail(ctx, BGMF_ERR_ARG, "grid_i*grid_j must be <= 65535");
  if (nnz < 0 || nnz >= (int64_t)0xFFFFFFFFll)
    return fail(ctx, BGMF_ERR_ARG, "nnz must be in [0, 2^32-1)");
  if (nnz > 0 && (!rows || !cols || !vals)) return fail(ctx, BGMF_ERR_ARG, "NULL input");
  if (ctx->exact) return fail(ctx, BGMF_ERR_STATE, "out-of-core partitioning is fast-mode only");
  if (nslots < 2 || nslots > 8) return fail(ctx, BGMF_ERR_ARG, "nslots must be in [2, 8]");
  if (ctx->streaming) stream_free(ctx);
  order_release(ctx);
  free_dev(ctx->d_lrow, ctx->stream); free_dev(ctx->d_lcol, ctx->stream);
  free_dev(ctx->d_val, ctx->stream); free_dev(ctx->d_val64, ctx->stream);
  free_dev(ctx->d_order, ctx->stream);
  ctx->partitioned = false;
  prof_mark(ctx, "ooc: release previous state");

  const int64_t rbase = n / I, rextra = n % I, cbase = m / J, cextra = m % J;
  const int rbits = bits_for((uint64_t)(rbase + (rextra ? 1 : 0)) - 1);
  const int cbits = bits_for((uint64_t)(cbase + (cextra ? 1 : 0)) - 1);
  const int bbits = bits_for((uint64_t)I * J - 1);
  if (rbits > 31 || cbits > 31) return fail(ctx, BGMF_ERR_ARG, "block slab wider than 2^31");
  ctx->n = n; ctx->m = m; ctx->I = I; ctx->J = J; ctx->nnz = nnz;
  ctx->rbits = rbits; ctx->cbits = cbits;
  ctx->row_bounds.assign(I + 1, 0);
  ctx->col_bounds.assign(J + 1, 0);
  for (int p = 0; p < I; ++p) ctx->row_bounds[p + 1] = ctx->row_bounds[p] + rbase + (p < rextra);
  for (int p = 0; p < J; ++p) ctx->col_bounds[p + 1] = ctx->col_bounds[p] + cbase + (p < cextra);
  const int nb = I * J;
  // closed-form slab index in 32-bit arithmetic (n, m < 2^31)
  auto slab = [](int64_t x, int64_t base, int64_t extra) -> int64_t {
    const uint32_t ux = (uint32_t)x, b = (uint32_t)base, e = (uint32_t)extra;
    const uint32_t big = e * (b + 1u);
    return ux < big ? ux / (b + 1u) : e + (ux - big) / b;
  };

  // 1. range checks + per-block counts
  int nth = 1;
#pragma omp parallel
  {
#pragma omp single
    nth = omp_get_num_threads();
  }
  std::vector<int64_t> tcount((size_t)nth * nb, 0);
  std::vector<int64_t> tbad(nth, -1);
  std::vector<char> tnonbyte(nth, 0);  // a value that is not an integer in 0..255
#pragma omp parallel num_threads(nth)
  {
    const int t = omp_get_thread_num();
    const int64_t lo = nnz * t / nth, hi = nnz * (t + 1) / nth;
    int64_t* cnt = tcount.data() + (size_t)t * nb;
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t r = rows[i], c = cols[i];
      if (r < 0 || r >= n || c < 0 || c >= m) { tbad[t] = i; break; }
      if (r < row_lo || r >= row_hi) continue;  // another rank's rows (checked, not kept)
      ++cnt[slab(r, rbase, rextra) * J + slab(c, cbase, cextra)];
      const float x = (float)vals[i];
      if (!(x >= 0.f && x <= 255.f && x == rintf(x))) tnonbyte[t] = 1;
    }
  }
  for (int t = 0; t < nth; ++t)
    if (tbad[t] >= 0) {
      const int64_t i = tbad[t];
      char buf[160];
      snprintf(buf, sizeof buf, "entry %lld: index (%lld, %lld) outside %lldx%lld matrix",
               (long long)i, (long long)rows[i], (long long)cols[i], (long long)n, (long long)m);
      return fail(ctx, BGMF_ERR_DATA, buf);
    }
  std::vector<int64_t> bcount(nb, 0);
  for (int t = 0; t < nth; ++t)
    for (int b = 0; b < nb; ++b) bcount[b] += tcount[(size_t)t * nb + b];
  ctx->h_offsets.assign(nb + 1, 0);
  for (int b = 0; b < nb; ++b) ctx->h_offsets[b + 1] = ctx->h_offsets[b] + bcount[b];
  const int64_t kept = ctx->h_offsets[nb];  // entries of rows [row_lo, row_hi)
  ctx->nnz = kept;
  int64_t max_block = 0;
  for (int b = 0; b < nb; ++b) max_block = std::max(max_block, bcount[b]);
  if (slot_ratings < max_block || slot_ratings < 1)
    return fail(ctx, BGMF_ERR_ARG, "slot smaller than the largest block (" +
                                       std::to_string(max_block) + " ratings)");

  // 2. chunks of whole row blocks
  const int64_t per_chunk = std::max<int64_t>(1, budget / kChunkBytes);
  std::vector<int> chunk_of(I, 0);
  std::vector<int64_t> chunk_cnt;
  std::vector<int> chunk_b0;  // first row block of each chunk
  {
    int64_t acc = 0;
    for (int bi = 0; bi < I; ++bi) {
      int64_t rc = 0;
      for (int bj = 0; bj < J; ++bj) rc += bcount[bi * J + bj];
      if (chunk_cnt.empty() || (acc > 0 && acc + rc > per_chunk)) {
        chunk_cnt.push_back(0);
        chunk_b0.push_back(bi);
        acc = 0;
      }
      acc += rc;
      chunk_cnt.back() += rc;
      chunk_of[bi] = (int)chunk_cnt.size() - 1;
    }
  }
  const int nch = (int)chunk_cnt.size();
  chunk_b0.push_back(I);
  std::vector<int64_t> chunk_base(nch + 1, 0);
  for (int k = 0; k < nch; ++k) chunk_base[k + 1] = chunk_base[k] + chunk_cnt[k];
  prof_mark(ctx, "ooc: host count pass");

  // the pinned diagonal layout (stream.cu) is sized now, so a side thread
  // maps, faults in and registers it (0.6-1.8 s for C5's 18 GB, mostly the
  // kernel's page pinning) while the bucket pass below runs; 1-byte value
  // codes (5 B records) when every kept value is an integer in 0..255
  ctx->packed = rbits + cbits <= 32;
  ctx->val8 = ctx->packed && !ctx->no_val8;
  for (int t = 0; t < nth; ++t) ctx->val8 = ctx->val8 && !tnonbyte[t];
  struct LayoutPin {
    std::thread t;
    cudaError_t err = cudaSuccess;
    void* p[4] = {nullptr, nullptr, nullptr, nullptr};
    ~LayoutPin() {
      if (t.joinable()) t.join();
      for (void* q : p) big_pinned_free(q);  // still owned: an error path
    }
  } lay;
  {
    const size_t NL = (size_t)(kept > 0 ? kept : 1);
    const size_t sz[4] = {NL * 4, ctx->packed ? 0 : NL * 4, NL * val_bytes(ctx), NL * 4};
    const int dev = ctx->device;
    lay.t = std::thread([&lay, sz, dev]() {
      cudaSetDevice(dev);
      for (int q = 0; q < 4 && lay.err == cudaSuccess; ++q)
        if (sz[q]) lay.err = big_pinned_alloc(&lay.p[q], sz[q], 4);
    });
  }

  // 3. buckets: narrowed entries + input index, per chunk in input order
  // buckets in THP-backed pageable memory (hostio.cu big_host_alloc): no
  // zero-fill (faulted in by the bucket pass's threads), and no pinning --
  // they cross PCIe once, through the pinned staging pair (staged_h2d).
  // Pinned buckets cost 1.3 s to register and ~2 s to unregister on C5's
  // 32 GB, the latter holding the driver lock (a std::vector's zero-fill and
  // plain pageable uploads cost 13 s and 3.5 s before that).
  const size_t N = (size_t)(kept > 0 ? kept : 1);
  struct Bucket {
    int32_t* r = nullptr;
    int32_t* c = nullptr;
    float* v = nullptr;
    uint32_t* x = nullptr;
    ~Bucket() { big_host_free(r); big_host_free(c); big_host_free(v); big_host_free(x); }
  } bk;
  bk.r = static_cast<int32_t*>(big_host_alloc(N * 4));
  bk.c = static_cast<int32_t*>(big_host_alloc(N * 4));
  bk.v = static_cast<float*>(big_host_alloc(N * 4));
  bk.x = static_cast<uint32_t*>(big_host_alloc(N * 4));
  if (!bk.r || !bk.c || !bk.v || !bk.x)
    return fail(ctx, BGMF_ERR_NOMEM, "out of host memory for the partition buckets");
  prof_mark(ctx, "ooc: bucket memory");
  int32_t* const br = bk.r;
  int32_t* const bc = bk.c;
  float* const bv = bk.v;
  uint32_t* const bx = bk.x;
  std::vector<int64_t> toff((size_t)nth * nch, 0);
  for (int k = 0; k < nch; ++k) {
    int64_t o = chunk_base[k];
    for (int t = 0; t < nth; ++t) {
      toff[(size_t)t * nch + k] = o;
      for (int bi = chunk_b0[k]; bi < chunk_b0[k + 1]; ++bi)
        for (int bj = 0; bj < J; ++bj) o += tcount[(size_t)t * nb + bi * J + bj];
    }
  }
#pragma omp parallel num_threads(nth)
  {
    // per-thread write-combining: 256 entries per chunk gathered in a small
    // (L2-resident) buffer, then copied out as 1 KB runs -- scattering every
    // entry straight into nch x 4 far-apart streams ran at ~6 GB/s on C5
    constexpr int WC = 256;
    const int t = omp_get_thread_num();
    const int64_t lo = nnz * t / nth, hi = nnz * (t + 1) / nth;
    int64_t* off = toff.data() + (size_t)t * nch;
    std::vector<int32_t> wr((size_t)nch * WC), wc((size_t)nch * WC);
    std::vector<float> wv((size_t)nch * WC);
    std::vector<uint32_t> wx((size_t)nch * WC);
    std::vector<int> fill(nch, 0);
    auto flush = [&](int k) {
      const int f = fill[k];
      const int64_t p = off[k];
      const size_t o = (size_t)k * WC;
      memcpy(br + p, wr.data() + o, (size_t)f * 4);
      memcpy(bc + p, wc.data() + o, (size_t)f * 4);
      memcpy(bv + p, wv.data() + o, (size_t)f * 4);
      memcpy(bx + p, wx.data() + o, (size_t)f * 4);
      off[k] += f;
      fill[k] = 0;
    };
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t r = rows[i];
      if (r < row_lo || r >= row_hi) continue;
      const int k = chunk_of[slab(r, rbase, rextra)];
      const size_t j = (size_t)k * WC + fill[k]++;
      wr[j] = (int32_t)r;
      wc[j] = (int32_t)cols[i];
      wv[j] = (float)vals[i];
      wx[j] = (uint32_t)i;
      if (fill[k] == WC) flush(k);
    }
    for (int k = 0; k < nch; ++k) flush(k);
  }
  prof_mark(ctx, "ooc: host bucket pass");

  // the layout's block positions (diagonal order)
  std::vector<int> order;
  order.reserve(nb);
  if (I == J) {
    for (int d = 0; d < I; ++d)
      for (int j = 0; j < J; ++j) order.push_back(((j + d) % I) * J + j);
  } else {
    for (int b = 0; b < nb; ++b) order.push_back(b);
  }
  ctx->h_pos.assign(nb, 0);
  {
    int64_t pos = 0;
    for (int b : order) { ctx->h_pos[b] = pos; pos += bcount[b]; }
  }
  lay.t.join();
  if (lay.err != cudaSuccess) return cuda_fail(ctx, lay.err, "pinned layout");
  ctx->h_lrow = static_cast<int32_t*>(lay.p[0]);
  ctx->h_lcol = static_cast<int32_t*>(lay.p[1]);
  ctx->h_val = static_cast<float*>(lay.p[2]);
  ctx->h_order = static_cast<uint32_t*>(lay.p[3]);
  for (void*& q : lay.p) q = nullptr;  // the context owns them now
  prof_mark(ctx, "ooc: pinned layout (wait)");

  // 4. chunk by chunk on the device
  cudaStream_t s = ctx->stream;
  const int total_bits = rbits + cbits + bbits;
  int64_t max_chunk = 0;
  for (int k = 0; k < nch; ++k) max_chunk = std::max(max_chunk, chunk_cnt[k]);
  const size_t C = (size_t)(max_chunk > 0 ? max_chunk : 1);
  int32_t *d_r = nullptr, *d_c = nullptr, *lr = nullptr, *lc = nullptr, *rec = nullptr;
  float *d_v = nullptr, *vv = nullptr;
  uint32_t *d_x = nullptr, *ia = nullptr, *ord = nullptr, *gord = nullptr;
  uint8_t* codes = nullptr;
  uint64_t* ka = nullptr;
  unsigned long long* d_bad = nullptr;
  int rc = BGMF_OK;
  std::thread releaser;
  auto cleanup = [&]() {
    if (releaser.joinable()) releaser.join();
    free_dev(d_r, s); free_dev(d_c, s); free_dev(d_v, s); free_dev(d_x, s); free_dev(ka, s);
    free_dev(ia, s); free_dev(lr, s); free_dev(lc, s); free_dev(vv, s); free_dev(ord, s);
    free_dev(rec, s); free_dev(gord, s); free_dev(d_bad, s); free_dev(codes, s);
  };
#define OCK(call)                                                                    \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess) { rc = cuda_fail(ctx, _e, #call); cleanup(); return rc; } \
  } while (0)
  OCK(dmalloc(&d_r, C * 4, s)); OCK(dmalloc(&d_c, C * 4, s)); OCK(dmalloc(&d_v, C * 4, s));
  OCK(dmalloc(&d_x, C * 4, s));
  OCK(dmalloc(&lr, C * 4, s)); OCK(dmalloc(&lc, C * 4, s)); OCK(dmalloc(&vv, C * 4, s));
  OCK(dmalloc(&ord, C * 4, s)); OCK(dmalloc(&gord, C * 4, s)); OCK(dmalloc(&d_bad, 8, s));
  if (ctx->val8) OCK(dmalloc(&codes, C, s));
  if (ctx->packed) OCK(dmalloc(&rec, C * 4, s));
  const int grid = ctx->num_sms * 8;
  for (int k = 0; k < nch; ++k) {
    const int64_t cnt = chunk_cnt[k], base = chunk_base[k];
    if (cnt == 0) continue;
    if (releaser.joinable()) releaser.join();
    rc = staged_h2d(ctx, d_r, br + base, cnt * 4);
    if (!rc) rc = staged_h2d(ctx, d_c, bc + base, cnt * 4);
    if (!rc) rc = staged_h2d(ctx, d_v, bv + base, cnt * 4);
    if (!rc) rc = staged_h2d(ctx, d_x, bx + base, cnt * 4);
    if (rc) { cleanup(); return rc; }
    // this chunk's bucket slices have crossed: a helper thread returns their
    // pages while this thread waits on the chunk's sort and layout copies
    releaser = std::thread([=]() {
      big_host_release(br + base, cnt * 4);
      big_host_release(bc + base, cnt * 4);
      big_host_release(bv + base, cnt * 4);
      big_host_release(bx + base, cnt * 4);
    });
    OCK(cudaMemsetAsync(d_bad, 0xFF, 8, s));
    OCK(dmalloc(&ka, (size_t)cnt * 8, s));  // the sort swaps buffers: per chunk
    OCK(dmalloc(&ia, (size_t)cnt * 4, s));
    // the chunk index rides in the key's spare low bits when they suffice
    // (then the fp32 value is the payload); else the payload is the index
    const int ib = cnt > 1 ? bits_for((uint64_t)cnt - 1) : 0;
    const bool embed = total_bits + ib <= 64;
    const int ibits = embed ? ib : 0;
    make_keys<int32_t><<<grid, 256, 0, s>>>(d_r, d_c, cnt, n, m, rbase, rextra, cbase, cextra,
                                            J, rbits, cbits, ibits, embed ? d_v : nullptr, ka,
                                            ia, d_bad);
    OCK(cudaGetLastError());
    // stable sort on the (block, row, col) bits above the embedded index
    uint64_t* kk = ka;
    uint32_t* ii = ia;
    rc = sort_pairs_device(ctx, &kk, &ii, cnt, total_bits, ibits);
    if (rc) { cleanup(); return rc; }
    ka = kk;
    ia = ii;
    if (embed)
      decode_embedded<<<grid, 256, 0, s>>>(ka, ia, cnt, ibits, cbits, (1ull << rbits) - 1,
                                           (1ull << cbits) - 1, lr, lc, vv, ord);
    else
      decode<float><<<grid, 256, 0, s>>>(ka, ia, d_v, cnt, cbits, (1ull << rbits) - 1,
                                         (1ull << cbits) - 1, lr, lc, vv, nullptr, ord);
    pack_and_order<<<grid, 256, 0, s>>>(lr, lc, ord, d_x, cnt, cbits, ctx->packed ? rec : nullptr,
                                        gord);
    if (ctx->val8) values_to_codes<<<grid, 256, 0, s>>>(vv, cnt, codes);
    OCK(cudaGetLastError());
    free_dev(ka, s);
    free_dev(ia, s);
    // blocks of this chunk, flat order = their order in the sorted chunk
    int64_t lo = 0;
    for (int b = chunk_b0[k] * J; b < chunk_b0[k + 1] * J; ++b) {
      const int64_t bc_ = bcount[b], dst = ctx->h_pos[b];
      if (bc_ > 0) {
        OCK(cudaMemcpyAsync(ctx->h_lrow + dst, (ctx->packed ? rec : lr) + lo, bc_ * 4,
                            cudaMemcpyDeviceToHost, s));
        if (!ctx->packed)
          OCK(cudaMemcpyAsync(ctx->h_lcol + dst, lc + lo, bc_ * 4, cudaMemcpyDeviceToHost, s));
        if (ctx->val8)
          OCK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(ctx->h_val) + dst, codes + lo, bc_,
                              cudaMemcpyDeviceToHost, s));
        else
          OCK(cudaMemcpyAsync(ctx->h_val + dst, vv + lo, bc_ * 4, cudaMemcpyDeviceToHost, s));
        OCK(cudaMemcpyAsync(ctx->h_order + dst, gord + lo, bc_ * 4, cudaMemcpyDeviceToHost, s));
      }
      lo += bc_;
    }
    OCK(cudaStreamSynchronize(s));  // the chunk buffers are reused by the next chunk
  }
  cleanup();
#undef OCK
  prof_mark(ctx, "ooc: device chunks");
  ctx->partitioned = true;
  ctx->streaming = true;
  rc = stream_slots(ctx, slot_ratings, nslots);
  if (rc) return rc;
  prof_mark(ctx, "ooc: stream slots");
  ctx->ooc_chunks = nch;
  return BGMF_OK;
}

}  // namespace bgmf
