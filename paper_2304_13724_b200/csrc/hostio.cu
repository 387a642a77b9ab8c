// hostio.cu -- host <-> device movement of the dataset and the model.
//
// The reference keeps everything in host numpy arrays (ratings int64/int64/
// fp64, factors fp64: core.py:12-108, 139-176).  The e2e path therefore has
// to move 24 B per rating in and 8k B per factor row out.  Measured on the
// B200 hosts (profiles/r01_host_probe.txt, scripts/host_probe.cu):
//   * pageable cudaMemcpy runs at ~11 GB/s (driver's single-threaded bounce);
//   * pinned DMA runs at ~55 GB/s, but pinning costs ~1.1 GB/s
//     (cudaHostRegister / cudaMallocHost), so pinning per call never pays;
//   * 16 host threads narrow int64 -> int32 at ~100 GB/s (read + write) and
//     fault fresh pages at 33-70 GB/s.
// So both directions go through a small process-wide pool of pinned staging
// buffers, allocated once (like a caching host allocator) and reused by every
// context: OpenMP threads convert between the reference's host types and the
// device types in the staging buffer while the DMA engine moves the other one.

#include <emmintrin.h>
#include <omp.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

constexpr size_t kStageBytes = size_t(16) << 20;  // per buffer

struct StagePool {
  std::mutex mu;
  char* buf[2] = {nullptr, nullptr};
  int device = -1;
};

StagePool& pool() {
  static StagePool p;
  return p;
}

// Locks the pool and makes sure both pinned buffers exist.
class Stage {
 public:
  explicit Stage(bgmf_ctx* c) : lk_(pool().mu) {
    StagePool& p = pool();
    for (int b = 0; b < 2 && !err_; ++b) {
      if (!p.buf[b]) err_ = cudaMallocHost(&p.buf[b], kStageBytes);
      if (!err_) err_ = cudaEventCreateWithFlags(&done_[b], cudaEventDisableTiming);
    }
    (void)c;
  }
  ~Stage() {
    for (int b = 0; b < 2; ++b)
      if (done_[b]) cudaEventDestroy(done_[b]);
  }
  cudaError_t error() const { return err_; }
  char* buf(int b) const { return pool().buf[b]; }
  cudaEvent_t done(int b) const { return done_[b]; }

 private:
  std::unique_lock<std::mutex> lk_;
  cudaError_t err_ = cudaSuccess;
  cudaEvent_t done_[2] = {nullptr, nullptr};
};

}  // namespace

// Small pinned buffers (the per-context step scratch: work table, per-block
// SSE, divergence flag) come from a process-wide cache and go back to it on
// release: cudaFreeHost measured 0.8 ms typically but 300-520 ms at times in
// a context teardown (profiles/r01_e2e_phases.txt), inside the e2e call.
// Size classes are powers of two >= 4 KiB; buffers above 64 MiB and a cache
// above 256 MiB are freed for real.
namespace {
constexpr size_t kPinCacheMax = size_t(64) << 20, kPinCacheTotal = size_t(256) << 20;
struct PinCache {
  std::mutex mu;
  std::multimap<size_t, void*> free_;
  std::unordered_map<void*, size_t> size_;
  size_t cached = 0;
};
PinCache& pin_cache() {
  static PinCache* p = new PinCache;  // never destroyed: outlives static teardown
  return *p;
}
size_t pin_class(size_t bytes) {
  size_t c = 4096;
  while (c < bytes) c <<= 1;
  return c;
}
}  // namespace

cudaError_t pinned_alloc(void** p, size_t bytes) {
  const size_t cls = pin_class(bytes ? bytes : 1);
  PinCache& pc = pin_cache();
  {
    std::lock_guard<std::mutex> lk(pc.mu);
    auto it = pc.free_.find(cls);
    if (it != pc.free_.end()) {
      *p = it->second;
      pc.free_.erase(it);
      pc.cached -= cls;
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMallocHost(p, cls);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(pc.mu);
    pc.size_[*p] = cls;
  }
  return e;
}

void pinned_free(void* p) {
  if (!p) return;
  PinCache& pc = pin_cache();
  {
    std::lock_guard<std::mutex> lk(pc.mu);
    auto it = pc.size_.find(p);
    if (it != pc.size_.end() && it->second <= kPinCacheMax &&
        pc.cached + it->second <= kPinCacheTotal) {
      pc.free_.emplace(it->second, p);
      pc.cached += it->second;
      return;
    }
    if (it != pc.size_.end()) pc.size_.erase(it);
  }
  cudaFreeHost(p);
}

// Large pinned host arrays (the out-of-core layout: GBs).  cudaMallocHost
// pins 4 KiB pages one by one (~2.5 GB/s measured for C5's 24 GB,
// profiles/r02_*); instead: anonymous memory advised MADV_HUGEPAGE, faulted
// in by all host threads (one write per 2 MiB page), then cudaHostRegister.
// Released on a detached thread: unpinning GBs costs seconds the caller
// does not need to wait for.
//
// Freed pinned buffers are cached (like a caching host allocator) up to a
// quarter of physical memory: unregistering tens of GB takes the driver lock
// for a few hundred ms, stalling the caller's next CUDA call (C5: the context
// release), and the next out-of-core partition of a similar size reuses the
// registered pages instead of pinning again (0.6-1.8 s for C5's layout).
// bgmf_release_host_cache() gives everything back.
namespace {
struct CachedPin {
  void* p;
  void* base;
  size_t len, span;
};
struct BigPinned {
  std::mutex mu;
  std::unordered_map<void*, std::pair<void*, size_t>> maps;  // user ptr -> (mmap base, len)
  std::unordered_map<void*, size_t> spans;                    // registered bytes
  std::vector<CachedPin> cache;  // registered, unused
  size_t cached = 0;
};
BigPinned& big_pinned() {
  static BigPinned* p = new BigPinned;
  return *p;
}
size_t& pin_span_of(void* p) { return big_pinned().spans[p]; }  // under mu
size_t pin_cache_cap() {
  static const size_t cap = [] {
    const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGE_SIZE);
    return pages > 0 && psz > 0 ? (size_t)pages * (size_t)psz / 4 : (size_t)0;
  }();
  return cap;
}
}  // namespace

cudaError_t big_pinned_alloc(void** out, size_t bytes, int threads) {
  const size_t huge = size_t(2) << 20;
  {  // a cached registered buffer of the same order of size
    const size_t want = (bytes + huge - 1) / huge * huge;
    std::lock_guard<std::mutex> lk(big_pinned().mu);
    auto& c = big_pinned().cache;
    int best = -1;
    for (int i = 0; i < (int)c.size(); ++i)
      if (c[i].span >= want && c[i].span <= 2 * want + huge &&
          (best < 0 || c[i].span < c[best].span))
        best = i;
    if (best >= 0) {
      const CachedPin h = c[best];
      c.erase(c.begin() + best);
      big_pinned().cached -= h.span;
      big_pinned().maps[h.p] = {h.base, h.len};
      pin_span_of(h.p) = h.span;
      *out = h.p;
      return cudaSuccess;
    }
  }
  const size_t len = (bytes + 2 * huge - 1) / huge * huge;
  void* base = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (base == MAP_FAILED) return cudaErrorMemoryAllocation;
  char* p = reinterpret_cast<char*>(((uintptr_t)base + huge - 1) / huge * huge);
  const size_t span = (bytes + huge - 1) / huge * huge;
  madvise(p, span, MADV_HUGEPAGE);
  const int64_t pages = (int64_t)(span / huge);
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : omp_get_max_threads())
  for (int64_t i = 0; i < pages; ++i) p[i * (int64_t)huge] = 0;
  cudaError_t e = cudaHostRegister(p, span, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    munmap(base, len);
    return e;
  }
  {
    std::lock_guard<std::mutex> lk(big_pinned().mu);
    big_pinned().maps[p] = {base, len};
    pin_span_of(p) = span;
  }
  *out = p;
  return cudaSuccess;
}

// Large pageable host buffer: THP-backed anonymous memory, faulted in by the
// writing threads (no zero-fill pass, no pinning).  For data that crosses
// PCIe once (the out-of-core partition's buckets): staged_h2d moves it, so
// neither the registration (~24 GB/s) nor the unregistration -- which holds
// the driver lock for seconds on tens of GB, stalling every CUDA call of the
// process -- is paid.
void* big_host_alloc(size_t bytes) {
  const size_t huge = size_t(2) << 20;
  const size_t len = (bytes + huge - 1) / huge * huge + huge;
  void* base = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (base == MAP_FAILED) return nullptr;
  char* p = reinterpret_cast<char*>(((uintptr_t)base + huge - 1) / huge * huge);
  madvise(p, len - huge, MADV_HUGEPAGE);
  {
    std::lock_guard<std::mutex> lk(big_pinned().mu);
    big_pinned().maps[p] = {base, len};
  }
  return p;
}

void big_host_free(void* p) {
  if (!p) return;
  std::pair<void*, size_t> m{nullptr, 0};
  {
    std::lock_guard<std::mutex> lk(big_pinned().mu);
    auto it = big_pinned().maps.find(p);
    if (it == big_pinned().maps.end()) return;
    m = it->second;
    big_pinned().maps.erase(it);
  }
  std::thread([m]() { munmap(m.first, m.second); }).detach();
}

// Give the physical pages of [p, p + bytes) back (whole 2 MiB pages inside
// the range only): madvise(MADV_DONTNEED) runs under the mm read lock, so
// other threads' faults and CUDA calls proceed -- unlike one munmap of tens
// of GB at the end, which holds the write lock for seconds.
void big_host_release(void* p, size_t bytes) {
  const uintptr_t huge = uintptr_t(2) << 20;
  const uintptr_t a = ((uintptr_t)p + huge - 1) / huge * huge;
  const uintptr_t e = ((uintptr_t)p + bytes) / huge * huge;
  if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_DONTNEED);
}

// Host -> device copy of pageable memory through the process's pinned staging
// pair: host threads copy piece p+1 into one buffer while the DMA engine moves
// piece p out of the other (pageable cudaMemcpy runs at ~11 GB/s; this at the
// pinned PCIe rate when the host copy keeps up).  Stream-ordered on
// ctx->stream; returns when the last piece has left the staging buffers.
int staged_h2d(bgmf_ctx* ctx, void* dst, const void* src, size_t bytes) {
  Stage st(ctx);
  if (st.error()) return cuda_fail(ctx, st.error(), "staging pool");
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  int k = 0;
  for (size_t o = 0; o < bytes; o += kStageBytes, ++k) {
    const int b = k & 1;
    const size_t n = std::min(kStageBytes, bytes - o);
    if (k >= 2) cudaEventSynchronize(st.done(b));
    char* buf = st.buf(b);
    const int64_t parts = 16;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < parts; ++q) {
      const size_t a = n * q / parts, e = n * (q + 1) / parts;
      memcpy(buf + a, s + o + a, e - a);
    }
    cudaError_t e = cudaMemcpyAsync(d + o, buf, n, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaEventRecord(st.done(b), ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "staged H2D");
  }
  for (int b = 0; b < 2 && k > 0; ++b) cudaEventSynchronize(st.done(b));
  return BGMF_OK;
}

// Frees a big_pinned_alloc buffer (asynchronously) or a cudaMallocHost one.
void big_pinned_free(void* p) {
  if (!p) return;
  std::pair<void*, size_t> m{nullptr, 0};
  size_t span = 0;
  {
    std::lock_guard<std::mutex> lk(big_pinned().mu);
    BigPinned& bp = big_pinned();
    auto it = bp.maps.find(p);
    if (it != bp.maps.end()) {
      m = it->second;
      bp.maps.erase(it);
      auto sp = bp.spans.find(p);
      if (sp != bp.spans.end()) {
        span = sp->second;
        bp.spans.erase(sp);
      }
      if (span && bp.cached + span <= pin_cache_cap()) {  // keep it registered
        bp.cache.push_back(CachedPin{p, m.first, m.second, span});
        bp.cached += span;
        return;
      }
    }
  }
  if (!m.first) {
    cudaFreeHost(p);
    return;
  }
  std::thread([p, m]() {
    cudaHostUnregister(p);
    munmap(m.first, m.second);
  }).detach();
}

// Unregister and unmap every cached pinned buffer (bgmf_release_host_cache).
void big_pinned_trim() {
  std::vector<CachedPin> c;
  {
    std::lock_guard<std::mutex> lk(big_pinned().mu);
    c.swap(big_pinned().cache);
    big_pinned().cached = 0;
  }
  for (const CachedPin& h : c) {
    cudaHostUnregister(h.p);
    munmap(h.base, h.len);
  }
}

// Dataset upload for the partitioner (partition.cu): int64 indices narrowed
// to int32 (and range-checked against n x m), fp64 values narrowed to fp32
// unless v64 (exact mode keeps them).  12 (16) instead of 24 B per rating
// cross PCIe.  Only entries with row in [row_lo, row_hi) are kept (compacted
// in input order; every entry is still range-checked) -- a multi-GPU rank
// uploads just its row shard without a host-side gather.  *kept = entries
// uploaded.  Returns the first entry whose index is outside n x m, or -1.
int64_t staged_upload(bgmf_ctx* ctx, const int64_t* rows, const int64_t* cols,
                      const double* vals, int64_t nnz, int64_t n, int64_t m, int32_t* d_r,
                      int32_t* d_c, void* d_v, bool v64, int* rc, int64_t row_lo,
                      int64_t row_hi, int64_t* kept) {
  *rc = BGMF_OK;
  *kept = 0;
  Stage st(ctx);
  if (st.error()) {
    *rc = cuda_fail(ctx, st.error(), "staging pool");
    return -1;
  }
  const bool filter = row_lo > 0 || row_hi < n;
  const size_t vb = v64 ? 8 : 4;
  const int64_t chunk = (int64_t)(kStageBytes / (8 + vb));
  const int nt = omp_get_max_threads();
  std::vector<int64_t> tcount((size_t)nt + 1);
  int64_t first_bad = INT64_MAX, out = 0;
  int k = 0;
  for (int64_t i0 = 0; i0 < nnz; i0 += chunk, ++k) {
    const int b = k & 1;
    const int64_t cnt = nnz - i0 < chunk ? nnz - i0 : chunk;
    if (k >= 2) cudaEventSynchronize(st.done(b));  // the DMA that last read this buffer
    int32_t* sr = reinterpret_cast<int32_t*>(st.buf(b));
    int32_t* sc = sr + chunk;
    char* sv = reinterpret_cast<char*>(sc + chunk);
    int64_t bad = INT64_MAX, nkeep = cnt;
    if (!filter) {
#pragma omp parallel for schedule(static) reduction(min : bad)
      for (int64_t i = 0; i < cnt; ++i) {
        const int64_t r = rows[i0 + i], c = cols[i0 + i];
        if (r < 0 || r >= n || c < 0 || c >= m) bad = i0 + i < bad ? i0 + i : bad;
        sr[i] = (int32_t)r;
        sc[i] = (int32_t)c;
        if (v64) reinterpret_cast<double*>(sv)[i] = vals[i0 + i];
        else reinterpret_cast<float*>(sv)[i] = (float)vals[i0 + i];
      }
    } else {
      // pass 1: per-thread counts (static ranges); pass 2: ordered compaction
      int team = 1;
#pragma omp parallel reduction(min : bad)
      {
        const int t = omp_get_thread_num(), T = omp_get_num_threads();
        const int64_t lo = cnt * t / T, hi = cnt * (t + 1) / T;
        int64_t my = 0;
        for (int64_t i = lo; i < hi; ++i) {
          const int64_t r = rows[i0 + i], c = cols[i0 + i];
          if (r < 0 || r >= n || c < 0 || c >= m) bad = i0 + i < bad ? i0 + i : bad;
          my += r >= row_lo && r < row_hi;
        }
        tcount[t + 1] = my;
#pragma omp barrier
#pragma omp single
        {
          team = T;
          tcount[0] = 0;
          for (int q = 0; q < T; ++q) tcount[q + 1] += tcount[q];
        }
        int64_t o = tcount[t];
        for (int64_t i = lo; i < hi; ++i) {
          const int64_t r = rows[i0 + i];
          if (r < row_lo || r >= row_hi) continue;
          sr[o] = (int32_t)r;
          sc[o] = (int32_t)cols[i0 + i];
          if (v64) reinterpret_cast<double*>(sv)[o] = vals[i0 + i];
          else reinterpret_cast<float*>(sv)[o] = (float)vals[i0 + i];
          ++o;
        }
      }
      nkeep = tcount[team];
    }
    if (bad < first_bad) first_bad = bad;
    if (nkeep > 0) {
      cudaMemcpyAsync(d_r + out, sr, nkeep * 4, cudaMemcpyHostToDevice, ctx->stream);
      cudaMemcpyAsync(d_c + out, sc, nkeep * 4, cudaMemcpyHostToDevice, ctx->stream);
      cudaMemcpyAsync(static_cast<char*>(d_v) + out * vb, sv, nkeep * vb,
                      cudaMemcpyHostToDevice, ctx->stream);
    }
    cudaEventRecord(st.done(b), ctx->stream);
    out += nkeep;
  }
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) *rc = cuda_fail(ctx, e, "staged upload");
  *kept = out;
  return first_bad == INT64_MAX ? -1 : first_bad;
}

// fp32 device rows (stride kp) -> fp64 host rows (stride k), the reference's
// FactorModel layout.  Piece p is DMA'd into one pinned buffer while the host
// threads widen piece p-1 out of the other; 4k B per row cross PCIe.
int download_rows(bgmf_ctx* c, const float* d, double* h, int64_t rows, int k, int kp) {
  if (rows == 0) return BGMF_OK;
  Stage st(c);
  if (st.error()) return cuda_fail(c, st.error(), "staging pool");
  const int64_t chunk = (int64_t)(kStageBytes / ((size_t)kp * 4));
  const int64_t np = (rows + chunk - 1) / chunk;
  auto issue = [&](int64_t p) -> cudaError_t {
    const int64_t r0 = p * chunk, nr = rows - r0 < chunk ? rows - r0 : chunk;
    cudaError_t e = cudaMemcpyAsync(st.buf(p & 1), d + r0 * kp, (size_t)nr * kp * 4,
                                    cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaEventRecord(st.done(p & 1), c->stream);
    return e;
  };
  cudaError_t e = issue(0);
  for (int64_t p = 0; p < np && e == cudaSuccess; ++p) {
    e = cudaEventSynchronize(st.done(p & 1));
    if (e == cudaSuccess && p + 1 < np) e = issue(p + 1);
    if (e != cudaSuccess) break;
    const int64_t r0 = p * chunk, nr = rows - r0 < chunk ? rows - r0 : chunk;
    const float* src = reinterpret_cast<const float*>(st.buf(p & 1));
    double* dst = h + r0 * k;
    if (kp == k && c->nt_download && ((uintptr_t)dst & 15) == 0 && (nr * k) % 2 == 0) {
      // widen with non-temporal 16-byte stores: the fp64 model is written once
      // and not read back here, so no read-for-ownership of its lines
      const int64_t pairs = nr * k / 2;
#pragma omp parallel
      {
#pragma omp for schedule(static)
        for (int64_t i = 0; i < pairs; ++i)
          _mm_stream_pd(dst + 2 * i, _mm_cvtps_pd(_mm_castsi128_ps(
                                          _mm_loadl_epi64(reinterpret_cast<const __m128i*>(src + 2 * i)))));
        _mm_sfence();
      }
    } else if (kp == k) {
      const int64_t tot = nr * k;
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < tot; ++i) dst[i] = (double)src[i];
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t r = 0; r < nr; ++r)
        for (int j = 0; j < k; ++j) dst[r * k + j] = (double)src[r * kp + j];
    }
  }
  if (e != cudaSuccess) {
    cudaStreamSynchronize(c->stream);
    return cuda_fail(c, e, "download_rows");
  }
  return BGMF_OK;
}

// fp64 host rows (stride k) -> fp32 device rows (stride kp, zero padding).
int upload_rows(bgmf_ctx* c, const double* h, float* d, int64_t rows, int k, int kp) {
  if (rows == 0) return BGMF_OK;
  Stage st(c);
  if (st.error()) return cuda_fail(c, st.error(), "staging pool");
  const int64_t chunk = (int64_t)(kStageBytes / ((size_t)kp * 4));
  cudaError_t e = cudaSuccess;
  int q = 0;
  for (int64_t r0 = 0; r0 < rows && e == cudaSuccess; r0 += chunk, ++q) {
    const int b = q & 1;
    const int64_t nr = rows - r0 < chunk ? rows - r0 : chunk;
    if (q >= 2) e = cudaEventSynchronize(st.done(b));
    if (e != cudaSuccess) break;
    float* dst = reinterpret_cast<float*>(st.buf(b));
    const double* src = h + r0 * k;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nr; ++r)
      for (int j = 0; j < kp; ++j) dst[r * kp + j] = j < k ? (float)src[r * k + j] : 0.f;
    e = cudaMemcpyAsync(d + r0 * kp, dst, (size_t)nr * kp * 4, cudaMemcpyHostToDevice,
                        c->stream);
    if (e == cudaSuccess) e = cudaEventRecord(st.done(b), c->stream);
  }
  cudaError_t e2 = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(c, e, "upload_rows");
  return BGMF_OK;
}

}  // namespace bgmf

// Faults in (and zero-fills) a fresh host buffer, one write per 4 KiB page.  The model download widens into freshly allocated
// numpy arrays; first-touch page faults made it run at 25-35 GB/s
// (profiles/r01_host_probe.txt), so the trainer faults the output buffers in
// on a side thread while the epochs run on the GPU.
// The interior 2 MiB-aligned span is advised MADV_HUGEPAGE first (this
// host's THP mode is "madvise"): 512x fewer faults, and fewer TLB misses for
// the widening writes.  Four threads: the epochs' launch thread keeps a core.
extern "C" int bgmf_host_prefault(void* p, int64_t bytes) {
  if (!p || bytes <= 0) return BGMF_OK;
  char* c = static_cast<char*>(p);
  const uintptr_t huge = uintptr_t(2) << 20;
  const uintptr_t a = ((uintptr_t)c + huge - 1) & ~(huge - 1);
  const uintptr_t b = ((uintptr_t)c + (uintptr_t)bytes) & ~(huge - 1);
  if (b > a) madvise(reinterpret_cast<void*>(a), b - a, MADV_HUGEPAGE);
  const int64_t pages = (bytes + 4095) / 4096;
#pragma omp parallel for schedule(static) num_threads(4)
  for (int64_t q = 0; q < pages; ++q) c[q * 4096] = 0;
  return BGMF_OK;
}

