// host_probe.cu -- host-memory / PCIe costs that bound the e2e path (upload of
// the rating triples, download of the fp64 model).  Build + run on the box:
//   nvcc -O2 -Xcompiler -fopenmp -o /tmp/host_probe scripts/host_probe.cu -lgomp && /tmp/host_probe
#include <cuda_runtime.h>
#include <omp.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

int main() {
  const int64_t nnz = 100000000;  // C4
  const size_t B8 = nnz * 8;
  int nt = omp_get_max_threads();
  printf("omp threads %d\n", nt);
  system("cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag");

  // fresh-page first touch: single vs all threads, with / without MADV_HUGEPAGE
  for (int huge = 0; huge < 2; ++huge)
    for (int par = 0; par < 2; ++par) {
      char* p = (char*)aligned_alloc(1 << 21, B8);
      if (huge) madvise(p, B8, MADV_HUGEPAGE);
      double t = now();
      if (par) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < (int64_t)B8; i += 4096) p[i] = 1;
      } else {
        for (int64_t i = 0; i < (int64_t)B8; i += 4096) p[i] = 1;
      }
      t = now() - t;
      printf("first touch 800MB huge=%d threads=%d: %.1f ms (%.1f GB/s)\n", huge, par ? nt : 1,
             t * 1e3, B8 / t / 1e9);
      free(p);
    }

  // source arrays as numpy would hold them (touched)
  int64_t* rows = (int64_t*)aligned_alloc(1 << 21, B8);
  int64_t* cols = (int64_t*)aligned_alloc(1 << 21, B8);
  double* vals = (double*)aligned_alloc(1 << 21, B8);
#pragma omp parallel for
  for (int64_t i = 0; i < nnz; ++i) { rows[i] = i % 480000; cols[i] = i % 17800; vals[i] = 3.0; }

  int32_t* o32 = (int32_t*)aligned_alloc(1 << 21, nnz * 4);
  memset(o32, 0, nnz * 4);
  for (int rep = 0; rep < 2; ++rep) {
    double t = now();
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nnz; ++i) o32[i] = (int32_t)rows[i];
    t = now() - t;
    printf("narrow int64->int32 (touched dst) 800MB read: %.1f ms (%.1f GB/s rd+wr)\n", t * 1e3,
           nnz * 12.0 / t / 1e9);
  }

  void *d_a, *d_b;
  CK(cudaMalloc(&d_a, B8 * 3));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // pageable H2D of the three arrays
  for (int rep = 0; rep < 2; ++rep) {
    double t = now();
    CK(cudaMemcpyAsync(d_a, rows, B8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync((char*)d_a + B8, cols, B8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync((char*)d_a + 2 * B8, vals, B8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    t = now() - t;
    printf("pageable H2D 2.4GB: %.1f ms (%.1f GB/s)\n", t * 1e3, 3 * B8 / t / 1e9);
  }
  // register + pinned DMA + unregister
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now();
    CK(cudaHostRegister(rows, B8, cudaHostRegisterDefault));
    CK(cudaHostRegister(cols, B8, cudaHostRegisterDefault));
    CK(cudaHostRegister(vals, B8, cudaHostRegisterDefault));
    double t1 = now();
    CK(cudaMemcpyAsync(d_a, rows, B8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync((char*)d_a + B8, cols, B8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync((char*)d_a + 2 * B8, vals, B8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    double t2 = now();
    CK(cudaHostUnregister(rows));
    CK(cudaHostUnregister(cols));
    CK(cudaHostUnregister(vals));
    double t3 = now();
    printf("register 2.4GB %.1f ms, DMA %.1f ms (%.1f GB/s), unregister %.1f ms\n",
           (t1 - t0) * 1e3, (t2 - t1) * 1e3, 3 * B8 / (t2 - t1) / 1e9, (t3 - t2) * 1e3);
  }
  // register in 64 MB pieces, overlapped with DMA of the previous piece
  {
    const size_t piece = 64 << 20;
    double t0 = now();
    char* srcs[3] = {(char*)rows, (char*)cols, (char*)vals};
    for (int a = 0; a < 3; ++a)
      for (size_t o = 0; o < B8; o += piece) {
        size_t len = B8 - o < piece ? B8 - o : piece;
        CK(cudaHostRegister(srcs[a] + o, len, cudaHostRegisterDefault));
        CK(cudaMemcpyAsync((char*)d_a + a * B8 + o, srcs[a] + o, len, cudaMemcpyHostToDevice, s));
      }
    CK(cudaStreamSynchronize(s));
    double t1 = now();
    for (int a = 0; a < 3; ++a)
      for (size_t o = 0; o < B8; o += piece) CK(cudaHostUnregister(srcs[a] + o));
    double t2 = now();
    printf("piecewise register+DMA 2.4GB %.1f ms, unregister %.1f ms\n", (t1 - t0) * 1e3,
           (t2 - t1) * 1e3);
  }

  // model download: 480000 x 128 fp32 on device -> fp64 host (fresh numpy-like memory)
  const int64_t un = 480000LL * 128;
  float* pin;
  CK(cudaMallocHost(&pin, un * 4));
  for (int huge = 0; huge < 2; ++huge) {
    double* dst = (double*)aligned_alloc(1 << 21, un * 8);
    if (huge) madvise(dst, un * 8, MADV_HUGEPAGE);
    double t0 = now();
    CK(cudaMemcpyAsync(pin, d_a, un * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double t1 = now();
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < un; ++i) dst[i] = pin[i];
    double t2 = now();
    printf("download U: D2H pinned fp32 %.1f ms, convert into fresh fp64 (huge=%d) %.1f ms\n",
           (t1 - t0) * 1e3, huge, (t2 - t1) * 1e3);
    free(dst);
  }
  {
    double* dst = (double*)aligned_alloc(1 << 21, un * 8);
    double t0 = now();
    CK(cudaMemcpyAsync(dst, d_a, un * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    printf("download U: pageable fp64 D2H into fresh memory %.1f ms\n", (now() - t0) * 1e3);
    double t1 = now();
    CK(cudaMemcpyAsync(dst, d_a, un * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    printf("download U: pageable fp64 D2H into touched memory %.1f ms\n", (now() - t1) * 1e3);
    free(dst);
  }
  return 0;
}
