// peer.cu -- V-block moves of the multi-GPU ring over peer memory.
//
// In the U-resident / V-rotating ring (distributed.py) every
// batch moves a few V blocks (C4: 570 KB) from rank g to rank g+1.  Instead
// of an NCCL send/recv pair per move, ranks map each other's V buffers and
// flag words once (CUDA IPC: cudaIpcGetMemHandle / cudaIpcOpenMemHandle, which
// also works between processes sharing one GPU) and the move becomes two
// stream-ordered operations on the engine stream:
//   sender:   one kernel copies V_j rows straight into the receiver's V_j
//             rows (NVLink P2P writes; no staging, no NCCL proxy) and, once
//             every CTA's stores are fenced system-wide, release-stores
//             flag[sender] = seq (system scope);
//   receiver: a one-warp kernel spins (acquire, system scope) until
//             flag[sender] >= seq before the next sweep is allowed to run.
// seq counts the moves sender -> receiver; both sides derive it from the same
// deterministic schedule, so no host handshake is needed per batch.
// Write-after-read safety comes from the ring's causality: a rank writes into
// a peer's V_j rows only after V_j has travelled away from that peer, and the
// peer pushed it only after its own kernels on V_j (sweep and SSE) finished.

#include <algorithm>

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

// The move itself: SM stores of the block into the peer's rows (NVLink P2P
// writes), then the CUDA "last block" pattern at system scope -- every thread
// fences its stores system-wide before its CTA counts itself done, and the
// last CTA fences again and release-stores the flag -- so a receiver that
// acquires the flag sees the whole block (PTX memory model; a copy-engine
// memcpy followed by a separate flag kernel would rely on stream-completion
// semantics across devices instead).  `done` is this context's counter, reset
// by the last CTA for the next (stream-ordered) push.
__global__ void __launch_bounds__(256)
peer_push_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n4,
                 unsigned char* __restrict__ dst_tail, const unsigned char* __restrict__ src_tail,
                 int tail, unsigned int* flag, unsigned int value, unsigned int* done) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldg(src + i);
  if (blockIdx.x == 0 && (int)threadIdx.x < tail) dst_tail[threadIdx.x] = src_tail[threadIdx.x];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
      *done = 0u;
    }
  }
}

// The receiver's wait is bounded: it gives up when the sender's rank has
// raised the ring's abort word (any rank that fails sets it in every peer's
// flag page, bgmf_peer_abort) or after `timeout_ns` of %globaltimer, and then
// records the reason in `err` (1: timeout, 2: abort) for bgmf_peer_error --
// a dead peer can never hang the surviving ranks' streams.
__global__ void peer_wait_kernel(const unsigned int* flag, unsigned int value,
                                 const unsigned int* abort_word, unsigned int* err,
                                 unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned int v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - value) >= 0) break;  // wrap-safe >=
    if (abort_word) {
      unsigned int a;
      asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(a) : "l"(abort_word) : "memory");
      if (a) { atomicMax(err, 2u); break; }
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) { atomicMax(err, 1u); break; }
    __nanosleep(256);
  }
}

}  // namespace
}  // namespace bgmf

using namespace bgmf;

extern "C" int bgmf_peer_alloc(bgmf_ctx* c, int64_t bytes, void** out) {
  if (!c || !out || bytes <= 0) return fail(c, BGMF_ERR_ARG, "bgmf_peer_alloc: bad argument");
  cudaSetDevice(c->device);
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);  // plain cudaMalloc: IPC-exportable
  if (e == cudaSuccess) e = cudaMemset(p, 0, (size_t)bytes);
  if (e != cudaSuccess) {
    if (p) cudaFree(p);
    return cuda_fail(c, e, "bgmf_peer_alloc");
  }
  c->peer_owned.push_back(p);
  *out = p;
  return BGMF_OK;
}

extern "C" int bgmf_peer_handle(bgmf_ctx* c, void* base, uint8_t* handle_out) {
  if (!c || !base || !handle_out) return fail(c, BGMF_ERR_ARG, "bgmf_peer_handle: bad argument");
  cudaSetDevice(c->device);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, base);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == BGMF_PEER_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  return BGMF_OK;
}

extern "C" int bgmf_peer_open(bgmf_ctx* c, const uint8_t* handle, void** out) {
  if (!c || !handle || !out) return fail(c, BGMF_ERR_ARG, "bgmf_peer_open: bad argument");
  cudaSetDevice(c->device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaIpcOpenMemHandle");
  c->peer_opened.push_back(p);
  *out = p;
  return BGMF_OK;
}

extern "C" int bgmf_peer_push(bgmf_ctx* c, void* dst, const void* src, int64_t bytes,
                              uint32_t* peer_flag, uint32_t value) {
  if (!c || !dst || !src || !peer_flag || bytes < 0)
    return fail(c, BGMF_ERR_ARG, "bgmf_peer_push: bad argument");
  if (((uintptr_t)dst | (uintptr_t)src) & 15)
    return fail(c, BGMF_ERR_ARG, "bgmf_peer_push: buffers must be 16-byte aligned");
  cudaSetDevice(c->device);
  if (!c->d_push_done) {
    BGMF_CK(c, cudaMalloc(&c->d_push_done, sizeof(unsigned int)));
    BGMF_CK(c, cudaMemsetAsync(c->d_push_done, 0, sizeof(unsigned int), c->stream));
  }
  const int64_t n4 = bytes / 16;
  const int tail = (int)(bytes % 16);
  int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 2 * (int64_t)c->num_sms);
  if (blocks < 1) blocks = 1;
  peer_push_kernel<<<blocks, 256, 0, c->stream>>>(
      static_cast<float4*>(dst), static_cast<const float4*>(src), n4,
      static_cast<unsigned char*>(dst) + n4 * 16, static_cast<const unsigned char*>(src) + n4 * 16,
      tail, peer_flag, value, c->d_push_done);
  BGMF_CK(c, cudaGetLastError());
  return BGMF_OK;
}

extern "C" int bgmf_peer_wait(bgmf_ctx* c, const uint32_t* flag, uint32_t value) {
  if (!c || !flag) return fail(c, BGMF_ERR_ARG, "bgmf_peer_wait: bad argument");
  cudaSetDevice(c->device);
  if (!c->d_peer_err) {
    BGMF_CK(c, cudaMalloc(&c->d_peer_err, sizeof(unsigned int)));
    BGMF_CK(c, cudaMemsetAsync(c->d_peer_err, 0, sizeof(unsigned int), c->stream));
  }
  peer_wait_kernel<<<1, 32, 0, c->stream>>>(flag, value, c->peer_abort, c->d_peer_err,
                                            c->peer_timeout_ns);
  BGMF_CK(c, cudaGetLastError());
  return BGMF_OK;
}

extern "C" int bgmf_peer_config(bgmf_ctx* c, const uint32_t* abort_word, double timeout_s) {
  if (!c || timeout_s <= 0) return fail(c, BGMF_ERR_ARG, "bgmf_peer_config: bad argument");
  c->peer_abort = reinterpret_cast<const unsigned int*>(abort_word);
  c->peer_timeout_ns = (unsigned long long)(timeout_s * 1e9);
  return BGMF_OK;
}

extern "C" int bgmf_peer_abort(bgmf_ctx* c, uint32_t* peer_abort_word) {
  if (!c || !peer_abort_word) return fail(c, BGMF_ERR_ARG, "bgmf_peer_abort: bad argument");
  cudaSetDevice(c->device);
  const uint32_t one = 1;
  // a plain copy into the peer's mapped page: no dependence on this rank's
  // (possibly failed) stream
  BGMF_CK(c, cudaMemcpy(peer_abort_word, &one, sizeof(one), cudaMemcpyHostToDevice));
  return BGMF_OK;
}

extern "C" int bgmf_peer_error(bgmf_ctx* c, int* out) {
  if (!c || !out) return fail(c, BGMF_ERR_ARG, "bgmf_peer_error: bad argument");
  cudaSetDevice(c->device);
  *out = 0;
  if (!c->d_peer_err) return BGMF_OK;
  unsigned int e = 0;
  BGMF_CK(c, cudaMemcpyAsync(&e, c->d_peer_err, sizeof(e), cudaMemcpyDeviceToHost, c->stream));
  BGMF_CK(c, cudaStreamSynchronize(c->stream));
  *out = (int)e;
  return BGMF_OK;
}

namespace bgmf {
void peer_release(bgmf_ctx* c) {
  if (c->d_push_done) cudaFree(c->d_push_done);
  c->d_push_done = nullptr;
  if (c->d_peer_err) cudaFree(c->d_peer_err);
  c->d_peer_err = nullptr;
  c->peer_abort = nullptr;
  for (void* p : c->peer_opened) cudaIpcCloseMemHandle(p);
  c->peer_opened.clear();
  for (void* p : c->peer_owned) cudaFree(p);
  c->peer_owned.clear();
}
}  // namespace bgmf
