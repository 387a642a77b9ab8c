// peer.cu -- V-block moves of the multi-GPU ring over peer memory.
//
// In the U-resident / V-rotating ring (distributed.py) every
// batch moves a few V blocks (C4: 570 KB) from rank g to rank g+1.  Instead
// of an NCCL send/recv pair per move, ranks map each other's V buffers and
// flag words once (CUDA IPC: cudaIpcGetMemHandle / cudaIpcOpenMemHandle, which
// also works between processes sharing one GPU) and the move becomes two
// stream-ordered operations on the engine stream:
//   sender:   copy V_j rows straight into the receiver's V_j rows (NVLink
//             P2P writes; no staging, no NCCL proxy), then a one-thread
//             kernel stores flag[sender] = seq with release semantics at
//             system scope;
//   receiver: a one-warp kernel spins (acquire, system scope) until
//             flag[sender] >= seq before the next sweep is allowed to run.
// seq counts the moves sender -> receiver; both sides derive it from the same
// deterministic schedule, so no host handshake is needed per batch.
// Write-after-read safety comes from the ring's causality: a rank writes into
// a peer's V_j rows only after V_j has travelled away from that peer, and the
// peer pushed it only after its own kernels on V_j (sweep and SSE) finished.

#include "bgmf_internal.cuh"

namespace bgmf {
namespace {

__global__ void peer_signal_kernel(unsigned int* flag, unsigned int value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

__global__ void peer_wait_kernel(const unsigned int* flag, unsigned int value) {
  if (threadIdx.x != 0) return;
  unsigned int v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - value) >= 0) break;  // wrap-safe >=
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
  cudaSetDevice(c->device);
  if (bytes > 0)
    BGMF_CK(c, cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, c->stream));
  peer_signal_kernel<<<1, 1, 0, c->stream>>>(peer_flag, value);
  BGMF_CK(c, cudaGetLastError());
  return BGMF_OK;
}

extern "C" int bgmf_peer_wait(bgmf_ctx* c, const uint32_t* flag, uint32_t value) {
  if (!c || !flag) return fail(c, BGMF_ERR_ARG, "bgmf_peer_wait: bad argument");
  cudaSetDevice(c->device);
  peer_wait_kernel<<<1, 32, 0, c->stream>>>(flag, value);
  BGMF_CK(c, cudaGetLastError());
  return BGMF_OK;
}

namespace bgmf {
void peer_release(bgmf_ctx* c) {
  for (void* p : c->peer_opened) cudaIpcCloseMemHandle(p);
  c->peer_opened.clear();
  for (void* p : c->peer_owned) cudaFree(p);
  c->peer_owned.clear();
}
}  // namespace bgmf
