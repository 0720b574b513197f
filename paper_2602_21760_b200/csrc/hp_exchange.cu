// hp_exchange.cu — pair exchange and pipeline staging over NVLink peer memory.
//
// The reference models a measured (condition-partitioned) step as two latent
// messages on an affine link (engine.py:217-231, trace.py:114-119) and a
// pipelined step as N-1 activation messages (engine.py:307-337). Here a
// "message" is a buffer the producer rank fills in its own HBM plus a
// system-scope release store of the step number into the consumer's flag
// word; the consumer's next kernel acquires the flag and reads the payload
// straight out of the producer's HBM through the IPC-mapped peer pointer
// (hp_sampler_step with wait_flag) or receives it pushed by hp_stage_send.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <chrono>
#include <thread>
#include "hybridpar_b200.h"
#include "hp_common.cuh"

namespace {

__global__ void signal_kernel(uint32_t* flag, uint32_t value) {
  __threadfence_system();  // everything this stream wrote before is visible first
  hp_st_release_sys_u32(flag, value);
}

__global__ void wait_kernel(const volatile uint32_t* flag, uint32_t value, int32_t* status,
                            uint64_t timeout_ns) {
  const uint64_t start = hp_globaltimer();
  if (status && *reinterpret_cast<volatile int32_t*>(status) == HP_ERR_TIMEOUT) return;   // run already lost
  while (hp_ld_acquire_sys_u32(flag) < value) {
    if (timeout_ns && hp_globaltimer() - start > timeout_ns) {
      if (status) *status = HP_ERR_TIMEOUT;
      return;
    }
    __nanosleep(128);
  }
}

__global__ void stage_copy_kernel(int4* __restrict__ dst, const int4* __restrict__ src, int64_t n16,
                                  uint8_t* dst_tail, const uint8_t* src_tail, int tail) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x) {
    dst[i] = src[i];
  }
  if (blockIdx.x == 0 && threadIdx.x < tail) dst_tail[threadIdx.x] = src_tail[threadIdx.x];
}

struct PeerPtrs {
  int4* dst[HP_MAX_PEERS];
  uint32_t* flag[HP_MAX_PEERS];
};

// one copy per destination (blockIdx.y); the source tile is read once per
// destination but stays in L2, so HBM sees ~one read and the NVLink ports
// carry the n_dst writes concurrently
__global__ void broadcast_copy_kernel(PeerPtrs p, const int4* __restrict__ src, int64_t n16,
                                      const uint8_t* src_tail, int tail) {
  int4* dst = p.dst[blockIdx.y];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x) {
    dst[i] = src[i];
  }
  if (blockIdx.x == 0 && threadIdx.x < tail)
    reinterpret_cast<uint8_t*>(dst + n16)[threadIdx.x] = src_tail[threadIdx.x];
}

__global__ void broadcast_signal_kernel(PeerPtrs p, int n, uint32_t value) {
  __threadfence_system();
  for (int i = 0; i < n; ++i)
    if (p.flag[i]) hp_st_release_sys_u32(p.flag[i], value);
}

}  // namespace

extern "C" {

int hp_ipc_get_handle(void* dev_ptr, uint8_t out_handle[HP_IPC_HANDLE_BYTES]) {
  if (!dev_ptr || !out_handle) return HP_ERR_PARAMETER;
  static_assert(sizeof(cudaIpcMemHandle_t) == HP_IPC_HANDLE_BYTES, "ipc handle size");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, dev_ptr) != cudaSuccess) return HP_ERR_CUDA;
  memcpy(out_handle, &h, sizeof(h));
  return HP_OK;
}

int hp_ipc_open(const uint8_t handle[HP_IPC_HANDLE_BYTES], void** out_ptr) {
  if (!handle || !out_ptr) return HP_ERR_PARAMETER;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return HP_ERR_CUDA;
  return HP_OK;
}

int hp_ipc_close(void* mapped_ptr) {
  if (!mapped_ptr) return HP_ERR_PARAMETER;
  return cudaIpcCloseMemHandle(mapped_ptr) == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

int hp_enable_peer(int32_t peer_device) {
  int dev = 0, can = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HP_ERR_CUDA;
  if (peer_device == dev) return HP_OK;
  if (cudaDeviceCanAccessPeer(&can, dev, peer_device) != cudaSuccess) return HP_ERR_CUDA;
  if (!can) return HP_ERR_UNSUPPORTED;
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); return HP_OK; }
  return e == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

int hp_signal(uint32_t* flag, uint32_t value, void* stream) {
  if (!flag) return HP_ERR_PARAMETER;
  signal_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag, value);
  return cudaGetLastError() == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

int hp_flag_wait(const volatile uint32_t* flag, uint32_t value, int32_t* status, uint64_t timeout_ns,
                 void* stream) {
  if (!flag) return HP_ERR_PARAMETER;
  wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag, value, status, timeout_ns);
  return cudaGetLastError() == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

int hp_flag_poll(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, uint32_t* observed) {
  if (!flag) return HP_ERR_PARAMETER;
  static thread_local cudaStream_t st = nullptr;
  static thread_local int st_dev = -1;
  static thread_local uint32_t* host = nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HP_ERR_CUDA;
  if (!st || st_dev != dev) {
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return HP_ERR_CUDA;
    if (!host && cudaMallocHost(&host, sizeof(uint32_t)) != cudaSuccess) return HP_ERR_CUDA;
    st_dev = dev;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    if (cudaMemcpyAsync(host, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return HP_ERR_CUDA;
    const uint32_t v = *reinterpret_cast<volatile uint32_t*>(host);
    if (v >= value) {
      if (observed) *observed = v;
      return HP_OK;
    }
    if (timeout_ns) {
      const auto ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0);
      if ((uint64_t)ns.count() > timeout_ns) return HP_ERR_TIMEOUT;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(5));
  }
}

int hp_stage_send(void* dst, const void* src, int64_t nbytes, uint32_t* flag, uint32_t value,
                  void* stream) {
  if (nbytes < 0 || (nbytes > 0 && (!dst || !src))) return HP_ERR_PARAMETER;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) return HP_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (nbytes > 0) {
    const int64_t n16 = nbytes / 16;
    const int tail = (int)(nbytes - n16 * 16);
    int blocks = (int)((n16 + 255) / 256);
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 4) blocks = 148 * 4;
    stage_copy_kernel<<<blocks, 256, 0, st>>>(static_cast<int4*>(dst), static_cast<const int4*>(src), n16,
                                              static_cast<uint8_t*>(dst) + n16 * 16,
                                              static_cast<const uint8_t*>(src) + n16 * 16, tail);
    if (cudaGetLastError() != cudaSuccess) return HP_ERR_CUDA;
  }
  if (flag) return hp_signal(flag, value, stream);
  return HP_OK;
}

int hp_stage_broadcast(void* const* dsts, uint32_t* const* flags, int32_t n_dst, const void* src,
                       int64_t nbytes, uint32_t value, void* stream) {
  if (n_dst < 0 || n_dst > HP_MAX_PEERS || nbytes < 0) return HP_ERR_PARAMETER;
  if (n_dst == 0) return HP_OK;
  if (nbytes > 0 && (!src || !dsts)) return HP_ERR_PARAMETER;
  PeerPtrs p{};
  uintptr_t align = reinterpret_cast<uintptr_t>(src);
  for (int i = 0; i < n_dst; ++i) {
    p.flag[i] = flags ? flags[i] : nullptr;
    if (nbytes == 0) continue;                 // signal-only (acknowledgements)
    if (!dsts[i]) return HP_ERR_PARAMETER;
    p.dst[i] = static_cast<int4*>(dsts[i]);
    align |= reinterpret_cast<uintptr_t>(dsts[i]);
  }
  if (align & 15) return HP_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (nbytes > 0) {
    const int64_t n16 = nbytes / 16;
    const int tail = (int)(nbytes - n16 * 16);
    int bx = (int)((n16 + 255) / 256);
    if (bx < 1) bx = 1;
    const int cap = (148 * 4 + n_dst - 1) / n_dst;
    if (bx > cap) bx = cap;
    broadcast_copy_kernel<<<dim3(bx, n_dst), 256, 0, st>>>(p, static_cast<const int4*>(src), n16,
                                                           static_cast<const uint8_t*>(src) + n16 * 16, tail);
    if (cudaGetLastError() != cudaSuccess) return HP_ERR_CUDA;
  }
  if (flags) {
    broadcast_signal_kernel<<<1, 1, 0, st>>>(p, n_dst, value);
    if (cudaGetLastError() != cudaSuccess) return HP_ERR_CUDA;
  }
  return HP_OK;
}

int hp_alloc(int64_t nbytes, void** out_ptr) {
  if (nbytes <= 0 || !out_ptr) return HP_ERR_PARAMETER;
  if (cudaMalloc(out_ptr, (size_t)nbytes) != cudaSuccess) return HP_ERR_CUDA;
  if (cudaMemset(*out_ptr, 0, (size_t)nbytes) != cudaSuccess) return HP_ERR_CUDA;
  return cudaDeviceSynchronize() == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

int hp_free(void* ptr) {
  if (!ptr) return HP_ERR_PARAMETER;
  return cudaFree(ptr) == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

const char* hp_version(void) { return "hybridpar_b200 0.1.0 (sm_100a)"; }

int hp_device_sm_count(int32_t* out) {
  if (!out) return HP_ERR_PARAMETER;
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HP_ERR_CUDA;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return HP_ERR_CUDA;
  *out = v;
  return HP_OK;
}

}  // extern "C"
