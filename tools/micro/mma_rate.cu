// Microbenchmark: tcgen05.mma rate for the attention kernel's shapes on one SM.
//   S  : M=128 N=128 K=64  (SS, both K-major)            4 instructions
//   PV : M=128 N=64  K=128 (TS: A=P in TMEM, B=V MN-major) 8 instructions
//   PVs: the same with P in shared memory (SS)
// Reports clocks per group and the issue time (how long the issuing thread is held).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2602_21760_b200/csrc \
//   tools/micro/mma_rate.cu -o tools/micro/mma_rate
#include <cstdio>
#include "hp_tc.cuh"
using namespace hptc;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int MODE>
__global__ void k(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idS = idesc_bf16_f32(128, 128, 0), idO = idesc_bf16_f32(128, 64, 1);
    const uint64_t dq = sdesc_sw128_kmajor(sm), dk = sdesc_sw128_kmajor(sm + 16384);
    long long issue = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const long long a = clock64();
      if (MODE == 0 || MODE == 3) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, dq + 2 * kk, dk + 2 * kk, idS, kk > 0);
      }
      if (MODE == 1 || MODE == 3) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tmem + 256, tmem + 384 + 8 * kk, sdesc_sw128_mnmajor(sm + 32768 + kk * 2048, 8192), idO, 1);
      }
      if (MODE == 2) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tmem + 256, sdesc_sw128_kmajor(sm + 65536 + (kk >> 2) * 16384) + 2 * (kk & 3),
                    sdesc_sw128_mnmajor(sm + 32768 + kk * 2048, 8192), idO, 1);
      }
      issue += clock64() - a;
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = issue;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  k<MODE><<<148, 128, 100 * 1024>>>(10, d);
  k<MODE><<<148, 128, 100 * 1024>>>(iters, d);
  cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-28s %8.1f clk/group  (issue held %.1f clk/group)  %s\n", name, (double)h[0] / iters,
         (double)h[1] / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("S 128x128x64 SS");
  run<1>("PV 128x64x128 TS");
  run<2>("PV 128x64x128 SS");
  run<3>("S + PV(TS)");
  return 0;
}
