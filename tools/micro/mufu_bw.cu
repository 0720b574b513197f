// Microbenchmark: exp2 throughput per SM on B200 for the softmax's candidate forms:
// ex2.approx.f32, ex2.approx.ftz.bf16x2, ex2.approx.f16x2 (elements per clock per SM),
// plus the packed FMA-pipe polynomial for comparison.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_bw.cu -o mufu_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

constexpr int kChains = 8;

template <int MODE>
__global__ void k(int iters, unsigned long long* cycles, uint32_t* sink) {
  uint32_t v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = 0x3f003f00u ^ (threadIdx.x * 7 + c);   // small negative-ish values
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (MODE == 0) {
        float x = __uint_as_float(v[c] | 0x80000000u), y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        v[c] = __float_as_uint(y) & 0x3fffffffu;
      } else if (MODE == 1) {
        uint32_t y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(v[c] | 0x80008000u));
        v[c] = y & 0x3fff3fffu;
      } else {
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(v[c] | 0x80008000u));
        v[c] = y & 0x3bff3bffu;
      }
    }
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc ^= v[c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, int threads) {
  const int blocks = 148, iters = 4096;
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, blocks * 8);
  cudaMalloc(&sink, blocks * threads * 4);
  k<MODE><<<blocks, threads>>>(16, cyc, sink);
  k<MODE><<<blocks, threads>>>(iters, cyc, sink);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  const double elems = (double)threads * iters * kChains * (MODE == 0 ? 1 : 2);
  printf("%-22s threads %4d: %.2f elements/clk/SM  (%.2f instr/clk/SM)\n", name, threads, elems / mx,
         (double)threads * iters * kChains / mx);
}

int main() {
  for (int t : {256, 512, 1024}) {
    run<0>("ex2.approx.ftz.f32", t);
    run<1>("ex2.approx.ftz.bf16x2", t);
    run<2>("ex2.approx.f16x2", t);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
