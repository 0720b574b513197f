// Microbenchmark: the attention softmax instruction stream alone (no TMEM, no MMA):
// per "block" each thread turns NV fp32 scores into bf16 P (row max, exp2 with 2 of 8
// pairs on the FMA-pipe polynomial, row sum), as attn_stream_kernel does. Compares
// 128 scores per thread with 8 warps/SM against 64 scores per thread with 16 warps/SM
// (two threads per row). Reports SM clocks per 16384 scores (one 128x128 block).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_21760_b200/csrc \
//   tools/micro/softmax_rate.cu -o tools/micro/softmax_rate
#include <cstdio>
#include "hp_tc.cuh"
using namespace hptc;

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  const float a = fmaxf(lo2(x2), -126.0f), b = fmaxf(hi2(x2), -126.0f);
  const uint64_t x = pack2(a, b);
  const uint64_t t = fadd2(x, pack2(12582912.0f, 12582912.0f));
  const uint64_t fi = fadd2(t, pack2(-12582912.0f, -12582912.0f));
  const uint64_t f = ffma2(fi, pack2(-1.0f, -1.0f), x);
  uint64_t pz = ffma2(pack2(0.05592212f, 0.05592212f), f, pack2(0.24264069f, 0.24264069f));
  pz = ffma2(pz, f, pack2(0.69312102f, 0.69312102f));
  pz = ffma2(pz, f, pack2(0.99992444f, 0.99992444f));
  const uint32_t lo = (uint32_t)pz + ((uint32_t)t << 23);
  const uint32_t hi = (uint32_t)(pz >> 32) + ((uint32_t)(t >> 32) << 23);
  return ((uint64_t)hi << 32) | lo;
}

template <int NV>
__global__ void k(int iters, long long* cyc, uint32_t* sink) {
  uint32_t r[NV];
#pragma unroll
  for (int e = 0; e < NV; ++e) r[e] = __float_as_uint(-(float)((threadIdx.x * 13 + e * 7) % 97) * 0.1f);
  uint32_t acc = 0;
  float l = 0.f, m_run = 0.f;
  const uint64_t scale2 = pack2(0.18f, 0.18f);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mx[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) mx[a] = __uint_as_float(r[a]);
#pragma unroll
    for (int e = 8; e < NV; e += 8) {
#pragma unroll
      for (int a = 0; a < 8; ++a) mx[a] = fmaxf(mx[a], __uint_as_float(r[e + a]));
    }
    const float m = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * 0.18f;
    m_run = fmaxf(m_run, m);
    const uint64_t negm2 = pack2(-m_run, -m_run);
    uint64_t sum2[4] = {0, 0, 0, 0};
    uint32_t packed[NV / 2];
#pragma unroll
    for (int e = 0; e < NV; e += 2) {
      const uint64_t x2 = ffma2(pack2u(r[e], r[e + 1]), scale2, negm2);
      uint64_t e2;
      const int pr = (e >> 1) & 7;
      if (pr == 3 || pr == 7) e2 = exp2_poly2(x2);
      else e2 = pack2(ex2f(lo2(x2)), ex2f(hi2(x2)));
      sum2[(e >> 1) & 3] = fadd2(sum2[(e >> 1) & 3], e2);
      packed[e >> 1] = pack_bf16(lo2(e2), hi2(e2));
    }
    const uint64_t s01 = fadd2(fadd2(sum2[0], sum2[1]), fadd2(sum2[2], sum2[3]));
    l += lo2(s01) + hi2(s01);
#pragma unroll
    for (int e = 0; e < NV / 2; ++e) acc ^= packed[e];
    // perturb the scores so the loop is not hoisted
#pragma unroll
    for (int e = 0; e < NV; ++e) r[e] ^= (acc & 1u);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(l);
}

template <int NV>
void run(int warps) {
  long long* cyc; uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 2000;
  k<NV><<<148, warps * 32>>>(10, cyc, sink);
  k<NV><<<148, warps * 32>>>(iters, cyc, sink);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double scores = (double)warps * 32 * NV * iters;   // per SM
  printf("NV=%3d warps/SM=%2d: %.0f clk per 16384 scores per SM (%.1f scores/clk/SM) %s\n", NV, warps,
         h[0] / (scores / 16384.0), scores / h[0], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<128>(8); run<128>(12); run<128>(16);
  run<64>(8); run<64>(16); run<64>(24); run<64>(32);
  return 0;
}
