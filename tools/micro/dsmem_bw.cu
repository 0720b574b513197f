// Microbenchmark: distributed-shared-memory exchange rate, the split-K GEMM's partial
// hand-off. Clusters of 4 CTAs (148 CTAs -> 37 clusters), 128 threads each; every CTA
// ships 80 KB (128 rows x 160 fp32) into CTA rank^2's shared memory:
//   v4   : per-thread st.shared::cluster.v4 (the kernel's current path)
//   bulk : stage locally, then one cp.async.bulk.shared::cluster.shared::cta per warp
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_21760_b200/csrc \
//   tools/micro/dsmem_bw.cu -o tools/micro/dsmem_bw
#include <cstdio>
#include "hp_tc.cuh"
using namespace hptc;

constexpr int kBytes = 80 * 1024;

template <int MODE>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(128, 1) k(int iters, long long* out, float4* gbuf) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* src = sm;              // local staging
  uint8_t* dst = sm + kBytes;     // receive area (written by the partner)
  __shared__ uint64_t bar;
  const uint32_t rank = cluster_ctarank();
  const uint32_t peer = rank ^ 2u;
  for (int i = threadIdx.x; i < kBytes / 4; i += 128) reinterpret_cast<float*>(src)[i] = (float)i;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  cluster_barrier();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      const uint32_t rdst = mapa_shared(dst, peer);
      for (int i = threadIdx.x; i < kBytes / 16; i += 128) {
        const float4 v = reinterpret_cast<const float4*>(src)[i];
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};"
                     :: "r"(rdst + i * 16), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
      }
      cluster_barrier();
    } else if (MODE == 2) {
      // through L2: write this CTA's partial to global, cluster barrier, partner reads it back
      float4* mine = gbuf + (size_t)blockIdx.x * (kBytes / 16);
      const float4* theirs = gbuf + (size_t)(blockIdx.x ^ 2) * (kBytes / 16);
      for (int i = threadIdx.x; i < kBytes / 16; i += 128) mine[i] = reinterpret_cast<const float4*>(src)[i];
      cluster_barrier();
      float acc = 0.f;
      for (int i = threadIdx.x; i < kBytes / 16; i += 128) {
        const float4 v = theirs[i];
        reinterpret_cast<float4*>(dst)[i] = v;
        acc += v.x;
      }
      if (acc == -1.f) out[1] = 1;
      cluster_barrier();
    } else {
      // one bulk copy per warp (20 KB each) into the partner, completion on the partner's barrier
      if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar, kBytes);
      cluster_barrier();                 // partner armed its barrier
      if ((threadIdx.x & 31) == 0) {
        const int w = threadIdx.x >> 5;
        const uint32_t rdst = mapa_shared(dst + w * (kBytes / 4), peer);
        const uint32_t rbar = mapa_shared(&bar, peer);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(rdst), "r"(smem_u32(src + w * (kBytes / 4))), "r"(kBytes / 4), "r"(rbar) : "memory");
      }
      mbar_wait(&bar, it & 1);
      cluster_barrier();
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

template <int MODE>
void run(const char* name) {
  long long* d;
  float4* gb;
  cudaMalloc(&d, 16);
  cudaMalloc(&gb, (size_t)148 * kBytes);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kBytes);
  k<MODE><<<148, 128, 2 * kBytes>>>(4, d, gb);
  k<MODE><<<148, 128, 2 * kBytes>>>(200, d, gb);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-5s: %lld clk per 80 KB exchange (%.0f B/clk per SM) %s\n", name, h, (double)kBytes / h,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("v4");
  run<1>("bulk");
  run<2>("L2");
  return 0;
}
