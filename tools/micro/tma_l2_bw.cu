// Microbenchmark: TMA L2 -> shared-memory throughput with the GEMM's load pattern
// (no MMA): each CTA streams K blocks of its A rows (128 x 64 bf16 box) and B rows
// (BNH x 64 box) through a STAGES-deep ring; one warp frees the stages as they land.
// Mode 0: unicast. Mode 1: A multicast across CTA pairs {r, r^2} of a 4-CTA cluster
// (the two CTAs with the same A rows each load half the box for both).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_l2_bw.cu -o tma_l2_bw -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { printf("err %d line %d\n", (int)e_, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint64_t* b, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(b)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(a) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
               "@!P bra W;\n\t}" :: "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               :: "r"(smem_u32(dst)), "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, uint16_t mask) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
               " [%0], [%1, {%3, %4}], [%2], %5;"
               :: "r"(smem_u32(dst)), "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask) : "memory");
}
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int STAGES = 6;
struct P { int num_kb, reps, m_tiles, n_tiles, bnh, mode; };

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                                            const __grid_constant__ CUtensorMap tAh, P p, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t A_BYTES = 128 * 64 * 2, B_BYTES = p.bnh * 64 * 2, ST = A_BYTES + ((B_BYTES + 1023) & ~1023u);
  uint64_t* full = (uint64_t*)(sm + STAGES * ST);
  uint64_t* empty = full + STAGES;
  const uint32_t r = ctarank();
  // tile of this CTA: 4-CTA cluster = 2 pairs; pair q = r>>1 takes n tile 2*cl+q, both pairs share m
  const int cl = blockIdx.x >> 2, q = (r >> 1) & 1, pr = r & 1;
  const int mt = cl % p.m_tiles, nt = ((cl / p.m_tiles) * 2 + q) % p.n_tiles;
  const int m0 = mt * 256 + pr * 128, nb = nt * 2 * p.bnh + pr * p.bnh;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], p.mode ? 2 : 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync();
  const int total = p.num_kb * p.reps;
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < total; ++it) {
      const int s = it % STAGES, kb = it % p.num_kb;
      wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      expect_tx(&full[s], A_BYTES + B_BYTES);
      uint8_t* a = sm + s * ST;
      if (p.mode == 0) tma2d(a, &tA, &full[s], kb * 64, m0);
      else  // half box (64 rows) for me and my A-partner r^2
        tma2d_mc(a + q * (A_BYTES / 2), &tAh, &full[s], kb * 64, m0 + q * 64, (uint16_t)((1u << r) | (1u << (r ^ 2))));
      tma2d(a + A_BYTES, &tB, &full[s], kb * 64, nb);
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < total; ++it) {
      const int s = it % STAGES;
      wait(&full[s], (it / STAGES) & 1);
      arrive(&empty[s]);
      if (p.mode) arrive_remote(&empty[s], r ^ 2);   // partner may overwrite its half of my A only when I am done
    }
  }
  __syncthreads();
  cluster_sync();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static CUtensorMap make(void* base, int rows, int cols, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
  CK(enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return m;
}

int main(int argc, char** argv) {
  const int M = atoi(argv[1]), N = atoi(argv[2]), K = atoi(argv[3]), bn = atoi(argv[4]), mode = atoi(argv[5]);
  const int reps = argc > 6 ? atoi(argv[6]) : 20;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  void *A, *B;
  CK(cudaMalloc(&A, (size_t)M * K * 2));
  CK(cudaMalloc(&B, (size_t)N * K * 2));
  CK(cudaMemset(A, 0, (size_t)M * K * 2));
  CK(cudaMemset(B, 0, (size_t)N * K * 2));
  CUtensorMap tA = make(A, M, K, 128), tB = make(B, N, K, bn / 2), tAh = make(A, M, K, 64);
  P p{K / 64, reps, M / 256, N / bn, bn / 2, mode};
  const int pairs = (M / 256) * (N / bn);
  const int grid = pairs * 2;
  const uint32_t st = 128 * 64 * 2 + ((bn / 2 * 128 + 1023) & ~1023);
  const size_t smem = STAGES * st + 2048;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned long long* out;
  CK(cudaMalloc(&out, grid * 8));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int w = 0; w < 3; ++w) CK(cudaLaunchKernelEx(&cfg, k, tA, tB, tAh, p, out));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  CK(cudaLaunchKernelEx(&cfg, k, tA, tB, tAh, p, out));
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)grid * p.num_kb * reps * (128 * 64 * 2 + bn / 2 * 64 * 2);
  printf("M=%d N=%d K=%d bn=%d mode=%s ctas=%d: %.1f us, %.2f us/kstep, smem fill %.2f TB/s\n", M, N, K, bn,
         mode ? "A-multicast" : "unicast", grid, ms * 1e3, ms * 1e3 / (p.num_kb * reps), bytes / ms / 1e9);
  return 0;
}
