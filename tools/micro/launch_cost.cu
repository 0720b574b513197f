// Microbenchmark: in-graph cost per kernel launch for the shapes of the denoiser's
// kernels: 148 CTAs x 256 threads, with / without PDL, 2-CTA clusters, ~200 KB of
// dynamic shared memory and a TMEM allocate/free. 200 back-to-back launches per graph.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_21760_b200/csrc \
//   tools/micro/launch_cost.cu -o tools/micro/launch_cost
#include <cstdio>
#include "hp_tc.cuh"
using namespace hptc;

template <bool TMEM, bool PDLW>
__global__ void k(int* p) {
  extern __shared__ uint8_t sm[];
  __shared__ uint32_t slot;
  if (PDLW) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (TMEM) {
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (PDLW) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
  if (TMEM) {
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(slot);
  }
  (void)sm;
}

template <bool TMEM, bool PDLW>
float run(int cluster, bool pdl, size_t smem) {
  int* d;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(k<TMEM, PDLW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaStream_t st;
  cudaStreamCreate(&st);
  auto launch = [&]() {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int n = 0;
    if (pdl) { at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[n].val.programmaticStreamSerializationAllowed = 1; ++n; }
    if (cluster > 1) { at[n].id = cudaLaunchAttributeClusterDimension; at[n].val.clusterDim.x = cluster; at[n].val.clusterDim.y = 1; at[n].val.clusterDim.z = 1; ++n; }
    cfg.attrs = at;
    cfg.numAttrs = n;
    cudaLaunchKernelEx(&cfg, k<TMEM, PDLW>, d);
  };
  for (int i = 0; i < 3; ++i) launch();
  cudaStreamSynchronize(st);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int reps = 200;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < reps; ++i) launch();
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1e3f / reps;
}

int main() {
  printf("plain                         %.2f us\n", run<false, false>(1, false, 0));
  printf("PDL                           %.2f us\n", run<false, true>(1, true, 0));
  printf("PDL + cluster 2               %.2f us\n", run<false, true>(2, true, 0));
  printf("PDL + cluster 4               %.2f us\n", run<false, true>(4, true, 0));
  printf("PDL + 200 KB smem             %.2f us\n", run<false, true>(1, true, 200 * 1024));
  printf("PDL + 200 KB smem + cluster 2 %.2f us\n", run<false, true>(2, true, 200 * 1024));
  printf("PDL + TMEM                    %.2f us\n", run<true, true>(1, true, 0));
  printf("PDL + TMEM + 200KB + cluster2 %.2f us\n", run<true, true>(2, true, 200 * 1024));
  printf("no PDL + TMEM + 200KB + cl2   %.2f us\n", run<true, false>(2, false, 200 * 1024));
  return 0;
}
