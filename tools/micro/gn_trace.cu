// Event timeline (clock64 from entry) of CTA (0,0) of the single-launch GroupNorm, built
// from the product kernel with HP_GN_TRACE: PDL passed, pixel chunk landed in smem,
// statistics written, image barrier passed, normalised chunk stored. 20 launches in a
// CUDA graph; per-launch time and the last launch's timeline.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHP_GN_TRACE -I include \
//   -I paper_2602_21760_b200/csrc tools/micro/gn_trace.cu -o tools/micro/gn_trace -lcuda
#include "../../paper_2602_21760_b200/csrc/hp_norm.cu"
#include <cstdio>
#include <cstdlib>

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 2, C = argc > 3 ? atoi(argv[3]) : 1280;
  const long hw = argc > 2 ? atol(argv[2]) : 1024;
  void *x, *y; float *g, *b, *st;
  cudaMalloc(&x, n * hw * C * 2); cudaMalloc(&y, n * hw * C * 2);
  cudaMalloc(&g, C * 4); cudaMalloc(&b, C * 4); cudaMalloc(&st, 2 * n * 32 * 256 * 4);
  cudaMemset(x, 0, n * hw * C * 2); cudaMemset(g, 0, C * 4); cudaMemset(b, 0, C * 4);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int i = 0; i < 3; ++i) hp_group_norm(x, C, nullptr, 0, n, hw, 32, 1e-5f, g, b, 1, y, st, s);
  cudaStreamSynchronize(s);
  cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 20; ++i) hp_group_norm(x, C, nullptr, 0, n, hw, 32, 1e-5f, g, b, 1, y, st, s);
  cudaStreamEndCapture(s, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long t[8];
  cudaMemcpyFromSymbol(t, g_gn_trace, sizeof(t));
  printf("GN n=%d hw=%ld C=%d: %.2f us per launch (%s) | CTA(0,0) clk: pdl %lld, chunk landed %lld, stats %lld, "
         "barrier %lld, stored %lld\n", n, hw, C, ms * 1e3 / 20, cudaGetErrorString(cudaGetLastError()), t[1] - t[0],
         t[2] - t[0], t[3] - t[0], t[4] - t[0], t[5] - t[0]);
  return 0;
}
