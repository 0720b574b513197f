// Event timeline (globaltimer ns from kernel entry) of cluster 0 of the CTA-pair GEMM,
// built from the product kernel with HP_GEMM_TRACE: setup done (barriers, TMEM), PDL
// wait passed, first TMA issued, first stage landed, first tile's MMAs issued,
// accumulator ready in the epilogue, epilogue done, final cluster barrier.
// Runs M x N x K 20 times back to back in a CUDA graph and reports the last launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHP_GEMM_TRACE \
//   -I include -I paper_2602_21760_b200/csrc tools/micro/gemm_trace.cu -o tools/micro/gemm_trace -lcuda
#include "../../paper_2602_21760_b200/csrc/hp_gemm.cu"
#include <cstdio>
#include <cstdlib>

int main(int argc, char** argv) {
  const long M = argc > 1 ? atol(argv[1]) : 2048, N = argc > 2 ? atol(argv[2]) : 1280, K = argc > 3 ? atol(argv[3]) : 1280;
  const int bn = argc > 4 ? atoi(argv[4]) : 0;
  void *a, *b, *d;
  cudaMalloc(&a, M * K * 2); cudaMalloc(&b, N * K * 2); cudaMalloc(&d, M * N * 2);
  cudaMemset(a, 0, M * K * 2); cudaMemset(b, 0, N * K * 2);
  hp_gemm_desc g{};
  g.a = a; g.lda = K; g.a_mode = HP_A_PLAIN; g.b = b; g.ldb = K; g.d = d; g.ldd = N;
  g.M = M; g.N = N; g.K = K; g.block_n = bn; g.alpha = 1.0f;
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int i = 0; i < 3; ++i) hp_gemm(&g, st);
  cudaStreamSynchronize(st);
  cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 20; ++i) hp_gemm(&g, st);
  cudaStreamEndCapture(st, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long ring[kRing][13];
  unsigned int ctr = 0;
  cudaMemcpyFromSymbol(ring, g_gemm_ring, sizeof(ring));
  cudaMemcpyFromSymbol(&ctr, g_gemm_ctr, sizeof(ctr));
  const unsigned long long* last = ring[(ctr - 1) % kRing];
  printf("%s; %ldx%ldx%ld bn=%d: %.2f us per launch in the graph\n", cudaGetErrorString(cudaGetLastError()), M, N, K,
         bn, ms * 1e3 / 20);
  const char* nm[9] = {"entry", "setup done", "pdl wait passed", "first TMA issued", "first stage landed",
                       "tile 0 MMAs issued", "acc ready (epi)", "epilogue done", "final barrier"};
  printf("last launch, cluster 0 leader (ns from entry):");
  for (int e = 0; e < 9; ++e) printf("  %s %lld", nm[e], last[e] ? (long long)(last[e] - last[0]) : -1);
  printf("\n");
  return 0;
}
