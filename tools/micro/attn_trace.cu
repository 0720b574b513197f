// Event timeline of one attention CTA (clock64), built from the product kernel with
// HP_ATTN_TRACE: for each key block of each stream, when the MMA warp saw K/V
// arrive (kv), saw S released (sfree_ok), issued S (S_iss), saw P (p_ok); when the
// softmax started waiting for S (sm_wait), got S (s_ok), released S (sfree), had P
// in registers (exp), saw PV(i-1) done (o_ok) and published P (p_full).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHP_ATTN_TRACE \
//   -I include -I paper_2602_21760_b200/csrc tools/micro/attn_trace.cu -o tools/micro/attn_trace -lcuda
#include "../../paper_2602_21760_b200/csrc/hp_attn.cu"
#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 1, H = argc > 2 ? atoi(argv[2]) : 2, S = argc > 3 ? atoi(argv[3]) : 16384;
  const int SKV = argc > 4 ? atoi(argv[4]) : S;   // <= 128: the single-block kernel
  const size_t n = (size_t)B * (S > SKV ? S : SKV) * H * 64;
  std::vector<__nv_bfloat16> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = __float2bfloat16((float)((i * 2654435761u) % 2001) / 1000.f - 1.f);
  void *q, *k, *v, *o;
  cudaMalloc(&q, n * 2); cudaMalloc(&k, n * 2); cudaMalloc(&v, n * 2); cudaMalloc(&o, n * 2);
  cudaMemcpy(q, h.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(k, h.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(v, h.data(), n * 2, cudaMemcpyHostToDevice);
  hp_attn_desc d{};
  d.q = q; d.k = k; d.v = v; d.o = o;
  d.ldq = d.ldk = d.ldv = d.ldo = H * 64;
  d.batch = B; d.heads = H; d.sq = S; d.skv = SKV; d.scale = 0.125f;
  for (int r = 0; r < 3; ++r) hp_attention(&d, nullptr);
  cudaDeviceSynchronize();
  if (SKV <= 128) {
    // graph of 20 launches: per-launch time and the last launch's CTA-0 timeline
    cudaStream_t st; cudaStreamCreate(&st);
    cudaGraph_t gr; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < 20; ++r) hp_attention(&d, st);
    cudaStreamEndCapture(st, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long st16[16];
    cudaMemcpyFromSymbol(st16, g_single_trace, sizeof(st16));
    const char* nm[9] = {"entry", "pdl passed", "Q,K,V landed", "S issued", "softmax got S", "P published",
                         "O ready", "stored", "CTA done"};
    printf("single-block B=%d H=%d Sq=%d Skv=%d: %.2f us per launch (graph); CTA 0:", B, H, S, SKV, ms * 1e3 / 20);
    for (int e = 0; e < 9; ++e) printf(" %s %lld |", nm[e], st16[e] - st16[0]);
    printf("\n");
    return 0;
  }
  static long long t[2][12][256];
  cudaMemcpyFromSymbol(t, g_attn_trace, sizeof(t));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  const char* names[12] = {"kv", "sfree_ok", "S_iss", "p_ok", "sm_wait", "s_ok", "sfree", "exp", "o_ok", "p_full",
                           "", ""};
  const long long t0 = t[0][0][0];  // CTA 0, stream 0, first block
  const int J = (S + 127) / 128;
  for (int q = 0; q < 2; ++q) {
    printf("stream %d\n  i ", q);
    for (int e = 0; e < 10; ++e) printf("%9s", names[e]);
    printf("\n");
    for (int i = 0; i < (J < 24 ? J : 24); ++i) {
      printf("%3d ", i);
      for (int e = 0; e < 10; ++e) printf("%9lld", t[q][e][i] ? t[q][e][i] - t0 : -1);
      printf("\n");
    }
  }
  // steady-state averages over blocks 8..J-8 of stream 0 (deltas)
  for (int q = 0; q < 2; ++q) {
    double per = 0, waitS = 0, ld = 0, exp = 0, owait = 0, pub = 0, sIss2ok = 0;
    int cnt = 0;
    for (int i = 8; i < J - 8 && i < 250; ++i, ++cnt) {
      per += t[q][5][i + 1] - t[q][5][i];
      waitS += t[q][5][i] - t[q][4][i];
      ld += t[q][6][i] - t[q][5][i];
      exp += t[q][7][i] - t[q][6][i];
      owait += t[q][8][i] - t[q][7][i];
      pub += t[q][9][i] - t[q][8][i];
      sIss2ok += t[q][5][i] - t[q][2][i];
    }
    if (cnt)
      printf("stream %d steady: period %.0f | wait S %.0f | ld+release %.0f | max+exp %.0f | o wait(+fold) %.0f | "
             "rescale+P st %.0f | S issue->softmax got it %.0f\n", q, per / cnt, waitS / cnt, ld / cnt, exp / cnt,
             owait / cnt, pub / cnt, sIss2ok / cnt);
  }
  return 0;
}
