// Microbenchmark: the GEMM epilogue's output store pattern in isolation. 148 CTAs x 128
// threads; each CTA writes a 128-row x BN-column bf16 tile of a row-major [M, N] matrix.
//   rowwise: thread = row, 32 columns (64 B) per chunk as two 256-bit stores (the epilogue)
//   coalesced: a warp writes 32 consecutive 16-byte pieces of one row per instruction
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/store_pattern.cu -o tools/micro/store_pattern
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE, int BN>
__global__ void k(uint16_t* d, int ldd) {
  const int tile_m = blockIdx.x % 16, tile_n = blockIdx.x / 16;   // 16 x (N / BN) tiles
  const int m0 = tile_m * 128, n0 = tile_n * BN;
  const uint32_t v = threadIdx.x * 0x10001u;
  if (MODE == 0) {
    uint16_t* row = d + (size_t)(m0 + threadIdx.x) * ldd + n0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(row + c * 32), "r"(v) : "memory");
      asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(row + c * 32 + 16), "r"(v) : "memory");
    }
  } else {
    // each warp: rows warp, warp+4, ...; lanes cover BN*2 bytes of the row in 16-B pieces
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kPieces = BN * 2 / 16;
#pragma unroll 1
    for (int r = warp; r < 128; r += 4) {
      uint16_t* row = d + (size_t)(m0 + r) * ldd + n0;
      for (int q = lane; q < kPieces; q += 32)
        *reinterpret_cast<uint4*>(row + q * 8) = make_uint4(v, v, v, v);
    }
  }
}

template <int MODE, int BN>
void run(const char* name) {
  const int M = 2048, N = 148 / 16 * BN + BN;   // enough tiles for 148 CTAs
  uint16_t* d;
  cudaMalloc(&d, (size_t)M * N * 2 + (1 << 20));
  cudaStream_t st; cudaStreamCreate(&st);
  k<MODE, BN><<<148, 128, 0, st>>>(d, N);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 50; ++i) k<MODE, BN><<<148, 128, 0, st>>>(d, N);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, st); cudaGraphLaunch(ge, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-10s BN=%d: %.2f us per launch (%s)\n", name, BN, ms * 1e3 / 50, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 160>("rowwise"); run<1, 160>("coalesced");
  run<0, 256>("rowwise"); run<1, 256>("coalesced");
  return 0;
}
