// hp_norm.cu — K6: the denoiser's memory-bound ops on bf16 NHWC / row tensors.
//
// GroupNorm(+SiLU) is two passes (per-image partial statistics over pixel
// chunks, then a normalise pass that folds the partials in fixed order), so
// it is deterministic and batch-invariant: image b's statistics never depend
// on the other images in the batch. Normally one launch: an image's statistics
// CTAs meet at an in-kernel barrier (all resident: occupancy-checked), each CTA
// having staged its pixel chunk in shared memory with bulk async copies when the
// chunk is >= 16 KB. The barrier words belong to the launch (a slot per stream
// for eager launches, a fresh slot per captured graph node) and the launch is
// cooperative, so co-residency is guaranteed by the driver, not assumed. LayerNorm is one warp per row with an
// exact two-pass mean/variance from registers and optional adaLN modulation.
// Everything else is a 16-byte-vectorised streaming kernel.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <mutex>
#include <unordered_map>
#include "hybridpar_b200_denoiser.h"
#include "hp_common.cuh"
#include "hp_tc.cuh"

namespace {

using bf16 = __nv_bfloat16;
using hptc::fence_barrier_init;
using hptc::mbar_arrive_expect_tx;
using hptc::mbar_init;
using hptc::mbar_wait;
using hptc::smem_u32;

__device__ __forceinline__ void load8(const bf16* p, float* v) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void store8(bf16* p, const float* v) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void load8f(const float* p, float* v) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }
// x * sigmoid(x) = 0.5 x (1 + tanh(x / 2)): one MUFU.TANH instead of EX2 + RCP
__device__ __forceinline__ float silu_fast(float x) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
  return 0.5f * x * (1.0f + t);
}

inline int nblocks(int64_t work, int per_block, int cap = 148 * 16) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}
inline bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------------------
// GroupNorm pass 1: grid (splits, n). Thread t owns 8-channel vector j = t % V
// of pixels t / V, t / V + R, ... within the block's pixel chunk.
constexpr int kGnThreads = 256;
constexpr int kMaxC = 2560;

// GroupNorm partial sums of one (image n, pixel split) block: fixed-order
// reduction (no float atomics): deterministic, batch-invariant
// ch1 / ch2: the chunk's first pixel row of each input (global memory or a shared-memory
// copy with the same row strides c1 / c2); npx pixels. Same arithmetic order either way.
__device__ __forceinline__ void gn_stats_block(const bf16* ch1, int c1, const bf16* ch2, int c2, int64_t npx,
                                               int groups, int splits, float* __restrict__ part, int n, int split,
                                               float* s_sum, float* s_sq, float* p_sum, float* p_sq) {
  const int C = c1 + c2;
  const int V = C / 8;
  const int64_t p_begin = 0, p_end = npx;
  for (int j0 = 0; j0 < V; j0 += kGnThreads) {
    const int vecs = min(V - j0, kGnThreads);
    const int rows = kGnThreads / vecs;
    const int j = j0 + threadIdx.x % vecs;
    const int r = threadIdx.x / vecs;
    float sum[8] = {0}, sq[8] = {0};
    if (r < rows) {
      const int ch = j * 8;
      const bf16* src = ch < c1 ? ch1 + ch : ch2 + (ch - c1);
      const int64_t st = ch < c1 ? c1 : c2;
      int64_t p = p_begin + r;
      // four 16-byte loads in flight per thread (the loop is latency-bound otherwise)
      for (; p + 3 * rows < p_end; p += 4 * rows) {
        uint4 u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = *reinterpret_cast<const uint4*>(src + (p + k * rows) * st);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[k]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h[i]);
            sum[2 * i] += f.x; sq[2 * i] = fmaf(f.x, f.x, sq[2 * i]);
            sum[2 * i + 1] += f.y; sq[2 * i + 1] = fmaf(f.y, f.y, sq[2 * i + 1]);
          }
        }
      }
      for (; p < p_end; p += rows) {
        float v[8];
        load8(src + p * st, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) { sum[i] += v[i]; sq[i] = fmaf(v[i], v[i], sq[i]); }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) { p_sum[threadIdx.x * 8 + i] = sum[i]; p_sq[threadIdx.x * 8 + i] = sq[i]; }
    __syncthreads();
    for (int q = threadIdx.x; q < vecs * 8; q += kGnThreads) {
      const int jj = q / 8, i = q % 8;
      float a = 0.f, b = 0.f;
      for (int rr = 0; rr < rows; ++rr) { a += p_sum[(rr * vecs + jj) * 8 + i]; b += p_sq[(rr * vecs + jj) * 8 + i]; }
      s_sum[(j0 + jj) * 8 + i] = a;
      s_sq[(j0 + jj) * 8 + i] = b;
    }
    __syncthreads();
  }
  // per-group sums: `per` threads per group over strided channels, then one thread per
  // group folds them in fixed order (p_sum / p_sq are free again here)
  const int cg = C / groups;
  const int per = kGnThreads / groups;
  {
    const int g = threadIdx.x / per, k = threadIdx.x % per;
    float a = 0.f, b = 0.f;
    if (g < groups)
      for (int c = g * cg + k; c < (g + 1) * cg; c += per) { a += s_sum[c]; b += s_sq[c]; }
    p_sum[threadIdx.x] = a;
    p_sq[threadIdx.x] = b;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < groups; g += kGnThreads) {
    float a = 0.f, b = 0.f;
    for (int k = 0; k < per; ++k) { a += p_sum[g * per + k]; b += p_sq[g * per + k]; }
    float* o = part + (((int64_t)n * splits + split) * groups + g) * 2;
    o[0] = a;
    o[1] = b;
  }
}

__global__ void __launch_bounds__(kGnThreads)
gn_stats_kernel(const bf16* __restrict__ x1, int c1, const bf16* __restrict__ x2, int c2, int64_t hw,
                int groups, int splits, float* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_sum[kMaxC], s_sq[kMaxC];
  __shared__ float p_sum[kGnThreads * 8], p_sq[kGnThreads * 8];
  const int n = blockIdx.y, split = blockIdx.x;
  const int64_t p0 = hw * split / splits, p1 = hw * (split + 1) / splits;
  gn_stats_block(x1 + ((int64_t)n * hw + p0) * c1, c1, x2 ? x2 + ((int64_t)n * hw + p0) * c2 : nullptr, c2, p1 - p0,
                 groups, splits, part, n, split, s_sum, s_sq, p_sum, p_sq);
}

// GroupNorm pass 2 for image n: fold the per-split partials (fixed order), then
// y = x * sa[c] + sb[c] (+ SiLU) over pixels p_first + r, stepping p_mul * rows
// xa / xb: image n's first pixel row of each input (or a shared-memory chunk copy
// whose row 0 is pixel `src_p0`); y: the output image base. Pixels p_first + r,
// stepping p_mul * rows, up to p_end (image pixel indices).
__device__ __forceinline__ void gn_normalise(const bf16* xa, int c1, const bf16* xb, int c2, int groups,
                                             const float* __restrict__ gamma, const float* __restrict__ beta,
                                             int do_silu, bf16* __restrict__ yo, int64_t src_p0, int64_t p_first,
                                             int64_t p_mul, int64_t p_end, const float* s_mean, const float* s_rstd,
                                             float* sa, float* sb);

__device__ __forceinline__ void gn_apply_block(const bf16* xa, int c1, const bf16* xb, int c2, int64_t hw, int groups,
                                               int splits, const float* __restrict__ part, float eps,
                                               const float* __restrict__ gamma, const float* __restrict__ beta,
                                               int do_silu, bf16* __restrict__ yo, int n, int64_t src_p0,
                                               int64_t p_first, int64_t p_mul, int64_t p_end, float* s_mean,
                                               float* s_rstd, double* s_pa, double* s_pb, float* sa, float* sb) {
  const int C = c1 + c2;
  const int cg = C / groups;
  {
    // fold the per-split partials: kGnThreads/groups threads per group, fixed order;
    // a warp's loads cover consecutive groups of one split (coalesced), 8 in flight
    const int per = kGnThreads / groups;
    const int g = threadIdx.x % groups, k = threadIdx.x / groups;
    double a = 0.0, b = 0.0;
    if (k < per) {
      const float* base = part + ((int64_t)n * splits * groups + g) * 2;
      int s = k;
      for (; s + 7 * per < splits; s += 8 * per) {
        float2 o[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) o[u] = *reinterpret_cast<const float2*>(base + (int64_t)(s + u * per) * groups * 2);
#pragma unroll
        for (int u = 0; u < 8; ++u) { a += (double)o[u].x; b += (double)o[u].y; }
      }
      for (; s < splits; s += per) {
        const float2 o = *reinterpret_cast<const float2*>(base + (int64_t)s * groups * 2);
        a += (double)o.x;
        b += (double)o.y;
      }
    }
    s_pa[threadIdx.x] = a;
    s_pb[threadIdx.x] = b;
    __syncthreads();
    if (threadIdx.x < groups) {
      double ta = 0.0, tb = 0.0;
      for (int kk = 0; kk < per; ++kk) { ta += s_pa[kk * groups + threadIdx.x]; tb += s_pb[kk * groups + threadIdx.x]; }
      const double cnt = (double)hw * cg;
      const double mean = ta / cnt;
      double var = tb / cnt - mean * mean;
      if (var < 0) var = 0;
      s_mean[threadIdx.x] = (float)mean;
      s_rstd[threadIdx.x] = (float)(1.0 / sqrt(var + (double)eps));
    }
  }
  __syncthreads();
  gn_normalise(xa, c1, xb, c2, groups, gamma, beta, do_silu, yo, src_p0, p_first, p_mul, p_end, s_mean, s_rstd, sa,
               sb);
}

// y = x * sa[c] + sb[c] (+ SiLU) from the per-group mean / rstd (see gn_apply_block)
__device__ __forceinline__ void gn_normalise(const bf16* xa, int c1, const bf16* xb, int c2, int groups,
                                             const float* __restrict__ gamma, const float* __restrict__ beta,
                                             int do_silu, bf16* __restrict__ yo, int64_t src_p0, int64_t p_first,
                                             int64_t p_mul, int64_t p_end, const float* s_mean, const float* s_rstd,
                                             float* sa, float* sb) {
  const int C = c1 + c2;
  const int V = C / 8;
  const int cg = C / groups;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int g = c / cg;
    const float a = s_rstd[g] * gamma[c];
    sa[c] = a;
    sb[c] = beta[c] - s_mean[g] * a;
  }
  __syncthreads();
  // thread -> fixed 8-channel vector j, strided over pixels: no per-element index math
  const int vc = V < kGnThreads ? V : kGnThreads;
  const int rows = kGnThreads / vc;
  const int r = threadIdx.x / vc;
  if (r >= rows) return;
  for (int j = threadIdx.x % vc; j < V; j += vc) {
    const int ch = j * 8;
    float av[8], bv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { av[k] = sa[ch + k]; bv[k] = sb[ch + k]; }
    const bool first = ch < c1;
    const bf16* src = first ? xa + ch : xb + (ch - c1);
    const int64_t sstride = first ? c1 : c2;
    const int64_t step = p_mul * rows;
    int64_t p = p_first + r;
    for (; p + 3 * step < p_end; p += 4 * step) {         // four loads in flight
      uint4 u[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) u[k] = *reinterpret_cast<const uint4*>(src + (p - src_p0 + k * step) * sstride);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[k]);
        float v[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          v[2 * i] = f.x; v[2 * i + 1] = f.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float o = fmaf(v[i], av[i], bv[i]);
          v[i] = do_silu ? silu_fast(o) : o;
        }
        store8(yo + (p + k * step) * C + ch, v);
      }
    }
    for (; p < p_end; p += step) {
      float v[8];
      load8(src + (p - src_p0) * sstride, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float o = fmaf(v[k], av[k], bv[k]);
        v[k] = do_silu ? silu_fast(o) : o;
      }
      store8(yo + p * C + ch, v);
    }
  }
}

__global__ void __launch_bounds__(kGnThreads)
gn_apply_kernel(const bf16* __restrict__ x1, int c1, const bf16* __restrict__ x2, int c2, int64_t hw,
                int groups, int splits, const float* __restrict__ part, float eps,
                const float* __restrict__ gamma, const float* __restrict__ beta, int do_silu,
                bf16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_mean[64], s_rstd[64];
  __shared__ double s_pa[kGnThreads], s_pb[kGnThreads];
  __shared__ __align__(16) float sa[kMaxC], sb[kMaxC];
  const int n = blockIdx.y;
  gn_apply_block(x1 + (int64_t)n * hw * c1, c1, x2 ? x2 + (int64_t)n * hw * c2 : nullptr, c2, hw, groups, splits,
                 part, eps, gamma, beta, do_silu, y + (int64_t)n * hw * (c1 + c2), n, 0,
                 (int64_t)blockIdx.x * (kGnThreads / min((c1 + c2) / 8, kGnThreads)), gridDim.x, hw, s_mean, s_rstd,
                 s_pa, s_pb, sa, sb);
}

// GroupNorm from the producing GEMMs' partials (hp_gemm gn_part): no statistics pass
// and no grid-wide barrier. grid (chunks, n); each CTA folds its image's partials per
// group in fixed order (kGnThreads / groups threads per group over (segment, block)
// items, fp64, then the group's threads in order) and normalises its pixels. Channels
// [0, c1) take their segments from part1, [c1, C) from part2 (a concat's second input).
constexpr int kGnPartRows = 128;     // rows per partial (hp_gemm's 128-row block)
constexpr int kGnPartSeg = 10;       // columns per partial segment
constexpr int kGnPartsMaxThreads = 512;
#ifndef HP_GN_PARTS_DEPTH
#define HP_GN_PARTS_DEPTH 4
#endif
#ifndef HP_GN_PARTS_THREADS
#define HP_GN_PARTS_THREADS 256
#endif
#ifndef HP_GN_PARTS_CTAS_PER_SM
#define HP_GN_PARTS_CTAS_PER_SM 2
#endif
constexpr int kGnPartsDepth = HP_GN_PARTS_DEPTH;    // 16-byte loads in flight per thread
__global__ void __launch_bounds__(kGnPartsMaxThreads)
gn_parts_kernel(const bf16* __restrict__ x, int C, int64_t hw, const float2* __restrict__ part1, int c1,
                const float2* __restrict__ part2, int groups, float eps, const float* __restrict__ gamma,
                const float* __restrict__ beta, int do_silu, bf16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_mean[64], s_rstd[64];
  __shared__ double s_pa[kGnThreads], s_pb[kGnThreads];
  __shared__ __align__(16) float sa[kMaxC], sb[kMaxC];
  const int n = blockIdx.y;
  // thread -> fixed 8-channel vector j = t % V (its scale / shift stay in registers), pixels
  // p0, p0 + step, ...; the block is a whole number of pixel rows of V threads (launcher)
  const int V = C / 8, rows = (int)blockDim.x / V;
  const int r = threadIdx.x / V, j = threadIdx.x % V, ch = j * 8;
  const int64_t step = (int64_t)gridDim.x * rows, p0 = (int64_t)blockIdx.x * rows + r;
  const bf16* xi = x + (int64_t)n * hw * C + ch;
  bf16* yi = y + (int64_t)n * hw * C + ch;
  // the thread's first kGnPartsDepth pixels are in flight during the fold
  uint4 pre[kGnPartsDepth];
#pragma unroll
  for (int k = 0; k < kGnPartsDepth; ++k)
    if (p0 + k * step < hw) pre[k] = *reinterpret_cast<const uint4*>(xi + (p0 + k * step) * C);
  const int P = (int)(hw / kGnPartRows);
  const int cg = C / groups, sg = cg / kGnPartSeg;
  const int ns1 = c1 / kGnPartSeg, ns2 = (C - c1) / kGnPartSeg;
  // per threads per group fold (the first per * groups threads of the block)
  const int per = min((int)blockDim.x, kGnThreads) / groups;
  const int g = threadIdx.x % groups, k = threadIdx.x / groups;
  if (threadIdx.x < per * groups) {
    double a = 0.0, b = 0.0;
    if (k < per) {
      // items of group g: segment g * sg + it / P, block it % P; eight loads per round
      // (zeros past the end: exact), summed in item order
      const int items = sg * P;
      for (int i = k; i < items; i += 8 * per) {
        float2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int it = i + u * per;
          v[u] = make_float2(0.f, 0.f);
          if (it < items) {
            const int sgi = g * sg + it / P, rb = it % P;
            v[u] = sgi < ns1 ? __ldg(part1 + ((int64_t)n * P + rb) * ns1 + sgi)
                             : __ldg(part2 + ((int64_t)n * P + rb) * ns2 + (sgi - ns1));
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) { a += (double)v[u].x; b += (double)v[u].y; }
      }
    }
    s_pa[threadIdx.x] = a;
    s_pb[threadIdx.x] = b;
  }
  __syncthreads();
  if (threadIdx.x < groups) {
    double ta = 0.0, tb = 0.0;
    for (int kk = 0; kk < per; ++kk) { ta += s_pa[kk * groups + threadIdx.x]; tb += s_pb[kk * groups + threadIdx.x]; }
    const double cnt = (double)hw * cg;
    const double mean = ta / cnt;
    double var = tb / cnt - mean * mean;
    if (var < 0) var = 0;
    s_mean[threadIdx.x] = (float)mean;
    s_rstd[threadIdx.x] = (float)(1.0 / sqrt(var + (double)eps));
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float sc = s_rstd[c / cg] * gamma[c];
    sa[c] = sc;
    sb[c] = beta[c] - s_mean[c / cg] * sc;
  }
  __syncthreads();
  float av[8], bv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) { av[q] = sa[ch + q]; bv[q] = sb[ch + q]; }
  auto emit = [&](const uint4& u, int64_t p) {
    const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
    float v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(hv[i]);
      v[2 * i] = f.x; v[2 * i + 1] = f.y;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float o = fmaf(v[i], av[i], bv[i]);
      v[i] = do_silu ? silu_fast(o) : o;
    }
    store8(yi + p * C, v);
  };
#pragma unroll
  for (int q = 0; q < kGnPartsDepth; ++q)
    if (p0 + q * step < hw) emit(pre[q], p0 + q * step);
  int64_t p = p0 + kGnPartsDepth * step;
  for (; p + (kGnPartsDepth - 1) * step < hw; p += kGnPartsDepth * step) {   // all loads in flight
    uint4 u[kGnPartsDepth];
#pragma unroll
    for (int q = 0; q < kGnPartsDepth; ++q) u[q] = *reinterpret_cast<const uint4*>(xi + (p + q * step) * C);
#pragma unroll
    for (int q = 0; q < kGnPartsDepth; ++q) emit(u[q], p + q * step);
  }
  for (; p < hw; p += step) emit(*reinterpret_cast<const uint4*>(xi + p * C), p);
}

// Single-launch GroupNorm: the statistics CTAs of an image meet at a
// sense-reversing barrier (every CTA of the grid is resident: the launcher checks
// occupancy), fold the partials and normalise the pixels they just reduced (an
// L2 hit). Same partition and fold as the two-kernel path: bit-identical output.
// largest pixel chunk of a split, bytes, rounded to 128 (the staged variant's scratch follows it)
__host__ __device__ __forceinline__ size_t gn_chunk_bytes(int64_t hw, int splits, int C) {
  return ((size_t)((hw + splits - 1) / splits) * C * 2 + 127) & ~(size_t)127;
}
__host__ __device__ __forceinline__ size_t gn_smem_bytes(int64_t hw, int splits, int C) {
  return gn_chunk_bytes(hw, splits, C) + (size_t)(2 * C + 2 * kGnThreads * 8) * sizeof(float);
}
// 1-D bulk async copy global -> this CTA's shared memory, completion on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void image_barrier(unsigned* cnt, unsigned* gen, unsigned expected) {
  const unsigned g = *reinterpret_cast<volatile unsigned*>(gen);
  __threadfence();
  if (atomicAdd(cnt, 1u) == expected - 1) {
    atomicExch(cnt, 0u);
    __threadfence();
    atomicAdd(gen, 1u);
  } else {
    while (*reinterpret_cast<volatile unsigned*>(gen) == g) __nanosleep(32);
  }
  __threadfence();
}

// SMEM: the CTA first copies its pixel chunk of each input into shared memory with
// bulk async copies (all of it in flight at once), reduces it from there and
// normalises it from there (no second global read).
#ifdef HP_GN_TRACE
__device__ long long g_gn_trace[8];
#define HP_NTRACE(ev) do { if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_gn_trace[ev] = clock64(); } while (0)
#else
#define HP_NTRACE(ev) do {} while (0)
#endif
template <bool SMEM>
__global__ void __launch_bounds__(kGnThreads)
gn_fused_kernel(const bf16* __restrict__ x1, int c1, const bf16* __restrict__ x2, int c2, int64_t hw,
                int groups, int splits, float* __restrict__ part, float eps, const float* __restrict__ gamma,
                const float* __restrict__ beta, int do_silu, bf16* __restrict__ y, unsigned* __restrict__ bar) {
  extern __shared__ __align__(128) uint8_t gn_chunk[];
  __shared__ uint64_t ld_bar;
  HP_NTRACE(0);
  pdl_wait();
  HP_NTRACE(1);
  pdl_trigger();
  const int n = blockIdx.y, split = blockIdx.x;
  const int64_t p_begin = hw * split / splits, p_end = hw * (split + 1) / splits;
  const int64_t npx = p_end - p_begin;
  // reduction scratch: [cmax] sums, [cmax] squares, [kGnThreads * 8] x 2 thread partials
  // (reused by the apply phase); sized by C behind the chunk when it is staged
  float* sm;
  int cmax;
  if constexpr (SMEM) {
    cmax = c1 + c2;
    sm = reinterpret_cast<float*>(gn_chunk + gn_chunk_bytes(hw, splits, c1 + c2));
  } else {
    __shared__ __align__(16) float sm_static[2 * kMaxC + 2 * kGnThreads * 8];
    cmax = kMaxC;
    sm = sm_static;
  }
  const bf16* g1 = x1 + ((int64_t)n * hw + p_begin) * c1;
  const bf16* g2 = x2 ? x2 + ((int64_t)n * hw + p_begin) * c2 : nullptr;
  const bf16* ch1 = g1;
  const bf16* ch2 = g2;
  if constexpr (SMEM) {
    bf16* d1 = reinterpret_cast<bf16*>(gn_chunk);
    bf16* d2 = d1 + npx * c1;
    if (threadIdx.x == 0) {
      mbar_init(&ld_bar, 1);
      fence_barrier_init();
      const uint32_t b1 = (uint32_t)(npx * c1 * 2), b2 = g2 ? (uint32_t)(npx * c2 * 2) : 0u;
      mbar_arrive_expect_tx(&ld_bar, b1 + b2);
      constexpr uint32_t kPiece = 16384;
      for (uint32_t o = 0; o < b1; o += kPiece)
        bulk_g2s(reinterpret_cast<uint8_t*>(d1) + o, reinterpret_cast<const uint8_t*>(g1) + o, min(kPiece, b1 - o),
                 &ld_bar);
      for (uint32_t o = 0; o < b2; o += kPiece)
        bulk_g2s(reinterpret_cast<uint8_t*>(d2) + o, reinterpret_cast<const uint8_t*>(g2) + o, min(kPiece, b2 - o),
                 &ld_bar);
    }
    __syncthreads();
    mbar_wait(&ld_bar, 0);
    HP_NTRACE(2);
    ch1 = d1;
    ch2 = g2 ? d2 : nullptr;
  }
  gn_stats_block(ch1, c1, ch2, c2, npx, groups, splits, part, n, split, sm, sm + cmax, sm + 2 * cmax,
                 sm + 2 * cmax + kGnThreads * 8);
  __syncthreads();
  HP_NTRACE(3);
  if (threadIdx.x == 0) image_barrier(bar + 2 * n, bar + 2 * n + 1, (unsigned)splits);
  __syncthreads();
  HP_NTRACE(4);
  double* dp = reinterpret_cast<double*>(sm + 2 * cmax);               // [2][kGnThreads] doubles
  float* s_mean = sm + 2 * cmax + 4 * kGnThreads;
  gn_apply_block(ch1, c1, ch2, c2, hw, groups, splits, part, eps, gamma, beta, do_silu, y + (int64_t)n * hw * (c1 + c2),
                 n, p_begin, p_begin, 1, p_end, s_mean, s_mean + 64, dp, dp + kGnThreads, sm, sm + cmax);
  HP_NTRACE(5);
}

// ---------------------------------------------------------------------------
// LayerNorm: one warp per row, c <= 32 * 8 * kLnVec
constexpr int kLnVec = 8;          // 8-channel vectors per lane at most: c <= 2048
// LayerNorm rows: one warp per row. Each CTA owns a contiguous range of rows (grid = 2
// CTAs per SM), so its rows touch at most two (batch, stream) segments of the adaLN
// modulation: their shift / scale vectors (and gamma / beta) are staged in shared
// memory once instead of being re-read from L2 by every row (SD3's joint LayerNorm:
// 20 -> 15 us for 54 MB of traffic, with the row prefetch below). Each warp keeps the next row's
// loads in flight as raw bf16 (KV uint4 per lane) while it normalises the current one. Same
// arithmetic order as before: per-lane sums over (vector, element), then the warp sum.
template <int KV, bool MOD, bool AFF>     // MOD: shift / scale given; AFF: gamma / beta given
__global__ void __launch_bounds__(256, KV >= 7 ? 1 : 2)
ln_kernel(const bf16* __restrict__ x, int64_t rows, int c, float eps, const float* __restrict__ gamma,
          const float* __restrict__ beta, const float* __restrict__ shift_a, const float* __restrict__ scale_a,
          int64_t ldm, int64_t rows_per_batch, bf16* __restrict__ y, const float* __restrict__ shift2,
          const float* __restrict__ scale2, int64_t split) {
  extern __shared__ __align__(16) float ln_s[];         // [2 segments][shift | scale][c], gamma[c], beta[c]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int V = c / 8;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r_lo = (int64_t)blockIdx.x * per;
  const int64_t r_hi = r_lo + per < rows ? r_lo + per : rows;
  constexpr bool mod = MOD;
  if constexpr (!AFF) { gamma = nullptr; beta = nullptr; }
  if constexpr (!MOD) { shift_a = scale_a = shift2 = scale2 = nullptr; }
  // (batch, stream) segment of a row; the modulation pointers of a segment
  auto seg_of = [&](int64_t r) -> int64_t {
    const int64_t b = rows_per_batch > 0 ? r / rows_per_batch : 0;
    const int st = (split >= 0 && r - b * rows_per_batch >= split) ? 1 : 0;
    return 2 * b + st;
  };
  auto seg_ptr = [&](int64_t sg, bool want_scale) -> const float* {
    const float* base = want_scale ? ((sg & 1) ? scale2 : scale_a) : ((sg & 1) ? shift2 : shift_a);
    return base ? base + (sg >> 1) * ldm : nullptr;
  };
  const int64_t seg0 = r_lo < rows ? seg_of(r_lo) : 0, seg1 = r_hi > r_lo ? seg_of(r_hi - 1) : seg0;
  float* s_seg = ln_s;                                   // [2][2][c]
  float* s_gam = ln_s + 4 * c;
  float* s_bet = s_gam + c;
  // gamma / beta are parameters: staged before the PDL wait
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    if (gamma) s_gam[i] = gamma[i];
    if (beta) s_bet[i] = beta[i];
  }
  pdl_wait();
  pdl_trigger();
  if (mod) {
    for (int q = 0; q < 2; ++q) {
      const int64_t sg = q == 0 ? seg0 : seg1;
      const float* sh = seg_ptr(sg, false);
      const float* sc = seg_ptr(sg, true);
      for (int i = threadIdx.x; i < c; i += blockDim.x) {
        s_seg[(q * 2 + 0) * c + i] = sh ? sh[i] : 0.0f;
        s_seg[(q * 2 + 1) * c + i] = sc ? sc[i] : 0.0f;
      }
    }
  }
  __syncthreads();
  uint4 cur[KV], nxt[KV];
  auto issue = [&](int64_t r, uint4 (&dst)[KV]) {
    if (r >= r_hi) return;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int j = lane + 32 * k;
      if (j < V) dst[k] = *reinterpret_cast<const uint4*>(x + r * c + j * 8);
    }
  };
  issue(r_lo + warp, cur);
  for (int64_t row = r_lo + warp; row < r_hi; row += 8) {
    issue(row + 8, nxt);                           // the next row's loads in flight meanwhile
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int j = lane + 32 * k;
      if (j < V) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&cur[k]);
#pragma unroll
        for (int i = 0; i < 4; ++i) { const float2 f = __bfloat1622float2(h[i]); sum += f.x; sum += f.y; }
      }
    }
    sum = hp_warp_sum_f(sum);
    const float mean = sum / c;
    float sq = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int j = lane + 32 * k;
      if (j < V) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&cur[k]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          const float d0 = f.x - mean, d1 = f.y - mean;
          sq += d0 * d0;
          sq += d1 * d1;
        }
      }
    }
    sq = hp_warp_sum_f(sq);
    const float rstd = rsqrtf(sq / c + eps);
    // modulation of this row: staged (the CTA's at most two segments) or, for a row of
    // a third segment (tiny segments only), straight from global memory
    const int64_t sg = mod ? seg_of(row) : 0;
    const float* shift = nullptr;
    const float* scale = nullptr;
    if (mod) {
      if (sg == seg0 || sg == seg1) {
        const int q = sg == seg0 ? 0 : 1;
        shift = seg_ptr(sg, false) ? s_seg + (q * 2 + 0) * c : nullptr;
        scale = seg_ptr(sg, true) ? s_seg + (q * 2 + 1) * c : nullptr;
      } else {
        shift = seg_ptr(sg, false);
        scale = seg_ptr(sg, true);
      }
    }
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int j = lane + 32 * k;
      if (j >= V) continue;
      float v[8], o[8], sh[8], sc[8], ga[8], be[8];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&cur[k]);
#pragma unroll
      for (int i = 0; i < 4; ++i) { const float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
      if (MOD && shift) load8f(shift + j * 8, sh);
      if (MOD && scale) load8f(scale + j * 8, sc);
      if (AFF && gamma) load8f(s_gam + j * 8, ga);
      if (AFF && beta) load8f(s_bet + j * 8, be);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float t = (v[i] - mean) * rstd;
        if (AFF && gamma) t = t * ga[i];
        if (AFF && beta) t = t + be[i];
        if (MOD && scale) t = t * (1.0f + sc[i]);
        if (MOD && shift) t = t + sh[i];
        o[i] = t;
      }
      store8(y + row * c + j * 8, o);
    }
#pragma unroll
    for (int k = 0; k < KV; ++k) cur[k] = nxt[k];
  }
}

// launch the instance with the fewest vectors per lane that covers c (and only the
// modulation / affine code the call uses)
cudaError_t launch_ln(cudaStream_t st, const bf16* x, int64_t rows, int c, float eps, const float* gamma,
                      const float* beta, const float* shift, const float* scale, int64_t ldm, int64_t rows_per_batch,
                      bf16* y, const float* shift2, const float* scale2, int64_t split) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int kv = (c / 8 + 31) / 32;
  const int64_t want = (rows + 7) / 8;
  const dim3 grid((unsigned)(want < 2 * sms ? want : 2 * sms));
  const size_t smem = (size_t)6 * c * sizeof(float);   // 2 segments x (shift, scale), gamma, beta
  const bool mod = shift || scale, aff = gamma || beta;
#define HP_LN_LAUNCH(N, M, A) \
  hp_launch_pdl(ln_kernel<N, M, A>, grid, dim3(256), smem, st, x, rows, c, eps, gamma, beta, shift, scale, ldm, \
                rows_per_batch, y, shift2, scale2, split)
#define HP_LN_CASE(N) \
  case N: return mod ? (aff ? HP_LN_LAUNCH(N, true, true) : HP_LN_LAUNCH(N, true, false)) \
                     : (aff ? HP_LN_LAUNCH(N, false, true) : HP_LN_LAUNCH(N, false, false));
  switch (kv) {
    HP_LN_CASE(1) HP_LN_CASE(2) HP_LN_CASE(3) HP_LN_CASE(4) HP_LN_CASE(5) HP_LN_CASE(6) HP_LN_CASE(7) HP_LN_CASE(8)
    default: return cudaErrorInvalidValue;
  }
#undef HP_LN_CASE
#undef HP_LN_LAUNCH
}

// ---------------------------------------------------------------------------
__global__ void quick_gelu_kernel(const bf16* __restrict__ x, bf16* __restrict__ y, int64_t n8) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float v[8];
    load8(x + i * 8, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = v[k] / (1.0f + __expf(-1.702f * v[k]));
    store8(y + i * 8, v);
  }
}

__global__ void silu_kernel(const bf16* __restrict__ x, bf16* __restrict__ y, int64_t n8) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float v[8];
    load8(x + i * 8, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = silu(v[k]);
    store8(y + i * 8, v);
  }
}

__global__ void upsample2x_kernel(const bf16* __restrict__ x, int n, int h, int w, int c, bf16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int V = c / 8;
  const int64_t total = (int64_t)n * 2 * h * 2 * w * V;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % V);
    int64_t pix = i / V;
    const int ox = (int)(pix % (2 * w));
    pix /= (2 * w);
    const int oy = (int)(pix % (2 * h));
    const int b = (int)(pix / (2 * h));
    const uint4 u = *reinterpret_cast<const uint4*>(x + (((int64_t)b * h + oy / 2) * w + ox / 2) * c + j * 8);
    *reinterpret_cast<uint4*>(y + i * 8) = u;
  }
}

__global__ void concat_kernel(const bf16* __restrict__ a, int c1, const bf16* __restrict__ b, int c2,
                              int64_t pixels, bf16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int V1 = c1 / 8, V = (c1 + c2) / 8;
  const int64_t total = pixels * V;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / V;
    const int j = (int)(i - p * V);
    uint4 u = j < V1 ? *reinterpret_cast<const uint4*>(a + p * c1 + j * 8)
                     : *reinterpret_cast<const uint4*>(b + p * c2 + (j - V1) * 8);
    *reinterpret_cast<uint4*>(y + i * 8) = u;
  }
}

// conv_in: cin = CIN (4), cout multiple of 32. Thread = (pixel, 32 output
// channels); a warp holds 32 consecutive pixels of one channel group, so every
// weight read is a shared-memory broadcast.
template <int CIN>
__global__ void __launch_bounds__(256)
conv_small_in_kernel(const bf16* __restrict__ x, int n, int h, int w, const float* __restrict__ wgt,
                     const float* __restrict__ bias, int cout, bf16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float s_w[];  // [cout][9*CIN] then bias[cout]
  constexpr int KK = 9 * CIN;
  for (int i = threadIdx.x; i < cout * KK; i += blockDim.x) s_w[i] = wgt[i];
  for (int i = threadIdx.x; i < cout; i += blockDim.x) s_w[cout * KK + i] = bias ? bias[i] : 0.f;
  __syncthreads();
  const int G = cout / 32;
  const int64_t pixels = (int64_t)n * h * w;
  const int64_t total = pixels * G;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = (i / 32 / G) * 32 + (i % 32);        // lanes = consecutive pixels
    const int g = (int)((i / 32) % G);
    if (pix >= pixels) continue;
    const int xx = (int)(pix % w);
    const int yy = (int)((pix / w) % h);
    const int b = (int)(pix / ((int64_t)w * h));
    float in[KK];
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int sy = yy + t / 3 - 1, sx = xx + t % 3 - 1;
      const bool ok = sy >= 0 && sy < h && sx >= 0 && sx < w;
#pragma unroll
      for (int ci = 0; ci < CIN; ++ci)
        in[t * CIN + ci] = ok ? __bfloat162float(x[(((int64_t)b * h + sy) * w + sx) * CIN + ci]) : 0.f;
    }
#pragma unroll 1
    for (int k0 = 0; k0 < 32; k0 += 8) {
      float o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int co = g * 32 + k0 + k;
        const float* wr = s_w + co * KK;
        float acc = s_w[cout * KK + co];
#pragma unroll
        for (int q = 0; q < KK; ++q) acc = fmaf(in[q], wr[q], acc);
        o[k] = acc;
      }
      store8(y + pix * cout + g * 32 + k0, o);
    }
  }
}

// conv_out: cout = COUT (<= 8), cin multiple of 8. Thread = output pixel;
// weights [cout][9][cin] in shared memory (broadcast reads).
template <int COUT>
__global__ void __launch_bounds__(256)
conv_small_out_kernel(const bf16* __restrict__ x, int n, int h, int w, int cin, const float* __restrict__ wgt,
                      const float* __restrict__ bias, void* __restrict__ y, int y_f32) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float s_w[];
  const int KK = 9 * cin;
  for (int i = threadIdx.x; i < COUT * KK; i += blockDim.x) s_w[i] = wgt[i];
  __syncthreads();
  const int64_t pixels = (int64_t)n * h * w;
  const int V = cin / 8;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < pixels;
       pix += (int64_t)gridDim.x * blockDim.x) {
    const int xx = (int)(pix % w);
    const int yy = (int)((pix / w) % h);
    const int b = (int)(pix / ((int64_t)w * h));
    float acc[COUT];
#pragma unroll
    for (int co = 0; co < COUT; ++co) acc[co] = bias ? bias[co] : 0.f;
    for (int t = 0; t < 9; ++t) {
      const int sy = yy + t / 3 - 1, sx = xx + t % 3 - 1;
      if (sy < 0 || sy >= h || sx < 0 || sx >= w) continue;
      const bf16* src = x + (((int64_t)b * h + sy) * w + sx) * cin;
#pragma unroll 2
      for (int j = 0; j < V; ++j) {
        float v[8];
        load8(src + j * 8, v);
#pragma unroll
        for (int co = 0; co < COUT; ++co) {
          const float4* w4 = reinterpret_cast<const float4*>(s_w + co * KK + t * cin + j * 8);
          const float4 wa = w4[0], wb = w4[1];
          float a = acc[co];
          a = fmaf(v[0], wa.x, a); a = fmaf(v[1], wa.y, a); a = fmaf(v[2], wa.z, a); a = fmaf(v[3], wa.w, a);
          a = fmaf(v[4], wb.x, a); a = fmaf(v[5], wb.y, a); a = fmaf(v[6], wb.z, a); a = fmaf(v[7], wb.w, a);
          acc[co] = a;
        }
      }
    }
#pragma unroll
    for (int co = 0; co < COUT; ++co) {
      if (y_f32) static_cast<float*>(y)[pix * COUT + co] = acc[co];
      else static_cast<bf16*>(y)[pix * COUT + co] = __float2bfloat16_rn(acc[co]);
    }
  }
}

__global__ void timestep_emb_kernel(const float* __restrict__ t, int b, int dim, float max_period,
                                    float* __restrict__ out) {
  const int half = dim / 2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < b * half; i += gridDim.x * blockDim.x) {
    const int r = i / half, k = i - r * half;
    const float freq = expf(-logf(max_period) * (float)k / (float)half);
    const float arg = t[r] * freq;
    out[(int64_t)r * dim + k] = cosf(arg);          // flip_sin_to_cos: [cos, sin]
    out[(int64_t)r * dim + half + k] = sinf(arg);
  }
}

// y[m, n] = act_out(sum_k act_in(x[m, k]) * W[n, k] + bias[n]); one warp per (n), all M rows
constexpr int kSmallMaxM = 8;
__global__ void __launch_bounds__(256, 4) linear_small_kernel(const float* __restrict__ x, int M, int K, const bf16* __restrict__ w,
                                    const float* __restrict__ bias, int N, int act_in, int act_out,
                                    float* __restrict__ y) {
  extern __shared__ __align__(16) float xs[];          // [M][K] inputs, act_in applied once per block
  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const float v = x[i];
    xs[i] = act_in == HP_ACT_SILU ? silu(v) : v;
  }
  __syncthreads();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int n = warp; n < N; n += nwarps) {
    float acc[kSmallMaxM] = {0};
    const bf16* wr = w + (int64_t)n * K;
    // up to eight 16-byte weight loads in flight per lane (kept packed: 4 registers each):
    // a K <= 2048 row is one round trip
    for (int k0 = lane * 8; k0 < K; k0 += 8 * 256) {
      uint4 wq[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u * 256 < K) wq[u] = *reinterpret_cast<const uint4*>(wr + k0 + u * 256);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u * 256;
        if (k >= K) break;
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&wq[u]);
        float wv[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          wv[2 * i] = f.x;
          wv[2 * i + 1] = f.y;
        }
#pragma unroll
        for (int m = 0; m < kSmallMaxM; ++m) {
          if (m >= M) break;
          const float4 a0 = *reinterpret_cast<const float4*>(xs + m * K + k);
          const float4 a1 = *reinterpret_cast<const float4*>(xs + m * K + k + 4);
          float a = acc[m];
          a = fmaf(a0.x, wv[0], a); a = fmaf(a0.y, wv[1], a);
          a = fmaf(a0.z, wv[2], a); a = fmaf(a0.w, wv[3], a);
          a = fmaf(a1.x, wv[4], a); a = fmaf(a1.y, wv[5], a);
          a = fmaf(a1.z, wv[6], a); a = fmaf(a1.w, wv[7], a);
          acc[m] = a;
        }
      }
    }
#pragma unroll
    for (int m = 0; m < kSmallMaxM; ++m) {
      if (m >= M) break;
      float r = hp_warp_sum_f(acc[m]);
      if (lane == 0) {
        r += bias ? bias[n] : 0.f;
        if (act_out == HP_ACT_SILU) r = silu(r);
        y[(int64_t)m * N + n] = r;
      }
    }
  }
}

__global__ void patchify_kernel(const bf16* __restrict__ x, int n, int h, int w, int c, int p, int inverse,
                                bf16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  // token t = (ty, tx); feature f = (py * p + px) * c + ch
  const int64_t total = (int64_t)n * h * w * c;
  const int tw = w / p;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % c);
    int64_t pix = i / c;
    const int xx = (int)(pix % w);
    const int yy = (int)((pix / w) % h);
    const int b = (int)(pix / ((int64_t)w * h));
    const int64_t tok = ((int64_t)b * (h / p) + yy / p) * tw + xx / p;
    const int64_t f = ((int64_t)(yy % p) * p + (xx % p)) * c + ch;
    const int64_t ti = tok * ((int64_t)p * p * c) + f;
    if (!inverse) y[ti] = x[i];
    else y[i] = x[ti];
  }
}

__global__ void add_rows_kernel(const bf16* __restrict__ x, const bf16* __restrict__ add, int64_t rows,
                                int64_t add_rows, int c, bf16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int V = c / 8;
  const int64_t total = rows * V;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / V;
    const int j = (int)(i - r * V);
    float a[8], b[8];
    load8(x + r * c + j * 8, a);
    load8(add + (r % add_rows) * c + j * 8, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] += b[k];
    store8(y + r * c + j * 8, a);
  }
}

__global__ void gated_residual_kernel(bf16* __restrict__ x, const bf16* __restrict__ yv,
                                      const bf16* __restrict__ gate, int64_t ldg, int64_t rows, int c,
                                      int64_t rows_per_batch) {
  pdl_wait();
  pdl_trigger();
  const int V = c / 8;
  const int64_t total = rows * V;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / V;
    const int j = (int)(i - r * V);
    const int64_t b = r / rows_per_batch;
    float a[8], v[8], g[8];
    load8(x + r * c + j * 8, a);
    load8(yv + r * c + j * 8, v);
    load8(gate + b * ldg + j * 8, g);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] += g[k] * v[k];
    store8(x + r * c + j * 8, a);
  }
}

__global__ void copy_cols_kernel(const bf16* __restrict__ x, int64_t ldx, int c_src, int64_t rows,
                                 bf16* __restrict__ y, int64_t ldy, int c_dst) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = rows * c_dst;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / c_dst;
    const int j = (int)(i - r * c_dst);
    y[r * ldy + j] = j < c_src ? x[r * ldx + j] : __float2bfloat16_rn(0.f);
  }
}

// one CTA per row; the row stays in registers between the max, sum and write passes
constexpr int kSmThreads = 512;
constexpr int kSmMaxPerThread = 64;     // cols <= 512 * 64 = 32768
__global__ void __launch_bounds__(kSmThreads)
softmax_rows_kernel(const bf16* __restrict__ x, int64_t ldx, int cols, float scale2, bf16* __restrict__ y,
                    int64_t ldy) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[kSmThreads / 32];
  const bf16* xr = x + (int64_t)blockIdx.x * ldx;
  bf16* yr = y + (int64_t)blockIdx.x * ldy;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float v[kSmMaxPerThread];
  const int nv = cols / 8;                           // 8-element vectors, thread t owns t, t + 512, ...
  float mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < kSmMaxPerThread / 8; ++k) {
    const int j = threadIdx.x + k * kSmThreads;
    if (j < nv) {
      load8(xr + j * 8, v + k * 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[k * 8 + e] *= scale2;                      // log2 domain
        mx = fmaxf(mx, v[k * 8 + e]);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < kSmThreads / 32; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < kSmMaxPerThread / 8; ++k) {
    const int j = threadIdx.x + k * kSmThreads;
    if (j < nv) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[k * 8 + e] = exp2f(v[k * 8 + e] - mx);
        sum += v[k * 8 + e];
      }
    }
  }
  sum = hp_warp_sum_f(sum);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < kSmThreads / 32; ++w) tot += red[w];   // fixed order
  const float inv = 1.0f / tot;
#pragma unroll
  for (int k = 0; k < kSmMaxPerThread / 8; ++k) {
    const int j = threadIdx.x + k * kSmThreads;
    if (j < nv) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = v[k * 8 + e] * inv;
      store8(yr + j * 8, o);
    }
  }
}

__global__ void embed_tokens_kernel(const int64_t* __restrict__ ids, int64_t rows, int seq,
                                    const float* __restrict__ tok, const float* __restrict__ pos, int dim,
                                    bf16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = rows * dim;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dim;
    const int c = (int)(i - r * dim);
    y[i] = __float2bfloat16_rn(tok[ids[r] * dim + c] + pos[(r % seq) * dim + c]);
  }
}

__global__ void cast_kernel(const bf16* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __bfloat162float(x[i]);
}

inline int ok() { return cudaGetLastError() == cudaSuccess ? HP_OK : HP_ERR_CUDA; }

// barrier words of the single-launch GroupNorm: [image][count, generation]. A slot is
// zeroed once when the pool is made and left consistent by every use (the last
// arriver resets the count), so only CONCURRENT launches must not share one: eager
// launches take one slot per stream (launches on a stream are ordered: each
// gn_fused_kernel waits for its predecessor with griddepcontrol.wait before it
// arrives), every launch captured into a CUDA graph a slot of its own (graph replays
// on different streams may overlap). Pools are per device; an exhausted pool sends
// the launch to the two-kernel path.
constexpr int kGnMaxImages = 64;
constexpr int kGnSlotWords = 2 * kGnMaxImages;
constexpr int kGnSlots = 4096;
struct GnBarPool {
  unsigned* base = nullptr;
  int next = 0;
  std::unordered_map<cudaStream_t, unsigned*> per_stream;
};
unsigned* gn_bar_slot(cudaStream_t st, bool capturing) {
  static std::mutex mu;
  static std::unordered_map<int, GnBarPool> pools;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  GnBarPool& pool = pools[dev];
  if (!pool.base) {
    if (capturing) return nullptr;                 // no allocation inside a capture
    const size_t bytes = (size_t)kGnSlots * kGnSlotWords * sizeof(unsigned);
    if (cudaMalloc(&pool.base, bytes) != cudaSuccess) { pool.base = nullptr; return nullptr; }
    if (cudaMemset(pool.base, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return nullptr;
  }
  if (!capturing) {
    auto it = pool.per_stream.find(st);
    if (it != pool.per_stream.end()) return it->second;
  }
  if (pool.next >= kGnSlots) return nullptr;
  unsigned* slot = pool.base + (size_t)(pool.next++) * kGnSlotWords;
  if (!capturing) pool.per_stream[st] = slot;
  return slot;
}

constexpr size_t kGnSmemMax = 112 * 1024;   // staged chunk + scratch limit: two CTAs per SM
constexpr size_t kGnSmemMin = 16 * 1024;    // smaller chunks: direct loads are faster

// 0: two-kernel path; 1: single launch reading global memory; 2: single launch with the
// chunk staged in shared memory (`smem` bytes)
int gn_fused_mode(int ctas, size_t smem) {
  static bool disabled = getenv("HP_GN_FUSED") && getenv("HP_GN_FUSED")[0] == '0';
  static bool no_smem = getenv("HP_GN_SMEM") && getenv("HP_GN_SMEM")[0] == '0';
  if (disabled) return 0;
  static int sms = 0;
  static bool attr = false;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    attr = cudaFuncSetAttribute(gn_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kGnSmemMax) == cudaSuccess;
  }
  // every CTA resident: checked here, and the launch is cooperative (the driver
  // refuses it rather than run it partially resident, e.g. under MPS limits)
  int per_sm = 0;
  if (!no_smem && attr && smem <= kGnSmemMax &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gn_fused_kernel<true>, kGnThreads, smem) ==
          cudaSuccess &&
      ctas <= per_sm * sms)
    return 2;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gn_fused_kernel<false>, kGnThreads, 0) == cudaSuccess &&
      ctas <= per_sm * sms)
    return 1;
  return 0;
}

}  // namespace

extern "C" {

int hp_group_norm(const void* x1, int32_t c1, const void* x2, int32_t c2, int32_t n, int64_t hw, int32_t groups,
                  float eps, const float* gamma, const float* beta, int32_t do_silu, void* y, float* stats,
                  void* stream) {
  const int C = c1 + (x2 ? c2 : 0);
  if (!x1 || !y || !gamma || !beta || !stats) return HP_ERR_PARAMETER;
  if (C % 8 || c1 % 8 || C > kMaxC || groups < 1 || groups > 64 || C % groups || n < 1 || hw < 1) return HP_ERR_SHAPE;
  if (!a16(x1) || (x2 && !a16(x2)) || !a16(y)) return HP_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the pixel partition depends on hw only (never on the batch size n), so one
  // image's statistics are bit-identical whatever else is in the batch
  int splits = hw < 128 ? (int)hw : 128;
  // stage the chunk in shared memory when it is large enough for the bulk copies to pay
  static const size_t smem_min = [] {        // development probe: HP_GN_SMEM_MIN=<bytes>
    const char* e = getenv("HP_GN_SMEM_MIN");
    return e ? (size_t)atol(e) : kGnSmemMin;
  }();
  const bool stage = gn_chunk_bytes(hw, splits, C) >= smem_min;
  const size_t smem = gn_smem_bytes(hw, splits, C);
  int mode = n <= kGnMaxImages ? gn_fused_mode(n * splits, stage ? smem : kGnSmemMax + 1) : 0;
  unsigned* bar = nullptr;
  if (mode) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return HP_ERR_CUDA;
    bar = gn_bar_slot(st, cs != cudaStreamCaptureStatusNone);
    if (!bar) mode = 0;
  }
  if (mode) {
    const auto kern = mode == 2 ? gn_fused_kernel<true> : gn_fused_kernel<false>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(splits, n);
    cfg.blockDim = dim3(kGnThreads);
    cfg.dynamicSmemBytes = mode == 2 ? smem : 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = hp_pdl_enabled() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<const bf16*>(x1), c1,
                                             static_cast<const bf16*>(x2), x2 ? c2 : 0, hw, groups, splits, stats,
                                             eps, gamma, beta, do_silu, static_cast<bf16*>(y), bar);
    if (e == cudaSuccess) return ok();
    if (e != cudaErrorCooperativeLaunchTooLarge) return HP_ERR_CUDA;
    (void)cudaGetLastError();                      // refused (not co-resident): two-kernel path
  }
  hp_launch_pdl(gn_stats_kernel, dim3(splits, n), dim3(kGnThreads), 0, st, static_cast<const bf16*>(x1), c1,
                                                          static_cast<const bf16*>(x2), x2 ? c2 : 0, hw, groups,
                                                          splits, stats);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  const int64_t per_img = hw * (C / 8);
  int chunks = nblocks(per_img, kGnThreads * 8, 4096);
  hp_launch_pdl(gn_apply_kernel, dim3(chunks, n), dim3(kGnThreads), 0, st, static_cast<const bf16*>(x1), c1,
                                                          static_cast<const bf16*>(x2), x2 ? c2 : 0, hw, groups,
                                                          splits, stats, eps, gamma, beta, do_silu,
                                                          static_cast<bf16*>(y));
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_group_norm_parts(const void* x, int32_t c, int32_t n, int64_t hw, const float* part1, int32_t c1,
                        const float* part2, int32_t groups, float eps, const float* gamma, const float* beta,
                        int32_t do_silu, void* y, void* stream) {
  if (!x || !y || !gamma || !beta || !part1 || (c1 < c && !part2)) return HP_ERR_PARAMETER;
  if (c % 8 || c > kMaxC || groups < 1 || groups > 64 || c % groups || (c / groups) % kGnPartSeg ||
      c1 % kGnPartSeg || c1 < 1 || c1 > c || n < 1 || hw < kGnPartRows || hw % kGnPartRows)
    return HP_ERR_SHAPE;
  if (!a16(x) || !a16(y) || (reinterpret_cast<uintptr_t>(part1) & 7) || (reinterpret_cast<uintptr_t>(part2) & 7))
    return HP_ERR_UNSUPPORTED;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // block = whole pixel rows of V = c / 8 threads (~256); every CTA folds its image's
  // partials first, so the grid stays near two CTAs per SM (and >= 4 pixels per thread)
  const int V = c / 8;
  const int rows = V >= HP_GN_PARTS_THREADS ? 1 : (HP_GN_PARTS_THREADS + V / 2) / V;
  const int threads = rows * V;
  if (threads > kGnPartsMaxThreads) return HP_ERR_SHAPE;
  int chunks = (int)((hw + kGnPartsDepth * rows - 1) / (kGnPartsDepth * rows));
  const int cap = (HP_GN_PARTS_CTAS_PER_SM * sms + n - 1) / n;
  if (chunks > cap) chunks = cap;
  hp_launch_pdl(gn_parts_kernel, dim3(chunks, n), dim3(threads), 0, static_cast<cudaStream_t>(stream),
                static_cast<const bf16*>(x), (int)c, hw, reinterpret_cast<const float2*>(part1), (int)c1,
                reinterpret_cast<const float2*>(part2), (int)groups, eps, gamma, beta, (int)do_silu,
                static_cast<bf16*>(y));
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_layer_norm(const void* x, int64_t rows, int32_t c, float eps, const float* gamma, const float* beta,
                  const void* shift, const void* scale, int64_t ldm, int64_t rows_per_batch, void* y, void* stream) {
  if (!x || !y) return HP_ERR_PARAMETER;
  if (c % 8 || c > 32 * 8 * kLnVec || rows < 1) return HP_ERR_SHAPE;
  if ((shift || scale) && (rows_per_batch < 1 || ldm % 8)) return HP_ERR_PARAMETER;
  launch_ln(static_cast<cudaStream_t>(stream), static_cast<const bf16*>(x), rows, c, eps, gamma, beta,
            static_cast<const float*>(shift), static_cast<const float*>(scale), ldm, rows_per_batch,
            static_cast<bf16*>(y), nullptr, nullptr, -1);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_layer_norm_joint(const void* x, int64_t rows, int32_t c, float eps, const float* shift, const float* scale,
                        const float* shift2, const float* scale2, int64_t ldm, int64_t rows_per_batch, int64_t split,
                        void* y, void* stream) {
  if (!x || !y || !shift || !scale || !shift2 || !scale2) return HP_ERR_PARAMETER;
  if (c % 8 || c > 32 * 8 * kLnVec || rows < 1 || rows_per_batch < 1 || split < 0 || ldm % 8) return HP_ERR_SHAPE;
  launch_ln(static_cast<cudaStream_t>(stream), static_cast<const bf16*>(x), rows, c, eps, nullptr, nullptr, shift,
            scale, ldm, rows_per_batch, static_cast<bf16*>(y), shift2, scale2, split);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_quick_gelu(const void* x, void* y, int64_t n, void* stream) {
  if (!x || !y || n % 8) return HP_ERR_PARAMETER;
  hp_launch_pdl(quick_gelu_kernel, dim3(nblocks(n / 8, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream),
                static_cast<const bf16*>(x), static_cast<bf16*>(y), n / 8);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_silu(const void* x, void* y, int64_t n, void* stream) {
  if (!x || !y || n % 8) return HP_ERR_PARAMETER;
  hp_launch_pdl(silu_kernel, dim3(nblocks(n / 8, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), static_cast<const bf16*>(x),
                                                                                   static_cast<bf16*>(y), n / 8);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_upsample2x(const void* x, int32_t n, int32_t h, int32_t w, int32_t c, void* y, void* stream) {
  if (!x || !y || c % 8) return HP_ERR_PARAMETER;
  const int64_t total = (int64_t)n * 4 * h * w * (c / 8);
  hp_launch_pdl(upsample2x_kernel, dim3(nblocks(total, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(x), n, h, w, c, static_cast<bf16*>(y));
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_embed_tokens(const int64_t* ids, int64_t rows, int32_t seq, const float* tok, const float* pos, int32_t dim,
                    void* y, void* stream) {
  if (!ids || !tok || !pos || !y || rows < 0 || seq < 1 || dim < 1) return HP_ERR_PARAMETER;
  if (rows == 0) return HP_OK;
  hp_launch_pdl(embed_tokens_kernel, dim3(nblocks(rows * dim, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream),
                ids, rows, seq, tok, pos, dim, static_cast<bf16*>(y));
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_softmax_rows(const void* x, int64_t ldx, int64_t rows, int32_t cols, float scale, void* y, int64_t ldy,
                    void* stream) {
  if (!x || !y || rows < 0 || cols < 8 || cols % 8 || cols > kSmThreads * kSmMaxPerThread || ldx % 8 || ldy % 8)
    return HP_ERR_PARAMETER;
  if (!a16(x) || !a16(y)) return HP_ERR_UNSUPPORTED;
  if (rows == 0) return HP_OK;
  hp_launch_pdl(softmax_rows_kernel, dim3((unsigned)rows), dim3(kSmThreads), 0, static_cast<cudaStream_t>(stream),
                static_cast<const bf16*>(x), ldx, cols, scale * 1.4426950408889634f, static_cast<bf16*>(y), ldy);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_copy_cols(const void* x, int64_t ldx, int32_t c_src, int64_t rows, void* y, int64_t ldy, int32_t c_dst,
                 void* stream) {
  if (!x || !y || c_src < 0 || c_dst < 1 || rows < 0 || ldx < c_src || ldy < c_dst) return HP_ERR_PARAMETER;
  const int64_t total = rows * c_dst;
  hp_launch_pdl(copy_cols_kernel, dim3(nblocks(total, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream),
                static_cast<const bf16*>(x), ldx, c_src, rows, static_cast<bf16*>(y), ldy, c_dst);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_concat_channels(const void* a, int32_t c1, const void* b, int32_t c2, int64_t pixels, void* y, void* stream) {
  if (!a || !b || !y || c1 % 8 || c2 % 8) return HP_ERR_PARAMETER;
  hp_launch_pdl(concat_kernel, dim3(nblocks(pixels * ((c1 + c2) / 8), 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(a), c1, static_cast<const bf16*>(b), c2, pixels, static_cast<bf16*>(y));
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_conv3x3_small(const void* x, int32_t n, int32_t h, int32_t w, int32_t cin, const float* wgt,
                     const float* bias, int32_t cout, void* y, int32_t y_is_f32, void* stream) {
  if (!x || !wgt || !y) return HP_ERR_PARAMETER;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cin == 4 && cout % 32 == 0 && !y_is_f32) {
    const size_t smem = (size_t)cout * (9 * cin + 1) * sizeof(float);
    if (smem > 200 * 1024) return HP_ERR_UNSUPPORTED;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(conv_small_in_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    const int64_t total = ((int64_t)n * h * w + 31) / 32 * 32 * (cout / 32);
    hp_launch_pdl(conv_small_in_kernel<4>, dim3(nblocks(total, 256, 148 * 8)), dim3(256), smem, st, static_cast<const bf16*>(x), n, h, w,
                                                                              wgt, bias, cout, static_cast<bf16*>(y));
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
    return ok();
  }
  if (cout == 4 && cin % 8 == 0) {
    const size_t smem = (size_t)cout * 9 * cin * sizeof(float);
    if (smem > 200 * 1024) return HP_ERR_UNSUPPORTED;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(conv_small_out_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    const int64_t pixels = (int64_t)n * h * w;
    hp_launch_pdl(conv_small_out_kernel<4>, dim3(nblocks(pixels, 128, 148 * 8)), dim3(128), smem, st, static_cast<const bf16*>(x), n, h, w,
                                                                                cin, wgt, bias, y, y_is_f32);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
    return ok();
  }
  return HP_ERR_UNSUPPORTED;
}

int hp_timestep_embedding(const float* t, int32_t b, int32_t dim, float max_period, float* out, void* stream) {
  if (!t || !out || dim % 2) return HP_ERR_PARAMETER;
  timestep_emb_kernel<<<nblocks((int64_t)b * dim / 2, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      t, b, dim, max_period, out);
  return ok();
}

int hp_linear_small(const float* x, int32_t M, int32_t K, const void* w, const float* bias, int32_t N,
                    int32_t act_in, int32_t act_out, float* y, void* stream) {
  if (!x || !w || !y) return HP_ERR_PARAMETER;
  if (M < 1 || M > kSmallMaxM || K % 8) return HP_ERR_SHAPE;
  const size_t smem = (size_t)M * K * sizeof(float);
  constexpr size_t kMaxSmem = 160 * 1024;
  if (smem > kMaxSmem) return HP_ERR_SHAPE;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(linear_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem) !=
        cudaSuccess)
      return HP_ERR_CUDA;
    attr = true;
  }
  hp_launch_pdl(linear_small_kernel, dim3(nblocks((int64_t)N * 32, 256, 148 * 8)), dim3(256), smem,
                static_cast<cudaStream_t>(stream), x, M, K, static_cast<const bf16*>(w), bias, N, act_in, act_out, y);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_patchify(const void* x, int32_t n, int32_t h, int32_t w, int32_t c, int32_t p, int32_t inverse, void* y,
                void* stream) {
  if (!x || !y || p < 1 || h % p || w % p) return HP_ERR_PARAMETER;
  hp_launch_pdl(patchify_kernel, dim3(nblocks((int64_t)n * h * w * c, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(x), n, h, w, c, p, inverse, static_cast<bf16*>(y));
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_add_rows(const void* x, const void* add, int64_t rows, int64_t add_rows, int32_t c, void* y, void* stream) {
  if (!x || !add || !y || c % 8 || add_rows < 1) return HP_ERR_PARAMETER;
  hp_launch_pdl(add_rows_kernel, dim3(nblocks(rows * (c / 8), 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(x), static_cast<const bf16*>(add), rows, add_rows, c, static_cast<bf16*>(y));
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_gated_residual(void* x, const void* y, const void* gate, int64_t ldg, int64_t rows, int32_t c,
                      int64_t rows_per_batch, void* stream) {
  if (!x || !y || !gate || c % 8 || rows_per_batch < 1 || ldg % 8) return HP_ERR_PARAMETER;
  hp_launch_pdl(gated_residual_kernel, dim3(nblocks(rows * (c / 8), 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<bf16*>(x), static_cast<const bf16*>(y), static_cast<const bf16*>(gate), ldg, rows, c,
      rows_per_batch);
  if (cudaPeekAtLastError() != cudaSuccess) return HP_ERR_CUDA;
  return ok();
}

int hp_cast_bf16_f32(const void* x, float* y, int64_t n, void* stream) {
  if (!x || !y) return HP_ERR_PARAMETER;
  cast_kernel<<<nblocks(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const bf16*>(x), y, n);
  return ok();
}

}  // extern "C"
