// hp_gemm.cu — K4: persistent warp-specialised tcgen05 GEMM for the denoiser.
//
//   D[M, N] = epilogue( alpha * A[M, K] . B[N, K]^T )
//
// A is a plain row-major activation matrix or an NHWC activation read as an
// implicit GEMM: 3x3 convolutions walk 9 taps x (Cin/64) channel blocks, each A
// tile one 4-D TMA box of the input shifted by the tap (TMA zero-fills the
// halo; stride 2 via TMA element strides); HP_A_UPCONV runs nearest-2x +
// 3x3 conv as four sub-pixel 2x2 convs (one per output phase, as batch
// entries). B is the K-major weight [N, K] (conv weights [Cout][taps][Cin]).
// No im2col buffer exists.
//
// Kernels:
//   gemm_kernel        one CTA per 128-row tile (M <= 128, and the cluster-LN mode)
//   gemm_pair_kernel   CTA pair (cta_group::2): 256-row tiles, each CTA loads its A
//                      rows and half of B; widths 64..320 (320 = two N=160 MMAs)
//   gemm_splitk_kernel two CTA pairs of a 4-CTA cluster split K of one 256x320 tile
//                      and exchange accumulator halves through DSMEM
// Roles (256 threads, 1 CTA/SM, persistent over output tiles):
//   warp 0      TMA producer   (smem ring of STAGES {A 128x64, B x64} tiles, SW128)
//   warp 1      MMA issuer     (tcgen05.mma; fp32 accumulators in TMEM)
//   warp 2      TMEM allocator (up to 4 accumulator buffers)
//   warps 4..7  epilogue       (tcgen05.ld 32x32b -> bias / per-image bias / residual /
//                               GELU / SiLU / GEGLU / column gate / LayerNorm fold or
//                               statistics -> 256-bit bf16 stores)
// The epilogue of tile i overlaps the MMAs of tile i+1 through the TMEM buffers;
// TMA runs STAGES k-blocks ahead of the tensor core. Activation and epilogue
// flavour are template parameters (each runtime branch in the unrolled epilogue
// costs the common case).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <mutex>
#include "hybridpar_b200_denoiser.h"
#include "hp_common.cuh"
#include "hp_tc.cuh"

using namespace hptc;

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;
constexpr uint32_t kABytes = BM * BK * 2;  // 16 KB

struct GemmParams {
  int M, N, K;
  int num_kb;
  int mode;          // HP_A_*
  int cin_blocks;    // conv: Cin / 64
  int out_h, out_w;  // conv output spatial size
  int box_w, box_h;  // conv tile (output pixels)
  int num_m_tiles, num_n_tiles;
  __nv_bfloat16* d; long long ldd;
  const float* bias;
  const float* bias2; long long bias2_div; long long bias2_ld;
  // fused LayerNorm of the output rows (cluster of all N tiles of a 128-row block)
  int ln_mode;
  const float* ln_g; const float* ln_b; float ln_eps;
  __nv_bfloat16* ln_y; long long ldy;
  const __nv_bfloat16* res; long long ldr;
  int act;
  int probe_noepi;
  int raster_n;                    // pair kernel tile order: 1 = N tiles fastest                 // dev probe (HP_GEMM_PROBE_NOEPI=1): skip the plain epilogue's stores
  float alpha;
  const float* colscale;
  int batch;                       // >= 1; plain mode only
  long long a_bs, d_bs, r_bs, cs_bs;  // element strides between batches
  // HP_A_UPCONV: batch index = output phase (py, px) = (bt >> 1, bt & 1), D offset
  // py * d_bs + px * d_bs2; rows map to the 2x grid: row = q * row_w + j ->
  // q * ld_hi + j * ldd (row_w = 0: ordinary rows)
  long long d_bs2, ld_hi;
  int row_w;
  // LayerNorm folding: producer writes per-(row, N tile) (mean, M2); consumer folds
  bool vec256;                     // output (and residual) rows 32-byte aligned: 256-bit accesses
  float2* stats_out;
  const float2* ln_stats; int ln_parts; float ln_part_n; const float* ln_colsum; float ln_fold_eps;
  // GroupNorm partials of the output (kEpiGn): (sum, sum of squares) per 128-row block and
  // 10-column segment at gn_part[idx * gn_ld + segment], idx = image * gn_P + block of the
  // image (upconv: phase-major within the image); gn_rows = rows per image per batch slice
  float2* gn_part; int gn_rows; int gn_P; int gn_ld;
  // GEGLU pair kernel, last partial wave (tiles_eff > 0): tiles [tail_full, num_tiles) run as
  // two half-width tiles each (64 outputs: 64 linear + 64 gate columns), tiles_eff in all
  int tail_full, tiles_eff;
};

// mean / rstd of one row from its (mean, M2) partials, Chan's pairwise update in
// a fixed order (deterministic, no E[x^2] - E[x]^2 cancellation)
constexpr int kMaxFoldParts = 16;
__device__ __forceinline__ void fold_row_stats(const GemmParams& p, int row, float& mean, float& rstd) {
  const float2* s = p.ln_stats + (long long)row * p.ln_parts;
  float2 v[kMaxFoldParts];
#pragma unroll
  for (int t = 0; t < kMaxFoldParts; ++t)          // all partial loads in flight at once
    if (t < p.ln_parts) v[t] = __ldg(s + t);
  float n = 0.f, mu = 0.f, m2 = 0.f;
#pragma unroll
  for (int t = 0; t < kMaxFoldParts; ++t) {
    if (t < p.ln_parts) {
      const float nn = n + p.ln_part_n;
      const float w = __fdividef(p.ln_part_n, nn);
      const float delta = v[t].x - mu;
      mu = fmaf(delta, w, mu);
      m2 += v[t].y + delta * delta * (n * w);
      n = nn;
    }
  }
  mean = mu;
  rstd = rsqrtf(fmaxf(m2, 0.f) / n + p.ln_fold_eps);
}

// pull this thread's residual row segment into L1 before the accumulator is ready
template <int BN>
__device__ __forceinline__ void prefetch_res_row(const GemmParams& p, int bt, int row, int n0) {
  if (!p.res || row >= p.M || p.act == HP_ACT_GEGLU) return;
  const char* r = reinterpret_cast<const char*>(p.res + (p.batch > 1 ? (long long)bt * p.r_bs : 0) +
                                                (long long)row * p.ldr + n0);
#pragma unroll
  for (int off = 0; off < BN * 2; off += 128) asm volatile("prefetch.global.L1 [%0];" :: "l"(r + off));
}

// epilogue flavours (one template instance each, chosen per launch)
constexpr int kEpiPlain = 0, kEpiStats = 1, kEpiFold = 2, kEpiGn = 3;
constexpr int kGnSeg = 10;     // GroupNorm partial segment (columns): divides every SDXL group width

// kEpiGn: GroupNorm partials of the STORED bf16 values, one (sum, sum of squares) per
// 10-column segment over the CTA's 128 rows. Each thread runs its row through the segment
// in column order (carried across 32-column chunks), a warp sums its 32 rows with a fixed
// xor tree, the four warps' sums meet in shared memory in fixed order: a segment's value
// depends on its columns and its 128-row block only, not on block_n, split-K or the rest
// of the batch (hp_group_norm_parts folds them per image: batch-invariant). PH = the
// 32-column chunk's index mod 5 (its first column mod 10 is 2 PH; tiles start at
// multiples of 160); seg0 = the tile segment of the chunk's 5-chunk group.
template <int PH>
__device__ __forceinline__ void gn_chunk(const uint32_t (&w)[16], float& s1, float& s2, float2* gsm, int quarter,
                                         int lane, int seg0) {
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float2 f = unpack_bf16(w[j >> 1]);
    const float v = (j & 1) ? f.y : f.x;
    s1 += v;
    s2 = fmaf(v, v, s2);
    if ((32 * PH + j) % kGnSeg == kGnSeg - 1) {
      float a = s1, b = s2;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      if (lane == 0) gsm[quarter * 32 + seg0 + (32 * PH + j) / kGnSeg] = make_float2(a, b);
      s1 = 0.f;
      s2 = 0.f;
    }
  }
}

template <int BN>
__device__ __forceinline__ void decode_tile(const GemmParams& p, int tile, int& b, int& m0, int& n0) {
  if (p.ln_mode) {             // one cluster = every N tile of one 128-row block
    b = 0;
    m0 = (tile / p.num_n_tiles) * BM;
    n0 = (tile % p.num_n_tiles) * BN;
    return;
  }
  const int mt_all = p.num_m_tiles * p.batch;
  const int mt = tile % mt_all;
  b = mt / p.num_m_tiles;
  m0 = (mt - b * p.num_m_tiles) * BM;
  n0 = (tile / mt_all) * BN;
}

// exact-erf GELU x * Phi(x) with erf from Abramowitz-Stegun 7.1.26 (|erf error| <= 1.5e-7,
// GELU error <= 2.2e-7 abs): one MUFU.RCP + one MUFU.EX2 per value instead of erff.
// Packed pair: the polynomial / scaling on FFMA2/FMUL2, two MUFU each for the
// reciprocal and the exponential (0.5 folded into the coefficients).
__device__ __forceinline__ uint64_t gelu_erf2(uint64_t x2) {
  const float x0 = lo2(x2), x1 = hi2(x2);
  const uint64_t z2 = fmul2(pack2(fabsf(x0), fabsf(x1)), pack2(0.70710678118654752f, 0.70710678118654752f));
  const uint64_t d2 = ffma2(pack2(0.3275911f, 0.3275911f), z2, pack2(1.0f, 1.0f));
  float t0, t1;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t0) : "f"(lo2(d2)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t1) : "f"(hi2(d2)));
  const uint64_t t2 = pack2(t0, t1);
  uint64_t poly = ffma2(t2, pack2(0.5307027145f, 0.5307027145f), pack2(-0.7265760135f, -0.7265760135f));
  poly = ffma2(poly, t2, pack2(0.7107068705f, 0.7107068705f));
  poly = ffma2(poly, t2, pack2(-0.142248368f, -0.142248368f));
  poly = ffma2(poly, t2, pack2(0.127414796f, 0.127414796f));
  poly = fmul2(poly, t2);
  const uint64_t arg = fmul2(fmul2(z2, z2), pack2(-1.44269504088896341f, -1.44269504088896341f));
  float e0, e1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(lo2(arg)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(hi2(arg)));
  const uint64_t h = fmul2(x2, fmul2(poly, pack2(e0, e1)));     // 0.5 x (1 - erf(|x|/sqrt2))
  const float h0 = lo2(h), h1 = hi2(h);
  return pack2(x0 >= 0.f ? x0 - h0 : h0, x1 >= 0.f ? x1 - h1 : h1);
}

// 64 contiguous bytes of one output row: two 256-bit stores when 32-byte aligned
__device__ __forceinline__ void st_row64(__nv_bfloat16* dst, const uint32_t (&w)[16], bool v8) {
  if (v8) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(dst), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                    "r"(w[7]) : "memory");
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(dst + 16), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]),
                    "r"(w[14]), "r"(w[15]) : "memory");
  } else {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) d4[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
}
__device__ __forceinline__ void ld_row64(const __nv_bfloat16* src, uint32_t (&w)[16], bool v8) {
  if (v8) {
    asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(src));
    asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]),
                   "=r"(w[15])
                 : "l"(src + 16));
  } else {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 u = s4[q];
      w[4 * q] = u.x; w[4 * q + 1] = u.y; w[4 * q + 2] = u.z; w[4 * q + 3] = u.w;
    }
  }
}
__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + __expf(-x)); }

// Epilogue for one 128 x BN tile; thread = one output row. `sb` is the tile's
// column bias (bias + per-image bias2 folded) staged in shared memory, or null.
// Statistics segments (stats_out) are kStatW columns wide: the whole tile, except
// 320-wide tiles, which report two 160-column segments (so a split-K pair, where
// each CTA finalises one half, writes the same layout).
template <int BN> struct StatW { static constexpr int value = BN > 256 ? BN / 2 : BN; };

// element offset of output row `row` (once per thread and tile, not per element)
__device__ __forceinline__ long long d_row_off(const GemmParams& p, int row) {
  if (p.row_w == 0) return (long long)row * p.ldd;
  const int q = row / p.row_w;
  return (long long)q * p.ld_hi + (long long)(row - q * p.row_w) * p.ldd;
}
// the per-batch (per-phase) operand offsets of batch index bt
__device__ __forceinline__ void batch_offsets(GemmParams& q, int bt) {
  if (q.mode == HP_A_UPCONV) {
    q.d += (long long)(bt >> 1) * q.d_bs + (long long)(bt & 1) * q.d_bs2;
    return;
  }
  q.d += (long long)bt * q.d_bs;
  if (q.res) q.res += (long long)bt * q.r_bs;
  if (q.colscale) q.colscale += (long long)bt * q.cs_bs;
}

// Epilogue columns [c_begin, c_begin + c_count) of one 128 x BN tile (default: all);
// `red` (split-K) holds the other K half's fp32 partial for these columns in shared
// memory, laid out [column / 4][128 rows][4].
// Epilogue modes compiled into an instance: the unrolled epilogue is shared by
// every denoiser GEMM, and each runtime branch it carries costs the common case
// time (measured per U-Net forward: GELU + SiLU branches 0.4 ms; alpha, column
// gate and the 16-byte store fallback another 0.2 ms). "Lean" modes (no
// activation or GEGLU; alpha 1, no column gate, 32-byte-aligned rows) carry
// none of that; kAmAny handles everything at run time.
constexpr int kAmNone = 0, kAmGeglu = 1, kAmGelu = 2, kAmAny = 3, kAmGate = 4;
template <int BN, int EPI, int AM = kAmAny>
__device__ __forceinline__ void epilogue_tile(const GemmParams& p, uint32_t tmem_acc, int m0, int n0, int quarter,
                                              int lane, const float* sb, float* row_stats, const float* scs,
                                              float f_mean, float f_rstd, int c_begin = 0, int c_count = BN,
                                              const float4* red = nullptr, float2* gsm = nullptr, int gn_idx = 0,
                                              int geglu_half = -1) {
  constexpr bool kLean = AM != kAmAny;
  const bool v8 = kLean ? true : p.vec256;
  const int row = m0 + quarter * 32 + lane;
  const bool row_ok = row < p.M;
  const uint32_t lane_addr = tmem_acc + ((uint32_t)(quarter * 32) << 16);
  if (AM == kAmGeglu || (AM == kAmAny && p.act == HP_ACT_GEGLU)) {
    // tile columns [0, gw/2) are the linear halves, [gw/2, gw) the gates of the same gw/2
    // outputs (weights interleaved on the host per BN block); a half-width tail tile
    // (geglu_half = 0 / 1) holds outputs [64 h, 64 h + 64) of its block
    const int gw = geglu_half >= 0 ? BN / 2 : BN;
    const int out0 = n0 / 2 + (geglu_half > 0 ? BN / 4 : 0);
#pragma unroll 1
    for (int c = 0; c < gw / 64; ++c) {
      uint32_t ra[32], rg[32];
      tmem_ld_32x32b_x32(lane_addr + c * 32, ra);
      tmem_ld_32x32b_x32(lane_addr + gw / 2 + c * 32, rg);
      tmem_ld_wait();
      if (!row_ok) continue;
      const int ocol = out0 + c * 32;
      uint32_t packed[16];
      const bool scale = !kLean && p.alpha != 1.0f;
      const uint64_t alpha2 = pack2(p.alpha, p.alpha);
      const uint64_t nmean2 = pack2(-f_mean, -f_mean), rstd2 = pack2(f_rstd, f_rstd);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        uint64_t a2 = pack2u(ra[j], ra[j + 1]), g2 = pack2u(rg[j], rg[j + 1]);
        if (scale) { a2 = fmul2(a2, alpha2); g2 = fmul2(g2, alpha2); }
        if constexpr (EPI == kEpiFold) {
          const float2 ca = *reinterpret_cast<const float2*>(scs + c * 32 + j);
          const float2 cg = *reinterpret_cast<const float2*>(scs + gw / 2 + c * 32 + j);
          a2 = fmul2(rstd2, ffma2(nmean2, pack2(ca.x, ca.y), a2));
          g2 = fmul2(rstd2, ffma2(nmean2, pack2(cg.x, cg.y), g2));
        }
        if (sb) {
          const float2 ba = *reinterpret_cast<const float2*>(sb + c * 32 + j);
          const float2 bg = *reinterpret_cast<const float2*>(sb + gw / 2 + c * 32 + j);
          a2 = fadd2(a2, pack2(ba.x, ba.y));
          g2 = fadd2(g2, pack2(bg.x, bg.y));
        }
        const uint64_t o2 = fmul2(a2, gelu_erf2(g2));
        packed[j / 2] = pack_bf16(lo2(o2), hi2(o2));
      }
      if (kLean || p.probe_noepi != 2) st_row64(p.d + d_row_off(p, row) + ocol, packed, v8);
      else if (packed[0] == 0x7fc07fc0u) p.d[row] = __float2bfloat16(0.f);   // keep the math live
    }
    return;
  }
  constexpr int kStatW = StatW<BN>::value;
  const bool has_res = p.res != nullptr && row_ok;
  const __nv_bfloat16* res_row = has_res ? p.res + (long long)row * p.ldr + n0 + c_begin : nullptr;
  uint32_t rn[16];
  float st_sum = 0.f, st_sq = 0.f;            // LayerNorm partials of the stored (bf16) row
  float sh_k = 0.f, sh_s1 = 0.f, sh_s2 = 0.f;   // stats_out: sums shifted by the segment's first value
  float g_s1 = 0.f, g_s2 = 0.f;                 // kEpiGn: the open 10-column segment of this row
  if (has_res) ld_row64(res_row, rn, v8);
  const long long drow = d_row_off(p, row);
  const int nch = c_count / 32;
#pragma unroll 1
  for (int cc = 0; cc < nch; ++cc) {
    const int c = c_begin / 32 + cc;             // chunk index within the tile
    uint32_t r[32];
    tmem_ld_32x32b_x32(lane_addr + c * 32, r);
    uint32_t rc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) rc[q] = rn[q];
    if (has_res && cc + 1 < nch) ld_row64(res_row + (cc + 1) * 32, rn, v8);   // next chunk in flight
    tmem_ld_wait();
    if (!row_ok) continue;
    const int col = n0 + c * 32;
    // packed fp32 pairs throughout: v2[q] = columns (2q, 2q+1) of this chunk
    uint64_t v2[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v2[q] = pack2u(r[2 * q], r[2 * q + 1]);
    if (red) {                                   // split-K: add the other K half's partial
      const float4* rr = red + (size_t)(cc * 8) * 128 + quarter * 32 + lane;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = rr[q * 128];
        v2[2 * q] = fadd2(v2[2 * q], pack2(f.x, f.y));
        v2[2 * q + 1] = fadd2(v2[2 * q + 1], pack2(f.z, f.w));
      }
    }
    if (!kLean && p.alpha != 1.0f) {
      const uint64_t alpha2 = pack2(p.alpha, p.alpha);
#pragma unroll
      for (int q = 0; q < 16; ++q) v2[q] = fmul2(v2[q], alpha2);
    }
    if constexpr (EPI == kEpiFold) {
      const uint64_t nmean2 = pack2(-f_mean, -f_mean), rstd2 = pack2(f_rstd, f_rstd);
      const float4* c4 = reinterpret_cast<const float4*>(scs + c * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 cs = c4[q];
        v2[2 * q] = fmul2(rstd2, ffma2(nmean2, pack2(cs.x, cs.y), v2[2 * q]));
        v2[2 * q + 1] = fmul2(rstd2, ffma2(nmean2, pack2(cs.z, cs.w), v2[2 * q + 1]));
      }
    }
    if (sb) {
      const float4* b4 = reinterpret_cast<const float4*>(sb + c * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 b = b4[q];
        v2[2 * q] = fadd2(v2[2 * q], pack2(b.x, b.y));
        v2[2 * q + 1] = fadd2(v2[2 * q + 1], pack2(b.z, b.w));
      }
    }
    if constexpr (AM == kAmGelu) {
#pragma unroll
      for (int q = 0; q < 16; ++q) v2[q] = gelu_erf2(v2[q]);
    } else if constexpr (AM == kAmAny) {
      if (p.act == HP_ACT_GELU) {
#pragma unroll
        for (int q = 0; q < 16; ++q) v2[q] = gelu_erf2(v2[q]);
      } else if (p.act == HP_ACT_SILU) {
#pragma unroll
        for (int q = 0; q < 16; ++q) v2[q] = pack2(silu_f(lo2(v2[q])), silu_f(hi2(v2[q])));
      }
    }
    if (AM == kAmGate || (!kLean && p.colscale)) {
      const float4* g4 = reinterpret_cast<const float4*>(p.colscale + col);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 g = __ldg(g4 + q);
        v2[2 * q] = fmul2(v2[2 * q], pack2(g.x, g.y));
        v2[2 * q + 1] = fmul2(v2[2 * q + 1], pack2(g.z, g.w));
      }
    }
    if (has_res) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float2 f = unpack_bf16(rc[q]);
        v2[q] = fadd2(v2[q], pack2(f.x, f.y));
      }
    }
    uint32_t w[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) w[q] = pack_bf16(lo2(v2[q]), hi2(v2[q]));
    if (kLean || p.probe_noepi != 2) st_row64(p.d + drow + col, w, v8);
    else if (w[0] == 0x7fc07fc0u) p.d[row] = __float2bfloat16(0.f);          // keep the math live
    if constexpr (EPI == kEpiGn) {
      const int q5 = c / 5;
      switch (c - 5 * q5) {
        case 0: gn_chunk<0>(w, g_s1, g_s2, gsm, quarter, lane, 16 * q5); break;
        case 1: gn_chunk<1>(w, g_s1, g_s2, gsm, quarter, lane, 16 * q5); break;
        case 2: gn_chunk<2>(w, g_s1, g_s2, gsm, quarter, lane, 16 * q5); break;
        case 3: gn_chunk<3>(w, g_s1, g_s2, gsm, quarter, lane, 16 * q5); break;
        default: gn_chunk<4>(w, g_s1, g_s2, gsm, quarter, lane, 16 * q5); break;
      }
    }
    if constexpr (EPI == kEpiStats) {
      if ((c * 32) % kStatW == 0) sh_k = unpack_bf16(w[0]).x;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float2 f = unpack_bf16(w[e]);
        const float d0 = f.x - sh_k, d1 = f.y - sh_k;
        sh_s1 += d0 + d1;
        sh_s2 = fmaf(d0, d0, fmaf(d1, d1, sh_s2));
      }
      if ((c * 32 + 32) % kStatW == 0) {          // segment complete: (mean, M2) of its kStatW values
        const float inv_n = 1.0f / (float)kStatW;
        const int nseg = p.N / kStatW;
        p.stats_out[(long long)row * nseg + (n0 + c * 32) / kStatW] =
            make_float2(fmaf(sh_s1, inv_n, sh_k), fmaxf(sh_s2 - sh_s1 * sh_s1 * inv_n, 0.f));
        sh_s1 = 0.f;
        sh_s2 = 0.f;
      }
    }
    if (row_stats) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float2 f = unpack_bf16(w[e]);
        st_sum += f.x + f.y;
        st_sq = fmaf(f.x, f.x, fmaf(f.y, f.y, st_sq));
      }
    }
  }
  if (row_stats) {
    row_stats[0] = st_sum;
    row_stats[1] = st_sq;
  }
  if constexpr (EPI == kEpiGn) {
    // the tile's segments: the four row quarters summed in fixed order (epilogue warps only)
    asm volatile("bar.sync 2, 128;" ::: "memory");
    const int t = quarter * 32 + lane;
    if (t < c_count / kGnSeg) {
      const int sg = c_begin / kGnSeg + t;
      const float2 a = gsm[sg], b = gsm[32 + sg], c2 = gsm[64 + sg], d2 = gsm[96 + sg];
      p.gn_part[(long long)gn_idx * p.gn_ld + n0 / kGnSeg + sg] =
          make_float2(((a.x + b.x) + c2.x) + d2.x, ((a.y + b.y) + c2.y) + d2.y);
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
  }
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(const float* local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

// Second pass of the fused LayerNorm: row statistics of the full N from every
// CTA of the cluster (DSMEM), then y = (h - mean) * rstd * gamma + beta on this
// CTA's N tile, re-reading the h values this very thread just stored.
template <int BN>
__device__ __forceinline__ void ln_pass2(const GemmParams& p, int m0, int n0, int quarter, int lane,
                                         const float* s_stats) {
  const int row = m0 + quarter * 32 + lane;
  if (row >= p.M) return;
  uint32_t ncta;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
  const int r = quarter * 32 + lane;
  float ps[8], pq[8];
#pragma unroll
  for (uint32_t c = 0; c < 8; ++c) {               // independent DSMEM loads, all in flight
    ps[c] = c < ncta ? ld_dsmem_f32(s_stats + 2 * r, c) : 0.f;
    pq[c] = c < ncta ? ld_dsmem_f32(s_stats + 2 * r + 1, c) : 0.f;
  }
  float sum = 0.f, sq = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) { sum += ps[c]; sq += pq[c]; }
  const float mean = sum / (float)p.N;
  const float var = fmaxf(sq / (float)p.N - mean * mean, 0.f);
  const float rstd = rsqrtf(var + p.ln_eps);
  const uint4* src = reinterpret_cast<const uint4*>(p.d + (long long)row * p.ldd + n0);
  uint4* dst = reinterpret_cast<uint4*>(p.ln_y + (long long)row * p.ldy + n0);
  constexpr int kG = 4;                              // 4 x 16 B of h in flight per round trip
  static_assert((BN / 8) % kG == 0, "BN/8 must be a multiple of the load group");
#pragma unroll 1
  for (int q0 = 0; q0 < BN / 8; q0 += kG) {
    uint4 u[kG];
#pragma unroll
    for (int i = 0; i < kG; ++i) u[i] = src[q0 + i];
#pragma unroll
    for (int i = 0; i < kG; ++i) {
      const int q = q0 + i;
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(p.ln_g + n0 + q * 8));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(p.ln_g + n0 + q * 8 + 4));
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.ln_b + n0 + q * 8));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.ln_b + n0 + q * 8 + 4));
      const float2 x0 = unpack_bf16(u[i].x), x1 = unpack_bf16(u[i].y), x2 = unpack_bf16(u[i].z),
                   x3 = unpack_bf16(u[i].w);
      dst[q] = make_uint4(pack_bf16((x0.x - mean) * rstd * g0.x + b0.x, (x0.y - mean) * rstd * g0.y + b0.y),
                          pack_bf16((x1.x - mean) * rstd * g0.z + b0.z, (x1.y - mean) * rstd * g0.w + b0.w),
                          pack_bf16((x2.x - mean) * rstd * g1.x + b1.x, (x2.y - mean) * rstd * g1.y + b1.y),
                          pack_bf16((x3.x - mean) * rstd * g1.z + b1.z, (x3.y - mean) * rstd * g1.w + b1.w));
    }
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
  constexpr uint32_t kBBytes = BN * BK * 2;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  constexpr uint32_t kIdesc = idesc_bf16_f32(BM, BN);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias = reinterpret_cast<float*>(smem + STAGES * kStageBytes + 256);   // [2][BN]
  float* s_stats = sbias + 2 * BN;                                               // [128][2]
  float* scolsum = s_stats + 2 * BM;                                             // [2][BN] folded-LN column sums

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = p.num_m_tiles * p.batch * p.num_n_tiles;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();        // previous kernel's outputs (our A / residual) are complete from here on
  pdl_trigger();     // let the next kernel's CTAs start their prologue on idle SMs

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------ TMA producer ------------------------------
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int bt, m0, n0;
        decode_tile<BN>(p, tile, bt, m0, n0);
        int img = 0, y0 = 0, x0 = 0;
        if (p.mode != HP_A_PLAIN) {
          const int hw = p.out_h * p.out_w;
          img = m0 / hw;
          const int rem = m0 - img * hw;
          y0 = rem / p.out_w;
          x0 = rem - y0 * p.out_w;
        }
        for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], kStageBytes);
          uint8_t* a_dst = smA + s * kABytes;
          if (p.mode == HP_A_PLAIN) {
            if (p.batch > 1) tma_load_3d(a_dst, &tmA, &full[s], kb * BK, m0, bt);
            else tma_load_2d(a_dst, &tmA, &full[s], kb * BK, m0);
          } else {
            const int tap = kb / p.cin_blocks;
            const int cb = kb - tap * p.cin_blocks;
            const int dy = tap / 3, dx = tap - dy * 3;
            if (p.mode == HP_A_CONV3X3) {
              tma_load_4d(a_dst, &tmA, &full[s], cb * BK, x0 + dx - 1, y0 + dy - 1, img);
            } else {
              tma_load_4d(a_dst, &tmA, &full[s], cb * BK, 2 * x0 + dx - 1, 2 * y0 + dy - 1, img);
            }
          }
          tma_load_2d(smB + s * kBBytes, &tmB, &full[s], kb * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------ MMA issuer ------------------------------
      uint32_t it = 0, local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const uint32_t acc = local & 1;
        const uint32_t use = local >> 1;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t da = sdesc_sw128_kmajor(smA + s * kABytes);
          const uint64_t db = sdesc_sw128_kmajor(smB + s * kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // +32 bytes along K inside the 128-byte swizzle atom = +2 in the address field
            umma_bf16(d_tmem, da + 2 * k, db + 2 * k, kIdesc, (kb | k) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------ epilogue ------------------------------
    const int quarter = warp & 3;
    const int et = threadIdx.x - 128;                 // 0..127 across the 4 epilogue warps
    const bool any_bias = p.bias != nullptr || p.bias2 != nullptr;
    uint32_t local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const uint32_t acc = local & 1;
      const uint32_t use = local >> 1;
      int bt, m0, n0;
      decode_tile<BN>(p, tile, bt, m0, n0);
      float* sb = any_bias ? sbias + acc * BN : nullptr;
      float* scs = scolsum + acc * BN;
      const bool fold = p.ln_stats != nullptr;
      if (any_bias || fold) {
        // stage this tile's column bias (and folded-LN column sums) while the tensor
        // core is still busy; every row of a tile belongs to one image (bias2_div is a
        // multiple of 128)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const long long img = p.batch > 1 ? (long long)bt : (long long)(m0 / p.bias2_div);
        for (int i = et; i < BN; i += 128) {
          if (any_bias) {
            float b = p.bias ? __ldg(p.bias + n0 + i) : 0.0f;
            if (p.bias2) b += __ldg(p.bias2 + img * p.bias2_ld + n0 + i);
            sb[i] = b;
          }
          if (fold) scs[i] = __ldg(p.ln_colsum + n0 + i);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      // folded LayerNorm: this row's mean / rstd, also before the accumulator is ready
      float f_mean = 0.f, f_rstd = 1.f;
      const int my_row = m0 + quarter * 32 + lane;
      if (fold && my_row < p.M) fold_row_stats(p, my_row, f_mean, f_rstd);
      prefetch_res_row<BN>(p, bt, my_row, n0);     // residual lines in flight while the MMAs finish
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const uint32_t t_acc = tmem_base + acc * BN;
      if (p.batch > 1) {
        GemmParams q = p;
        q.d += (long long)bt * p.d_bs;
        if (q.res) q.res += (long long)bt * p.r_bs;
        if (q.colscale) q.colscale += (long long)bt * p.cs_bs;
        epilogue_tile<BN, kEpiPlain>(q, t_acc, m0, n0, quarter, lane, sb, nullptr, nullptr, 0.f, 1.f);
      } else if (fold) {
        epilogue_tile<BN, kEpiFold>(p, t_acc, m0, n0, quarter, lane, sb, nullptr, scs, f_mean, f_rstd);
      } else if (p.stats_out) {
        epilogue_tile<BN, kEpiStats>(p, t_acc, m0, n0, quarter, lane, sb, nullptr, nullptr, 0.f, 1.f);
      } else {
        epilogue_tile<BN, kEpiPlain>(p, t_acc, m0, n0, quarter, lane, sb,
                                     p.ln_mode ? s_stats + 2 * (quarter * 32 + lane) : nullptr, nullptr, 0.f, 1.f);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  if (p.ln_mode) {
    // every CTA of the cluster has published its per-row partial sums
    cluster_sync_all();
    if (warp >= 4) {
      int bt, m0, n0;
      decode_tile<BN>(p, blockIdx.x, bt, m0, n0);
      ln_pass2<BN>(p, m0, n0, warp & 3, lane, s_stats);
    }
    cluster_sync_all();   // nobody leaves while a peer may still read its partials
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<kTmemCols>(tmem_base);
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x BN tile. Each CTA TMA-loads its own 128 rows of A and HALF of the BN
// B rows (both complete on the leader's barrier); the leader's single thread
// issues M=256 MMAs that read A and B from both CTAs' shared memory and write
// each CTA's 128 x BN accumulator into its own TMEM. Per CTA and k-block the
// L2 traffic drops from (16 + BN/8) KB to (16 + BN/16) KB for the same MMA
// work: the 1-CTA kernel is L2-bandwidth-bound on B200 (LTS cap), this is not.
//   warp 0  TMA producer (both CTAs)   warp 1  MMA issuer (leader CTA)
//   warp 2  TMEM allocator (both)      warps 4..7  epilogue (both, own rows)
#ifdef HP_GEMM_TRACE
// per-launch event ring of the pair kernel's first cluster (tools/gemm_ring.py): globaltimer
// ns per event; [slot][0..8] events, [slot][9..12] M, N, K, block_n
constexpr int kRing = 4096;
__device__ unsigned long long g_gemm_ring[kRing][13];
__device__ unsigned int g_gemm_ctr;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HP_GTRACE(ev) do { if (blockIdx.x == 0 && g_slot >= 0) g_gemm_ring[g_slot % kRing][ev] = gtime(); } while (0)
#else
#define HP_GTRACE(ev) do {} while (0)
#endif
constexpr int kEpRuntime = -1;   // epilogue flavour chosen per tile at run time (kAmAny instances)
template <int BN, int STAGES, int AM, int EP>
__global__ void __launch_bounds__(kThreads, 1)
gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
  constexpr uint32_t kBHalfBytes = (BN / 2) * BK * 2;
  constexpr uint32_t kStageBytes = kABytes + kBHalfBytes;
  // BN > 256 (320): two N=160 MMAs per K step into adjacent TMEM columns. Shared memory
  // bandwidth (TMA writes + MMA operand reads) bounds narrow tiles; a 320-wide tile moves
  // 88 KB per 640 MMA cycles per SM where two 160-wide tiles move 104 KB.
  constexpr int kSub = BN > 256 ? 2 : 1;
  constexpr int kSubN = BN / kSub;
  constexpr uint32_t kSubBytes = (kSubN / 2) * BK * 2;
  // as many TMEM accumulator buffers as fit: the epilogue of one tile may lag the MMAs by
  // several tiles without stalling the tensor core
  constexpr int kAcc = BN > 256 ? 1 : (BN <= 128 ? 4 : (BN <= 170 ? 3 : 2));
  constexpr uint32_t kTmemCols = (kAcc * BN <= 64) ? 64 : (kAcc * BN <= 128) ? 128 : (kAcc * BN <= 256) ? 256 : 512;
  constexpr uint32_t kIdesc = idesc_bf16_f32(2 * BM, kSubN);
  constexpr uint32_t kIdescHalf = idesc_bf16_f32(2 * BM, kSubN / 2);   // GEGLU half-width tail tiles

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + kAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAcc);
  float* sbias = reinterpret_cast<float*>(smem + STAGES * kStageBytes + 256);   // [2][BN]
  float* scolsum = sbias + 2 * BN;                                               // [2][BN]
  float2* gsm = reinterpret_cast<float2*>(scolsum + 2 * BN);                    // [4][32] GroupNorm partials

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef HP_GEMM_TRACE
  __shared__ int s_slot;
  if (threadIdx.x == 0) s_slot = blockIdx.x == 0 ? (int)atomicAdd(&g_gemm_ctr, 1u) : -1;
  __syncthreads();
  const int g_slot = s_slot;
  if (threadIdx.x == 0 && g_slot >= 0) {
    g_gemm_ring[g_slot % kRing][9] = p.M; g_gemm_ring[g_slot % kRing][10] = p.N;
    g_gemm_ring[g_slot % kRing][11] = p.K; g_gemm_ring[g_slot % kRing][12] = BN;
  }
#endif
  if (threadIdx.x == 0) HP_GTRACE(0);
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1, num_clusters = gridDim.x >> 1;
  const int mp_all = p.num_m_tiles * p.batch;               // 256-row tiles (all batches)
  // GEGLU: the last partial wave may run as half-width tiles (p.tiles_eff, p.tail_full)
  const int num_tiles = (AM == kAmGeglu && p.tiles_eff) ? p.tiles_eff : mp_all * p.num_n_tiles;
  const int tail_full = (AM == kAmGeglu && p.tiles_eff) ? p.tail_full : num_tiles;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < kAcc; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_barrier();                 // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) HP_GTRACE(1);
  // the TMA producer (warp 0, lane 0) waits for the previous kernel only after it has
  // staged the weight (B) tiles of its first k-blocks: weights never depend on it
  if (threadIdx.x != 0) pdl_wait();
  pdl_trigger();

  auto decode = [&](int tile, int& bt, int& m0, int& n0, int& half) {
    half = -1;
    if (tile >= tail_full) {                 // GEGLU tail: tile = two half tiles
      half = (tile - tail_full) & 1;
      tile = tail_full + ((tile - tail_full) >> 1);
    }
    int mt, nt;
    if (p.raster_n) { nt = tile % p.num_n_tiles; mt = tile / p.num_n_tiles; }   // N fastest
    else { mt = tile % mp_all; nt = tile / mp_all; }                              // M fastest
    bt = mt / p.num_m_tiles;
    m0 = (mt - bt * p.num_m_tiles) * (2 * BM) + (int)rank * BM;   // this CTA's 128 rows
    n0 = nt * BN;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------ TMA producer (both CTAs) ------------------------------
      // B of the first tile's first k-blocks before the PDL wait (stage s = k-block s; the
      // stage's expect_tx covers A and B, A follows once the previous kernel is done)
      const int pre = cluster_id < num_tiles ? min(STAGES, p.num_kb) : 0;
      if (pre > 0) {
        int bt, m0, n0, half;
        decode(cluster_id, bt, m0, n0, half);
        const int nb = n0 + (int)rank * (kSubN / 2) + (p.mode == HP_A_UPCONV ? bt * p.N : 0) +
                       (half > 0 ? BN / 4 : 0);
        for (int kb = 0; kb < pre; ++kb) {
          if (leader) mbar_arrive_expect_tx(&full[kb], 2 * kStageBytes);
          const uint32_t fb = mapa_shared(&full[kb], 0);
#pragma unroll
          for (int sub = 0; sub < kSub; ++sub)
            tma_load_2d_pair(smB + kb * kBHalfBytes + sub * kSubBytes, &tmB, fb, kb * BK, nb + sub * kSubN);
        }
      }
      pdl_wait();
      HP_GTRACE(2);
      uint32_t it = 0;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int bt, m0, n0, half;
        decode(tile, bt, m0, n0, half);
        int img = 0, y0 = 0, x0 = 0;
        if (p.mode != HP_A_PLAIN) {
          const int hw = p.out_h * p.out_w;
          img = m0 / hw;
          const int rem = m0 - img * hw;
          y0 = rem / p.out_w;
          x0 = rem - y0 * p.out_w;
        }
        // a half tile loads the same 128-row B box from its 64 rows on (the MMA reads the
        // first 64 of each CTA's box: linear rows on the leader, gate rows on the peer)
        const int nb = n0 + (int)rank * (kSubN / 2) + (p.mode == HP_A_UPCONV ? bt * p.N : 0) +
                       (half > 0 ? BN / 4 : 0);
        for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          const bool staged = (int)it < pre;         // B already in flight, expect_tx done
          if (!staged) {
            mbar_wait(&empty[s], ph ^ 1);
            if (leader) mbar_arrive_expect_tx(&full[s], 2 * kStageBytes);
          }
          if (it == 0) HP_GTRACE(3);
          const uint32_t fb = mapa_shared(&full[s], 0);
          uint8_t* a_dst = smA + s * kABytes;
          if (p.mode == HP_A_PLAIN) {
            if (p.batch > 1) tma_load_3d_pair(a_dst, &tmA, fb, kb * BK, m0, bt);
            else tma_load_2d_pair(a_dst, &tmA, fb, kb * BK, m0);
          } else {
            const int tap = kb / p.cin_blocks;
            const int cb = kb - tap * p.cin_blocks;
            int dy, dx;
            if (p.mode == HP_A_UPCONV) {           // 2x2 taps shifted by the output phase
              dy = (tap >> 1) + (bt >> 1);
              dx = (tap & 1) + (bt & 1);
            } else {
              dy = tap / 3;
              dx = tap - dy * 3;
            }
            if (p.mode != HP_A_CONV3X3_S2) {
              tma_load_4d_pair(a_dst, &tmA, fb, cb * BK, x0 + dx - 1, y0 + dy - 1, img);
            } else {
              tma_load_4d_pair(a_dst, &tmA, fb, cb * BK, 2 * x0 + dx - 1, 2 * y0 + dy - 1, img);
            }
          }
          if (!staged) {
#pragma unroll
            for (int sub = 0; sub < kSub; ++sub)
              tma_load_2d_pair(smB + s * kBHalfBytes + sub * kSubBytes, &tmB, fb, kb * BK, nb + sub * kSubN);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ------------------------------ MMA issuer (leader) ------------------------------
      uint32_t it = 0, local = 0;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++local) {
        const uint32_t acc = local % kAcc;
        const uint32_t use = local / kAcc;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const uint32_t idesc = tile >= tail_full ? kIdescHalf : kIdesc;
        for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          if (it == 0) HP_GTRACE(4);
          tc_fence_after();
          const uint64_t da = sdesc_sw128_kmajor(smA + s * kABytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
#pragma unroll
            for (int sub = 0; sub < kSub; ++sub) {
              const uint64_t db = sdesc_sw128_kmajor(smB + s * kBHalfBytes + sub * kSubBytes);
              umma_bf16_pair(d_tmem + sub * kSubN, da + 2 * k, db + 2 * k, idesc, (kb | k) ? 1u : 0u);
            }
          }
          umma_commit_pair(&empty[s], 0x3);
        }
        umma_commit_pair(&tfull[acc], 0x3);
        if (local == 0) HP_GTRACE(5);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------ epilogue (both CTAs, own 128 rows) ------------------------------
    const int quarter = warp & 3;
    const int et = threadIdx.x - 128;
    const bool any_bias = p.bias != nullptr || p.bias2 != nullptr;
    const bool fold = EP == kEpiFold || (EP == kEpRuntime && p.ln_stats != nullptr);
    uint32_t local = 0;
    for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++local) {
      const uint32_t acc = local % kAcc;
      const uint32_t use = local / kAcc;
      int bt, m0, n0, half;
      decode(tile, bt, m0, n0, half);
      float* sb = any_bias ? sbias + (local & 1) * BN : nullptr;      // staging stays double-buffered
      float* scs = scolsum + (local & 1) * BN;
      if (any_bias || fold) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const long long img = p.batch > 1 ? (long long)bt : (long long)(m0 / p.bias2_div);
        // a half tile's columns: B rows n0 + 64 h + [0, 64) (linear), n0 + BN/2 + 64 h + [0, 64) (gate)
        const int ncols = half >= 0 ? BN / 2 : BN;
        for (int i = et; i < ncols; i += 128) {
          const int col = half < 0 ? n0 + i : n0 + half * (BN / 4) + (i < BN / 4 ? i : i + BN / 4);
          if (any_bias) {
            float b = p.bias ? __ldg(p.bias + col) : 0.0f;
            if (p.bias2) b += __ldg(p.bias2 + img * p.bias2_ld + col);
            sb[i] = b;
          }
          if (fold) scs[i] = __ldg(p.ln_colsum + col);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      float f_mean = 0.f, f_rstd = 1.f;
      const int my_row = m0 + quarter * 32 + lane;
      if (fold && my_row < p.M) fold_row_stats(p, my_row, f_mean, f_rstd);
      prefetch_res_row<BN>(p, bt, my_row, n0);     // residual lines in flight while the MMAs finish
      mbar_wait(&tfull[acc], use & 1);
      if (et == 0 && local == 0) HP_GTRACE(6);
      tc_fence_after();
      const uint32_t t_acc = tmem_base + acc * BN;
      const int gn_idx = p.gn_part ? (m0 / p.gn_rows) * p.gn_P + bt * (p.gn_rows / BM) + (m0 % p.gn_rows) / BM : 0;
      if constexpr (EP != kEpRuntime) {            // one epilogue flavour compiled in
        GemmParams q = p;                          // batched: this tile's image (or phase)
        if (p.batch > 1) batch_offsets(q, bt);
        epilogue_tile<BN, EP, AM>(q, t_acc, m0, n0, quarter, lane, sb, nullptr, scs, f_mean, f_rstd, 0, BN, nullptr,
                                  gsm, gn_idx, half);
      } else if (p.batch > 1) {
        GemmParams q = p;
        batch_offsets(q, bt);
        bool done = false;
        if constexpr (BN % 160 == 0) {             // the upsampler's GroupNorm partials
          if (p.gn_part) {
            epilogue_tile<BN, kEpiGn, AM>(q, t_acc, m0, n0, quarter, lane, sb, nullptr, nullptr, 0.f, 1.f, 0, BN,
                                          nullptr, gsm, gn_idx);
            done = true;
          }
        }
        if (!done) epilogue_tile<BN, kEpiPlain, AM>(q, t_acc, m0, n0, quarter, lane, sb, nullptr, nullptr, 0.f, 1.f);
      } else if (fold) {
        epilogue_tile<BN, kEpiFold, AM>(p, t_acc, m0, n0, quarter, lane, sb, nullptr, scs, f_mean, f_rstd);
      } else if (p.stats_out) {
        epilogue_tile<BN, kEpiStats, AM>(p, t_acc, m0, n0, quarter, lane, sb, nullptr, nullptr, 0.f, 1.f);
      } else {
        if (p.probe_noepi != 1) epilogue_tile<BN, kEpiPlain, AM>(p, t_acc, m0, n0, quarter, lane, sb, nullptr, nullptr, 0.f, 1.f);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(mapa_shared(&tempty[acc], 0));   // the leader's TMEM-free barrier
      if (et == 0 && local == 0) HP_GTRACE(7);
    }
  }
  tc_fence_before();
  cluster_barrier();                 // all MMAs consumed, both epilogues done
  if (threadIdx.x == 0) HP_GTRACE(8);
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
}

// ---------------------------------------------------------------------------
// Split-K over two CTA pairs (cluster of 4): small-M GEMMs whose 256 x 320 tiles
// number at most SMs/4 (SDXL level 2: M=2048, N=1280 -> 32 tiles). Pair kh = rank/2
// runs K blocks [kh*kb/2, (kh+1)*kb/2) of the SAME tile at the efficient 320 width;
// then each CTA ships the half of its accumulator it does not finalise (128 x 160
// fp32) into its K-partner's (rank ^ 2) now idle smem ring through distributed
// shared memory, and finalises its own half: acc + partner partial -> epilogue.
template <int STAGES, int EP>
__global__ void __launch_bounds__(kThreads, 1)
gemm_splitk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
  constexpr int BN = 320, kSubN = 160;
  constexpr uint32_t kSubBytes = (kSubN / 2) * BK * 2;
  constexpr uint32_t kBHalfBytes = 2 * kSubBytes;
  constexpr uint32_t kStageBytes = kABytes + kBHalfBytes;
  constexpr uint32_t kTmemCols = 512;
  constexpr uint32_t kIdesc = idesc_bf16_f32(2 * BM, kSubN);
  static_assert((size_t)STAGES * kABytes >= (size_t)kSubN * BM * 4, "partial must fit the A ring");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* sbias = reinterpret_cast<float*>(smem + STAGES * kStageBytes + 256);   // [BN]
  float* scolsum = sbias + BN;                                                   // [BN]
  float2* gsm = reinterpret_cast<float2*>(scolsum + BN);                        // [4][32] GroupNorm partials

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef HP_GEMM_TRACE
  __shared__ int s_slot;
  if (threadIdx.x == 0) s_slot = blockIdx.x == 0 ? (int)atomicAdd(&g_gemm_ctr, 1u) : -1;
  __syncthreads();
  const int g_slot = s_slot;
  if (threadIdx.x == 0 && g_slot >= 0) {
    g_gemm_ring[g_slot % kRing][9] = p.M; g_gemm_ring[g_slot % kRing][10] = p.N;
    g_gemm_ring[g_slot % kRing][11] = p.K; g_gemm_ring[g_slot % kRing][12] = 1000 + BN;   // split-K
  }
#endif
  if (threadIdx.x == 0) HP_GTRACE(0);
  const uint32_t rank = cluster_ctarank();
  const uint32_t pr = rank & 1, kh = rank >> 1;          // CTA within pair, K half
  const bool leader = pr == 0;
  const uint16_t pair_mask = (uint16_t)(0x3u << (rank & 2));
  const int tile = blockIdx.x >> 2;
  const int m0 = (tile % p.num_m_tiles) * (2 * BM) + (int)pr * BM;
  const int n0 = (tile / p.num_m_tiles) * BN;
  const int kb_half = p.num_kb / 2;
  const int kb_lo = kh ? kb_half : 0, kb_hi = kh ? p.num_kb : kb_half;
  const int h0 = (int)kh * kSubN;                        // the 160 columns this CTA finalises

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_barrier();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x != 0) pdl_wait();          // the producer waits after staging its weights
  pdl_trigger();

  float f_mean = 0.f, f_rstd = 1.f;
  if (warp == 0) {
    if (lane == 0) {
      int img = 0, y0 = 0, x0 = 0;
      if (p.mode != HP_A_PLAIN) {
        const int hw = p.out_h * p.out_w;
        img = m0 / hw;
        const int rem = m0 - img * hw;
        y0 = rem / p.out_w;
        x0 = rem - y0 * p.out_w;
      }
      const uint32_t nb = n0 + pr * (kSubN / 2);
      // weights of the first k-blocks before the PDL wait (they never depend on the
      // previous kernel); A follows once it is done
      const int pre = min(STAGES, kb_hi - kb_lo);
      for (int i = 0; i < pre; ++i) {
        if (leader) mbar_arrive_expect_tx(&full[i], 2 * kStageBytes);
        const uint32_t fb = mapa_shared(&full[i], rank & ~1u);
#pragma unroll
        for (int sub = 0; sub < 2; ++sub)
          tma_load_2d_pair(smB + i * kBHalfBytes + sub * kSubBytes, &tmB, fb, (kb_lo + i) * BK, nb + sub * kSubN);
      }
      pdl_wait();
      HP_GTRACE(2);
      uint32_t it = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        const bool staged = (int)it < pre;
        if (!staged) {
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * kStageBytes);
        }
        const uint32_t fb = mapa_shared(&full[s], rank & ~1u);
        uint8_t* a_dst = smA + s * kABytes;
        if (p.mode == HP_A_PLAIN) {
          tma_load_2d_pair(a_dst, &tmA, fb, kb * BK, m0);
        } else {
          const int tap = kb / p.cin_blocks;
          const int cb = kb - tap * p.cin_blocks;
          const int dy = tap / 3, dx = tap - dy * 3;
          if (p.mode == HP_A_CONV3X3) tma_load_4d_pair(a_dst, &tmA, fb, cb * BK, x0 + dx - 1, y0 + dy - 1, img);
          else tma_load_4d_pair(a_dst, &tmA, fb, cb * BK, 2 * x0 + dx - 1, 2 * y0 + dy - 1, img);
        }
        if (!staged) {
#pragma unroll
          for (int sub = 0; sub < 2; ++sub)
            tma_load_2d_pair(smB + s * kBHalfBytes + sub * kSubBytes, &tmB, fb, kb * BK, nb + sub * kSubN);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      uint32_t it = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        if (it == 0) HP_GTRACE(4);
        tc_fence_after();
        const uint64_t da = sdesc_sw128_kmajor(smA + s * kABytes);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            const uint64_t db = sdesc_sw128_kmajor(smB + s * kBHalfBytes + sub * kSubBytes);
            umma_bf16_pair(tmem_base + sub * kSubN, da + 2 * k, db + 2 * k, kIdesc, (it | k) ? 1u : 0u);
          }
        }
        umma_commit_pair(&empty[s], pair_mask);
      }
      umma_commit_pair(tfull, pair_mask);
      HP_GTRACE(5);
    }
  } else if (warp >= 4) {
    const int et = threadIdx.x - 128;
    const int quarter = warp & 3;
    const bool any_bias = p.bias != nullptr || p.bias2 != nullptr;
    const bool fold = EP == kEpiFold;
    const long long img = (long long)(m0 / p.bias2_div);
    for (int i = et; i < BN; i += 128) {
      if (any_bias) {
        float b = p.bias ? __ldg(p.bias + n0 + i) : 0.0f;
        if (p.bias2) b += __ldg(p.bias2 + img * p.bias2_ld + n0 + i);
        sbias[i] = b;
      }
      if (fold) scolsum[i] = __ldg(p.ln_colsum + n0 + i);
    }
    const int my_row = m0 + quarter * 32 + lane;
    if (fold && my_row < p.M) fold_row_stats(p, my_row, f_mean, f_rstd);
    prefetch_res_row<kSubN>(p, 0, my_row, n0 + h0);   // only the 160 columns this CTA finalises
    mbar_wait(tfull, 0);
    if (et == 0) HP_GTRACE(6);
    tc_fence_after();
  }
  __syncwarp();
  tc_fence_before();
  cluster_barrier();                   // #1: every MMA of both pairs done, both rings idle
  tc_fence_after();
  if (warp >= 4) {
    // ship the half this CTA does not finalise into the K-partner's A ring: [col/4][row][4]
    const int quarter = warp & 3;
    const int rloc = quarter * 32 + lane;
    const uint32_t lane_addr = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const int oh0 = (int)(kh ^ 1) * kSubN;
    const uint32_t dst = mapa_shared(smA, rank ^ 2u);
#pragma unroll 1
    for (int c = 0; c < kSubN / 32; ++c) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(lane_addr + oh0 + c * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t a = dst + (uint32_t)(((c * 8 + q) * 128 + rloc) * 16);
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};"
                     :: "r"(a), "f"(__uint_as_float(r[4 * q])), "f"(__uint_as_float(r[4 * q + 1])),
                        "f"(__uint_as_float(r[4 * q + 2])), "f"(__uint_as_float(r[4 * q + 3])) : "memory");
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_barrier();                   // #2: partials delivered
  if (threadIdx.x == 128) HP_GTRACE(3);
  tc_fence_after();
  if (warp >= 4) {
    const int quarter = warp & 3;
    const float* sb = (p.bias != nullptr || p.bias2 != nullptr) ? sbias : nullptr;
    const float4* red = reinterpret_cast<const float4*>(smA);
    const int gn_idx = p.gn_part ? (m0 / p.gn_rows) * p.gn_P + (m0 % p.gn_rows) / BM : 0;
    epilogue_tile<BN, EP, kAmNone>(p, tmem_base, m0, n0, quarter, lane, sb, nullptr, scolsum, f_mean, f_rstd, h0,
                                   kSubN, red, gsm, gn_idx);
  }
  __syncwarp();
  tc_fence_before();
  if (threadIdx.x == 128) HP_GTRACE(7);
  cluster_barrier();                   // #3: nobody frees TMEM while its pair partner still reads
  if (threadIdx.x == 0) HP_GTRACE(8);
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
}

// ---------------------------------------------------------------------------
// host side: tensor maps (driver entry point, no -lcuda link dependency)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
              const uint32_t* box, const uint32_t* estride) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = estride ? estride[i] : 1; }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, s, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <int BN, int STAGES>
int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, cudaStream_t st) {
  constexpr size_t smem = 1024 + (size_t)STAGES * (kABytes + BN * BK * 2) + 256 + 4 * BN * sizeof(float) +
                         2 * BM * sizeof(float);
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return HP_ERR_CUDA;
    attr_set = true;
  }
  const int tiles = p.num_m_tiles * p.batch * p.num_n_tiles;
  if (p.ln_mode) {
    // non-persistent: one CTA per tile, a cluster spans the N tiles of a row block
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.num_n_tiles;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = hp_pdl_enabled() ? 2 : 1;
    if (cudaLaunchKernelEx(&cfg, gemm_kernel<BN, STAGES>, ta, tb, p) != cudaSuccess) return HP_ERR_CUDA;
    return HP_OK;
  }
  const int grid = tiles < num_sms() ? tiles : num_sms();
  if (hp_launch_pdl(gemm_kernel<BN, STAGES>, dim3(grid), dim3(kThreads), smem, st, ta, tb, p) != cudaSuccess)
    return HP_ERR_CUDA;
  return HP_OK;
}

template <int BN, int STAGES, int AM, int EP = kEpRuntime>
int launch_gemm_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, cudaStream_t st) {
  constexpr size_t smem = 1024 + (size_t)STAGES * (kABytes + (BN / 2) * BK * 2) + 256 + 4 * BN * sizeof(float) +
                         4 * 32 * sizeof(float2);
  static_assert(smem <= 227 * 1024, "pair GEMM smem");
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_pair_kernel<BN, STAGES, AM, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return HP_ERR_CUDA;
    attr_set = true;
  }
  const int tiles = p.num_m_tiles * p.batch * p.num_n_tiles;
  const int pairs = num_sms() / 2;
  const int clusters = tiles < pairs ? tiles : pairs;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = hp_pdl_enabled() ? 2 : 1;
  if (cudaLaunchKernelEx(&cfg, gemm_pair_kernel<BN, STAGES, AM, EP>, ta, tb, p) != cudaSuccess) return HP_ERR_CUDA;
  return HP_OK;
}

template <int STAGES, int EP>
int launch_gemm_splitk(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, cudaStream_t st) {
  constexpr size_t smem = 1024 + (size_t)STAGES * (kABytes + 160 * BK * 2) + 256 + 2 * 320 * sizeof(float) +
                         4 * 32 * sizeof(float2);
  static_assert(smem <= 227 * 1024, "split-K GEMM smem");
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_splitk_kernel<STAGES, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return HP_ERR_CUDA;
    attr_set = true;
  }
  const int tiles = p.num_m_tiles * p.num_n_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(4 * tiles);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 4;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = hp_pdl_enabled() ? 2 : 1;
  if (cudaLaunchKernelEx(&cfg, gemm_splitk_kernel<STAGES, EP>, ta, tb, p) != cudaSuccess) return HP_ERR_CUDA;
  return HP_OK;
}

bool splitk_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HP_GEMM_SPLITK");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

bool pair_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HP_GEMM_PAIR");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// split-K over two CTA pairs for wide-N, small-M layers (SDXL level 2: N = 1280).
// Depends on N and K only, never on M, so one image's rows are computed identically
// whatever else is in the batch (batch invariance: split-K changes the summation).
bool splitk_ok(int64_t M, int64_t N, int64_t K, int act, int batch, int mode) {
  if (!splitk_enabled() || !pair_enabled() || act != HP_ACT_NONE || batch > 1 || M <= BM) return false;
  // the exchange + half epilogue costs ~4 us: worth it from K = 4096 on (ff2, 3x3 convs)
  return N % 320 == 0 && N >= 1280 && K / BK >= 64;
}

// block_n for an M x N x K problem: whole-wave tile counts on the SMs (CTA pairs for
// M > 128) times the per-tile time, k-blocks x N / (measured main-loop rate of that
// width), plus exposed epilogues (~5 k-blocks' worth each). 320 keeps one accumulator
// (no epilogue/MMA overlap), so each of its tiles exposes one.
int pick_bn(int64_t M, int64_t N, int64_t K, int act, int batch = 1, int mode = HP_A_PLAIN, bool gn = false) {
  const int cands[5] = {320, 256, 160, 128, 64};
  int best = 0;
  double best_cost = 1e30;
  // M = rows per batch slice: every slice rounds up to whole row tiles on its own
  const bool pair = pair_enabled() && M > BM;
  const int64_t mt = (int64_t)(batch > 1 ? batch : 1) * (pair ? (M + 2 * BM - 1) / (2 * BM) : (M + BM - 1) / BM);
  const int sms = (g_num_sms ? g_num_sms : 148) / (pair ? 2 : 1);
  const double kb = (double)((K + BK - 1) / BK);
  // measured main-loop rate per SM relative to block_n 256 (pair kernel, B200): every MMA
  // re-reads its 128-row A slab from shared memory, so wide N tiles amortise it best
  auto rate = [](int bn) { return bn >= 256 ? 1.0 : bn >= 160 ? 0.72 : bn >= 128 ? 0.6 : 0.35; };
  if (pair && splitk_ok(M, N, K, act, batch, mode)) return 320;   // fixed choice (see splitk_ok)
  for (int bn : cands) {
    if (N % bn) continue;
    if (gn && bn % 160) continue;                                  // GroupNorm partials: 160-column tile groups
    if (bn > 256 && (!pair || act == HP_ACT_GEGLU)) continue;    // 320 = two N=160 MMAs, pair kernel only
    if (act == HP_ACT_GEGLU && bn != 256 && bn != 128) continue;
    const int64_t tiles = mt * (N / bn);
    const int64_t waves = (tiles + sms - 1) / sms;
    // the last tile's epilogue is always exposed; with one accumulator (320) every tile's is
    const double epi = 5.0 * bn;
    const double cost = (double)waves * (kb * bn / rate(bn) + 48.0) + epi * (bn > 256 ? (double)waves : 1.0);
    if (cost < best_cost - 1e-9) { best_cost = cost; best = bn; }
  }
  return best;
}

}  // namespace

extern "C" {

int32_t hp_gemm_pick_block_n(int64_t M, int64_t N, int64_t K, int32_t act) { return pick_bn(M, N, K, act); }

int32_t hp_gemm_stats_block_n(int64_t M, int64_t N, int64_t K) {
  num_sms();
  const int bn = pick_bn(M, N, K, HP_ACT_NONE);
  if (bn == 320 || N % 160) return bn;        // 320 (split or not) writes 160-wide segments
  return 160;
}

int hp_gemm(const hp_gemm_desc* d, void* stream) {
  if (!d || !d->a || !d->b || !d->d) return HP_ERR_PARAMETER;
  if (d->M <= 0 || d->N <= 0 || d->K <= 0) return HP_ERR_SHAPE;
  if ((d->K % 8) || (d->ldb % 8)) return HP_ERR_UNSUPPORTED;   // 16-byte TMA strides
  if ((reinterpret_cast<uintptr_t>(d->a) | reinterpret_cast<uintptr_t>(d->b)) & 15) return HP_ERR_UNSUPPORTED;
  num_sms();
  const bool upconv = d->a_mode == HP_A_UPCONV;
  const int nbatch = upconv ? 4 : (d->batch > 1 ? d->batch : 1);
  const bool gn = d->gn_part != nullptr;
  const int bn = d->block_n ? d->block_n : pick_bn(d->M, d->N, d->K, d->act, nbatch, d->a_mode, gn);
  if (bn == 0 || d->N % bn) return HP_ERR_UNSUPPORTED;
  // GroupNorm partials: CTA-pair or split-K kernel, whole 128-row blocks of one image,
  // 160-multiple tiles (segments never straddle a tile), plain epilogue values
  if (gn && (bn % 160 || d->M % BM || (d->alpha != 0.0f && d->alpha != 1.0f) || d->M <= BM || !pair_enabled() || d->act != HP_ACT_NONE || d->ln_y ||
             d->stats_out || d->ln_stats || d->colscale || d->gn_rows <= 0 || d->gn_rows % BM ||
             d->M % d->gn_rows || d->gn_parts <= 0 || (reinterpret_cast<uintptr_t>(d->gn_part) & 7)))
    return HP_ERR_UNSUPPORTED;
  if (d->act == HP_ACT_GEGLU && (bn % 64)) return HP_ERR_UNSUPPORTED;
  const int64_t n_out = d->act == HP_ACT_GEGLU ? d->N / 2 : d->N;
  if ((d->ldd % 8) || (d->residual && (d->ldr % 8)) || (n_out % 32)) return HP_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(d->d) & 15) || (d->bias && (reinterpret_cast<uintptr_t>(d->bias) & 15)))
    return HP_ERR_UNSUPPORTED;

  GemmParams p{};
  p.M = (int)d->M; p.N = (int)d->N; p.K = (int)d->K;
  p.mode = d->a_mode;
  p.d = static_cast<__nv_bfloat16*>(d->d); p.ldd = d->ldd;
  p.bias = d->bias; p.bias2 = d->bias2; p.bias2_div = d->bias2_div > 0 ? d->bias2_div : 1;
  p.bias2_ld = d->bias2_ld > 0 ? d->bias2_ld : d->N;
  if (d->bias2 && (p.bias2_div % BM)) return HP_ERR_UNSUPPORTED;   // one image per 128-row tile
  p.res = static_cast<const __nv_bfloat16*>(d->residual); p.ldr = d->ldr;
  p.act = d->act;
  p.colscale = d->colscale;
  if (d->colscale && (reinterpret_cast<uintptr_t>(d->colscale) & 15)) return HP_ERR_UNSUPPORTED;
  p.alpha = d->alpha == 0.0f ? 1.0f : d->alpha;
  p.batch = nbatch;
  if (upconv && (d->batch > 1 || d->residual || d->colscale || d->bias2 || d->ln_y || d->stats_out ||
                 d->ln_stats || d->act == HP_ACT_GEGLU || d->M <= BM || !pair_enabled()))
    return HP_ERR_UNSUPPORTED;
  p.ln_mode = d->ln_y != nullptr;
  p.ln_g = d->ln_gamma; p.ln_b = d->ln_beta; p.ln_eps = d->ln_eps;
  p.ln_y = static_cast<__nv_bfloat16*>(d->ln_y); p.ldy = d->ldy;
  if (p.ln_mode && (p.batch > 1 || d->act == HP_ACT_GEGLU || !d->ln_gamma || !d->ln_beta || (d->ldy % 8) ||
                    (reinterpret_cast<uintptr_t>(d->ln_y) & 15)))
    return HP_ERR_UNSUPPORTED;
  p.vec256 = ((d->ldd % 16) == 0) && ((reinterpret_cast<uintptr_t>(d->d) & 31) == 0) &&
             (!d->residual || (((d->ldr % 16) == 0) && ((reinterpret_cast<uintptr_t>(d->residual) & 31) == 0))) &&
             (p.batch <= 1 || upconv || (((d->d_bstride | d->r_bstride) % 16) == 0));
  // development probes, read once: HP_GEMM_PROBE_NOEPI=1 skips the plain epilogue, =2 only
  // its stores (isolates the main loop); HP_GEMM_RASTER_N=1 walks N tiles fastest
  static const int probe = [] {
    const char* e = getenv("HP_GEMM_PROBE_NOEPI");
    return e ? (e[0] == '2' ? 2 : 1) : 0;
  }();
  static const bool raster_n = getenv("HP_GEMM_RASTER_N") != nullptr;
  p.probe_noepi = probe;
  p.raster_n = raster_n;
  p.stats_out = reinterpret_cast<float2*>(d->stats_out);
  if (p.stats_out && (p.batch > 1 || d->act == HP_ACT_GEGLU || p.ln_mode || d->a_mode != HP_A_PLAIN ||
                      (reinterpret_cast<uintptr_t>(d->stats_out) & 7)))
    return HP_ERR_UNSUPPORTED;
  p.ln_stats = reinterpret_cast<const float2*>(d->ln_stats);
  p.ln_parts = d->ln_parts; p.ln_part_n = (float)d->ln_part_n;
  p.ln_colsum = d->ln_colsum; p.ln_fold_eps = d->ln_fold_eps;
  if (p.ln_stats) {
    if (p.batch > 1 || p.ln_mode || d->a_mode != HP_A_PLAIN || !d->ln_colsum || d->ln_parts <= 0 ||
        d->ln_part_n <= 0 || d->ln_parts > kMaxFoldParts || (int64_t)d->ln_parts * d->ln_part_n != d->K ||
        (reinterpret_cast<uintptr_t>(d->ln_stats) & 7) || (reinterpret_cast<uintptr_t>(d->ln_colsum) & 15))
      return HP_ERR_UNSUPPORTED;
  }
  p.gn_part = reinterpret_cast<float2*>(d->gn_part);
  p.gn_rows = (int)d->gn_rows; p.gn_P = d->gn_parts; p.gn_ld = (int)(d->N / kGnSeg);
  p.a_bs = d->a_bstride; p.d_bs = d->d_bstride; p.r_bs = d->r_bstride; p.cs_bs = d->cs_bstride;
  if (upconv) {      // output phases (py, px) of the 2x grid: see HP_A_UPCONV
    p.ldd = 2 * d->ldd;
    p.row_w = d->img_w;
    p.ld_hi = 4LL * d->img_w * d->ldd;
    p.d_bs = 2LL * d->img_w * d->ldd;
    p.d_bs2 = d->ldd;
    p.a_bs = p.r_bs = p.cs_bs = 0;
  }
  if (p.batch > 1 && d->a_mode != HP_A_PLAIN && !upconv) return HP_ERR_UNSUPPORTED;
  if (p.batch > 1 && ((p.a_bs | p.d_bs | p.r_bs) % 8 || p.cs_bs % 4)) return HP_ERR_UNSUPPORTED;
  p.num_m_tiles = (int)((d->M + BM - 1) / BM);
  p.num_n_tiles = (int)(d->N / bn);
  if (p.ln_mode && p.num_n_tiles > 8) return HP_ERR_UNSUPPORTED;     // portable cluster size

  CUtensorMap ta, tb;
  if (d->a_mode == HP_A_PLAIN) {
    if (d->lda % 8) return HP_ERR_UNSUPPORTED;
    p.num_kb = (int)((d->K + BK - 1) / BK);
    if (p.batch > 1) {
      const uint64_t dims[3] = {(uint64_t)d->K, (uint64_t)d->M, (uint64_t)p.batch};
      const uint64_t str[2] = {(uint64_t)d->lda * 2, (uint64_t)p.a_bs * 2};
      const uint32_t box[3] = {BK, BM, 1};
      if (!make_map(&ta, d->a, 3, dims, str, box, nullptr)) return HP_ERR_CUDA;
    } else {
      const uint64_t dims[2] = {(uint64_t)d->K, (uint64_t)d->M};
      const uint64_t str[1] = {(uint64_t)d->lda * 2};
      const uint32_t box[2] = {BK, BM};
      if (!make_map(&ta, d->a, 2, dims, str, box, nullptr)) return HP_ERR_CUDA;
    }
  } else if (d->a_mode == HP_A_CONV3X3 || d->a_mode == HP_A_CONV3X3_S2 || upconv) {
    const int s = d->a_mode == HP_A_CONV3X3_S2 ? 2 : 1;
    const int c = d->img_c;
    if (c % BK || d->K != (upconv ? 4LL : 9LL) * c) return HP_ERR_SHAPE;
    p.out_h = d->img_h / s;
    p.out_w = d->img_w / s;
    if ((int64_t)d->img_n * p.out_h * p.out_w != d->M) return HP_ERR_SHAPE;
    p.box_w = p.out_w < BM ? p.out_w : BM;
    p.box_h = BM / p.box_w;
    if (BM % p.box_w || p.out_w % p.box_w || p.out_h % p.box_h) return HP_ERR_UNSUPPORTED;
    p.cin_blocks = c / BK;
    p.num_kb = (upconv ? 4 : 9) * p.cin_blocks;
    const uint64_t dims[4] = {(uint64_t)c, (uint64_t)d->img_w, (uint64_t)d->img_h, (uint64_t)d->img_n};
    const uint64_t str[3] = {(uint64_t)c * 2, (uint64_t)d->img_w * c * 2, (uint64_t)d->img_h * d->img_w * c * 2};
    const uint32_t box[4] = {BK, (uint32_t)(p.box_w * s), (uint32_t)(p.box_h * s), 1};
    const uint32_t es[4] = {1, (uint32_t)s, (uint32_t)s, 1};
    if (!make_map(&ta, d->a, 4, dims, str, box, es)) return HP_ERR_CUDA;
  } else {
    return HP_ERR_PARAMETER;
  }
  // CTA pairs for every GEMM with more than one 128-row block (not the cluster-LN mode)
  const bool pair = pair_enabled() && !p.ln_mode && d->M > BM;
  {
    const uint64_t dims[2] = {(uint64_t)d->K, (uint64_t)d->N * (upconv ? 4 : 1)};   // upconv: 4 phases
    const uint64_t str[1] = {(uint64_t)d->ldb * 2};
    const uint32_t box[2] = {BK, (uint32_t)(pair ? (bn > 256 ? bn / 4 : bn / 2) : bn)};
    if (!make_map(&tb, d->b, 2, dims, str, box, nullptr)) return HP_ERR_CUDA;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // lean epilogue: no activation code, alpha 1, no column gate, 32-byte rows, no probe
  const bool lean = p.alpha == 1.0f && !p.colscale && p.vec256 && p.probe_noepi == 0 && p.batch == 1 &&
                    (d->act == HP_ACT_NONE || d->act == HP_ACT_GEGLU);
  // lean batched / gated / GELU instances (the MMDiT's joint blocks): plain epilogue flavour
  const bool lean2 = p.alpha == 1.0f && p.vec256 && p.probe_noepi == 0 && !p.ln_stats && !p.stats_out &&
                     !p.ln_mode && (bn == 256 || bn == 128 || bn == 64) &&
                     ((d->act == HP_ACT_GELU && !p.colscale) || (d->act == HP_ACT_NONE && (p.colscale || p.batch > 1)));
  // GroupNorm partials: the lean instances (batch 1) or the batched runtime branch (upconv)
  if (p.gn_part && (!pair || (p.batch == 1 && !lean))) return HP_ERR_UNSUPPORTED;
  if (pair && lean && bn == 320 && splitk_ok(d->M, d->N, d->K, d->act, p.batch, d->a_mode)) {
    p.num_m_tiles = (int)((d->M + 2 * BM - 1) / (2 * BM));
    return p.ln_stats ? launch_gemm_splitk<5, kEpiFold>(ta, tb, p, st)
         : p.stats_out ? launch_gemm_splitk<5, kEpiStats>(ta, tb, p, st)
         : p.gn_part ? launch_gemm_splitk<5, kEpiGn>(ta, tb, p, st)
                       : launch_gemm_splitk<5, kEpiPlain>(ta, tb, p, st);
  }
  if (pair) {
    p.num_m_tiles = (int)((d->M + 2 * BM - 1) / (2 * BM));
    if (lean && d->act == HP_ACT_GEGLU) {
      const bool f = p.ln_stats != nullptr;
      // last partial wave of 256-wide tiles: run it as twice as many half-width tiles when
      // they fit one round of the CTA pairs (tile width does not change the arithmetic)
      static const bool tail = [] {
        const char* e = getenv("HP_GEMM_GEGLU_TAIL");
        return !(e && e[0] == '0');
      }();
      const int tiles = p.num_m_tiles * p.batch * p.num_n_tiles, pairs = num_sms() / 2;
      const int rem = tiles % pairs;
      if (tail && bn == 256 && tiles > pairs && rem > 0 && 2 * rem <= pairs) {
        p.tail_full = tiles - rem;
        p.tiles_eff = tiles + rem;
      }
      switch (bn) {
        case 256: return f ? launch_gemm_pair<256, 6, kAmGeglu, kEpiFold>(ta, tb, p, st)
                           : launch_gemm_pair<256, 6, kAmGeglu, kEpiPlain>(ta, tb, p, st);
        case 128: return f ? launch_gemm_pair<128, 8, kAmGeglu, kEpiFold>(ta, tb, p, st)
                           : launch_gemm_pair<128, 8, kAmGeglu, kEpiPlain>(ta, tb, p, st);
        default: return HP_ERR_UNSUPPORTED;
      }
    }
    if (lean2 && pair) {
      const bool gelu = d->act == HP_ACT_GELU;
      const bool gate = p.colscale != nullptr;
#define HP_PAIR_LEAN2(BN_, ST_)                                                                         \
  return gelu ? launch_gemm_pair<BN_, ST_, kAmGelu, kEpiPlain>(ta, tb, p, st)                          \
       : gate ? launch_gemm_pair<BN_, ST_, kAmGate, kEpiPlain>(ta, tb, p, st)                          \
              : launch_gemm_pair<BN_, ST_, kAmNone, kEpiPlain>(ta, tb, p, st)
      switch (bn) {
        case 256: HP_PAIR_LEAN2(256, 6);
        case 128: HP_PAIR_LEAN2(128, 8);
        case 64: HP_PAIR_LEAN2(64, 8);
        default: break;
      }
#undef HP_PAIR_LEAN2
    }
    if (!lean || d->act != HP_ACT_NONE) {
      switch (bn) {
        case 320: return launch_gemm_pair<320, 5, kAmAny>(ta, tb, p, st);
        case 256: return launch_gemm_pair<256, 6, kAmAny>(ta, tb, p, st);
        case 160: return launch_gemm_pair<160, 7, kAmAny>(ta, tb, p, st);
        case 128: return launch_gemm_pair<128, 8, kAmAny>(ta, tb, p, st);
        case 64: return launch_gemm_pair<64, 8, kAmAny>(ta, tb, p, st);
        default: return HP_ERR_UNSUPPORTED;
      }
    }
    if (p.gn_part) {
      if (bn == 320) return launch_gemm_pair<320, 5, kAmNone, kEpiGn>(ta, tb, p, st);
      return launch_gemm_pair<160, 7, kAmNone, kEpiGn>(ta, tb, p, st);
    }
    const int ep = p.ln_stats ? kEpiFold : (p.stats_out ? kEpiStats : kEpiPlain);
#define HP_PAIR_LEAN(BN_, ST_)                                                                          \
  return ep == kEpiFold ? launch_gemm_pair<BN_, ST_, kAmNone, kEpiFold>(ta, tb, p, st)                 \
       : ep == kEpiStats ? launch_gemm_pair<BN_, ST_, kAmNone, kEpiStats>(ta, tb, p, st)               \
                         : launch_gemm_pair<BN_, ST_, kAmNone, kEpiPlain>(ta, tb, p, st)
    switch (bn) {
      case 320: HP_PAIR_LEAN(320, 5);
      case 256: HP_PAIR_LEAN(256, 6);
      case 160: HP_PAIR_LEAN(160, 7);
      case 128: HP_PAIR_LEAN(128, 8);
      case 64: HP_PAIR_LEAN(64, 8);
      default: return HP_ERR_UNSUPPORTED;
    }
#undef HP_PAIR_LEAN
  }
  switch (bn) {
    case 256: return launch_gemm<256, 4>(ta, tb, p, st);
    case 160: return launch_gemm<160, 5>(ta, tb, p, st);
    case 128: return launch_gemm<128, 6>(ta, tb, p, st);
    case 64: return launch_gemm<64, 8>(ta, tb, p, st);
    default: return HP_ERR_UNSUPPORTED;
  }
}

}  // extern "C"

#ifdef HP_GEMM_TRACE
#include <string.h>
// trace builds only (tools/gemm_ring.py): copy the launch ring / counter to the host
extern "C" int hp_debug_symbol(const char* name, void* dst, size_t bytes) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (!strcmp(name, "g_gemm_ring")) return cudaMemcpyFromSymbol(dst, g_gemm_ring, bytes) == cudaSuccess ? 0 : -1;
  if (!strcmp(name, "g_gemm_ctr")) return cudaMemcpyFromSymbol(dst, g_gemm_ctr, bytes) == cudaSuccess ? 0 : -1;
  return -2;
}
#endif
