// hp_attn.cu — K5: fused multi-head attention (head_dim 64) on tcgen05.
//
// One CTA = two 128-query tiles of one (head, batch); 320 threads:
//   warps 0-3   softmax for query tile 0 (thread i owns query row i)
//   warps 4-7   softmax for query tile 1
//   warp 8      TMA: Q0, Q1 once, then K/V tiles of 128 keys (3-stage ring)
//   warp 9      TMEM allocation + MMA issue:
//                 S_q(j) = Q_q K(j)^T           -> TMEM S_q   (128 cols fp32)
//                 O_q   += P_q(j) V(j)          -> TMEM O_q   (64 cols fp32, accumulated)
//               issued S0(j), PV0(j-1), S1(j), PV1(j-1), so the tensor core
//               works on one tile while the other tile's softmax runs.
// Softmax (per row, fp32, log2 domain): one TMEM pass over S, block max, lazy
// rescale of O in TMEM only when the running max grows by more than 2^8
// (otherwise the stale max is kept: p <= 2^8, exact after the final 1/l), and
// exp2 split between MUFU.EX2 and a degree-3 polynomial on the FMA pipe (P is
// rounded to bf16 anyway). P goes to shared memory as the SW128 K-major A
// operand of the PV MMA; V is consumed MN-major straight from its TMA tile.
//
// Launch variants (hp_attention picks one):
//   S_kv <= 128        single-block kernel, 2 CTAs/SM (cross-attention)
//   short last wave    split-KV kernel: one query tile per CTA, its key range cut
//                      in two halves processed by the two warpgroups and merged
//                      (fixed split point: batch-invariant); there P goes to TMEM
//                      (bf16 pairs) and the PV MMA reads it from there (TS-MMA)
//   otherwise          the two-tile kernel above
// (Measured and dropped: P kept in TMEM as the A operand of a TS-MMA with the
// whole S row in 200 registers: 180 us vs 169 us at S=4096; 64-key blocks with
// double-buffered S: slower; 2 threads per score row: slower.)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>
#include <mutex>
#include <stdlib.h>
#include "hybridpar_b200_denoiser.h"
#include "hp_common.cuh"
#include "hp_tc.cuh"

using namespace hptc;

namespace {

constexpr int kBQ = 128, kBK = 128, kD = 64;
constexpr int kStages = 3;
constexpr int kThreads = 320;
constexpr uint32_t kTileBytes = kBQ * kD * 2;        // 16 KB (Q, K or V tile)
constexpr uint32_t kPBytes = kBQ * kBK * 2;          // 32 KB (two 64-key SW128 atoms)
constexpr uint32_t kIdescS = idesc_bf16_f32(kBQ, kBK, 0);
constexpr uint32_t kIdescO = idesc_bf16_f32(kBQ, kD, 1);  // B (= V) MN-major
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;            // log2 units

struct AttnParams {
  int sq, skv, heads;
  int causal;
  int q_col0, k_col0, v_col0;
  __nv_bfloat16* o; long long ldo;
  float scale_log2;
  int n_kv;
};

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for a pair (x <= 0) on the FMA pipe: x = i + f, |f| <= 1/2, 2^f by a degree-3
// polynomial, then i added into the exponent field (t = x + 1.5*2^23 holds i in its mantissa)
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  const float a = fmaxf(lo2(x2), -126.0f), b = fmaxf(hi2(x2), -126.0f);
  const uint64_t x = pack2(a, b);
  const uint64_t magic = pack2(12582912.0f, 12582912.0f);
  const uint64_t t = fadd2(x, magic);
  const uint64_t fi = fadd2(t, pack2(-12582912.0f, -12582912.0f));
  const uint64_t f = ffma2(fi, pack2(-1.0f, -1.0f), x);
  // degree-3 fit of 2^f on [-1/2, 1/2]: max relative error 1.0e-4, well inside bf16's 2^-9
  uint64_t pz = ffma2(pack2(0.05592212f, 0.05592212f), f, pack2(0.24264069f, 0.24264069f));
  pz = ffma2(pz, f, pack2(0.69312102f, 0.69312102f));
  pz = ffma2(pz, f, pack2(0.99992444f, 0.99992444f));
  const uint32_t lo = (uint32_t)pz + ((uint32_t)t << 23);
  const uint32_t hi = (uint32_t)(pz >> 32) + ((uint32_t)(t >> 32) << 23);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
         "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
         "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
#define HP_R8(b) "=r"(r[(b) + 0]), "=r"(r[(b) + 1]), "=r"(r[(b) + 2]), "=r"(r[(b) + 3]), \
                 "=r"(r[(b) + 4]), "=r"(r[(b) + 5]), "=r"(r[(b) + 6]), "=r"(r[(b) + 7])
// 32 columns of TMEM into r[base .. base+31] (base a compile-time constant after inlining)
__device__ __forceinline__ void tmem_ld_x32_at(uint32_t taddr, uint32_t* r, const int base) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : HP_R8(base), HP_R8(base + 8), HP_R8(base + 16), HP_R8(base + 24)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// D (TMEM) += A (TMEM: lane = row, K packed two bf16 per column) . B (smem descriptor)
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t desc_b, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      :: "r"(tmem_d), "r"(tmem_a), "l"(desc_b), "r"(idesc), "r"(accumulate) : "memory");
}

// SINGLE: every key fits one 128-key block (cross-attention, skv <= 128). Then no
// rescale exists, O_q reuses S_q's TMEM columns once the softmax has consumed S_q,
// and one K/V stage suffices: 256 TMEM columns and 97 KB of smem, so two CTAs
// share an SM and one's latency chain (TMA -> MMA -> softmax -> PV -> store)
// overlaps the other's.
constexpr int kModePair = 0, kModeSingle = 1;
template <int MODE> struct AttnCfg {
  static constexpr bool kSingle = MODE == kModeSingle;
  static constexpr int kNq = 2;
  static constexpr int kThr = 32 * (4 * kNq + 2);
  static constexpr int kMinBlocks = MODE == kModePair ? 1 : 2;
  static constexpr int kSt = kSingle ? 1 : kStages;
  static constexpr uint32_t kCols = MODE == kModePair ? kTmemCols : 256;
  static constexpr size_t kSmem = kSingle ? kTileBytes * 5 + 256
                                          : (size_t)kTileBytes * (kNq + 2 * kSt) + kNq * kPBytes + 256;
};

template <int MODE, bool MASK>     // MASK: some key block is partial (or causal)
__global__ void __launch_bounds__(AttnCfg<MODE>::kThr, AttnCfg<MODE>::kMinBlocks)
attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  using Cfg = AttnCfg<MODE>;
  constexpr bool SINGLE = Cfg::kSingle;
  constexpr int NQ = Cfg::kNq;
  constexpr int kSt = Cfg::kSt;
  constexpr uint32_t kCols = Cfg::kCols;
  constexpr int kTmaWarp = 4 * NQ, kMmaWarp = 4 * NQ + 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                  // NQ tiles
  uint8_t* sK = sQ + NQ * kTileBytes;
  uint8_t* sV = sK + kSt * kTileBytes;
  uint8_t* sP = sV + kSt * kTileBytes;                // 2 tiles (one P buffer per query tile)
  // SINGLE: P_0 overwrites Q_0|Q_1 and P_1 overwrites K|X once both S MMAs are done
  // (80 KB in all instead of 128 KB), so two CTAs fit an SM
  uint64_t* bars = reinterpret_cast<uint64_t*>(SINGLE ? sP + kTileBytes : sP + NQ * kPBytes);
  auto p_atom = [&](int q, int a) -> uint8_t* {       // 64-key SW128 atom a of P_q
    if constexpr (SINGLE) return q == 0 ? sQ + a * kTileBytes : (a == 0 ? sK : sP);
    return sP + q * kPBytes + a * (kBQ * 128);
  };
  uint64_t* q_full = bars;
  uint64_t* kv_full = q_full + 1;
  uint64_t* kv_empty = kv_full + kSt;
  uint64_t* s_full = kv_empty + kSt;       // [2] per query tile
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* o_done = p_full + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = blockIdx.x * NQ * kBQ;
  const int J = SINGLE ? 1 : p.n_kv;

  if (warp == kTmaWarp && lane == 0) {
    prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < kSt; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&p_full[i], 4); mbar_init(&o_done[i], 1); }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<kCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == kTmaWarp) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, NQ * kTileBytes);
#pragma unroll
      for (int q = 0; q < NQ; ++q) tma_load_3d(sQ + q * kTileBytes, &tmQ, q_full, p.q_col0 + h * kD, q0 + q * kBQ, b);
      for (int j = 0; j < J; ++j) {
        const int s = j % kSt;
        mbar_wait(&kv_empty[s], ((j / kSt) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[s], 2 * kTileBytes);
        tma_load_3d(sK + s * kTileBytes, &tmK, &kv_full[s], p.k_col0 + h * kD, j * kBK, b);
        tma_load_3d(sV + s * kTileBytes, &tmV, &kv_full[s], p.v_col0 + h * kD, j * kBK, b);
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      mbar_wait(q_full, 0);
      auto issue_s = [&](int q, int j) {
        const int s = j % kSt;
        const uint64_t dq = sdesc_sw128_kmajor(sQ + q * kTileBytes);
        const uint64_t dk = sdesc_sw128_kmajor(sK + s * kTileBytes);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) umma_bf16(tmem + q * kBK, dq + 2 * k, dk + 2 * k, kIdescS, k > 0 ? 1u : 0u);
        umma_commit(&s_full[q]);
      };
      auto issue_pv = [&](int q, int j, bool wait) {
        const int s = j % kSt;
        if (wait) {
          mbar_wait(&p_full[q], j & 1);
          tc_fence_after();
        }
        const uint32_t d_o = tmem + (SINGLE ? q * kBK : NQ * kBK + q * kD);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint64_t da = sdesc_sw128_kmajor(p_atom(q, k >> 2)) + 2 * (k & 3);
          const uint64_t dv = sdesc_sw128_mnmajor(sV + s * kTileBytes + k * 2048, 8192);
          umma_bf16(d_o, da, dv, kIdescO, (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&o_done[q]);
      };
      for (int j = 0; j < J; ++j) {
        mbar_wait(&kv_full[j % kSt], (j / kSt) & 1);
        tc_fence_after();
        for (int q = 0; q < NQ; ++q) {
          if (j > 0) {
            // S_q(j) overwrites S_q(j-1): the softmax has consumed it once P_q(j-1) is out
            mbar_wait(&p_full[q], (j - 1) & 1);
            tc_fence_after();
          }
          issue_s(q, j);
          if (j > 0) {
            issue_pv(q, j - 1, false);      // P_q(j-1) was waited for above
            if (q == NQ - 1) umma_commit(&kv_empty[(j - 1) % kSt]);
          }
        }
      }
      for (int q = 0; q < NQ; ++q) issue_pv(q, J - 1, true);
      umma_commit(&kv_empty[(J - 1) % kSt]);
    }
  } else {
    // ------------------------------ softmax ------------------------------
    const int q = warp >> 2;                  // query tile of this warpgroup
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_s = tmem + lane_base + q * kBK;
    const uint32_t t_o = tmem + lane_base + (SINGLE ? q * kBK : NQ * kBK + q * kD);
    float m_run = -INFINITY, l_run = 0.f;
    const uint64_t scale2 = pack2(p.scale_log2, p.scale_log2);
    for (int j = 0; j < J; ++j) {
      mbar_wait(&s_full[q], j & 1);
      tc_fence_after();
      // keys of this block this row may see: the sequence end and, when causal (single
      // block), the row's own position
      const int valid = p.causal ? min(min(kBK, p.skv - j * kBK), q0 + q * kBQ + row - j * kBK + 1)
                                 : min(kBK, p.skv - j * kBK);
      // pass 1: block row max straight from TMEM (32 columns at a time)
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kBK / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_s + c * 32, r);
        tmem_ld_wait();
        if (MASK && valid < kBK) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i >= valid) r[i] = __float_as_uint(-INFINITY);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(r[i]));
      }
      const float m_blk = mx * p.scale_log2;
      // lazy rescale: move the reference max only when it grows by > 2^8
      const bool grow = (j == 0) || (m_blk > m_run + kRescaleThreshold);
      if (!SINGLE && j > 0) {
        // PV(j-1) must be complete before O is rescaled or P is overwritten
        mbar_wait(&o_done[q], (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, grow)) {
          const float alpha = grow ? ex2f(m_run - fmaxf(m_run, m_blk)) : 1.0f;
          uint32_t o[32];
#pragma unroll
          for (int c = 0; c < kD / 32; ++c) {
            tmem_ld_32x32b_x32(t_o + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_32x32b_x32(t_o + c * 32, o);
          }
          tmem_st_wait();
          if (grow) l_run *= alpha;
        }
      }
      if (grow) m_run = fmaxf(m_run, m_blk);
      const uint64_t negm2 = pack2(-m_run, -m_run);
      uint64_t sum2 = 0ull;
      if constexpr (SINGLE) {
        // P overwrites Q and K: both tiles' score MMAs must have finished reading them
        // (the commit behind S_1 covers S_0 too)
        if (q == 0) {
          mbar_wait(&s_full[1], 0);
          tc_fence_after();
        }
      }
      // pass 2: P = 2^(s*scale - m) in packed fp32 pairs; 3 of 8 pairs on the FMA-pipe polynomial
#pragma unroll
      for (int c = 0; c < kBK / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_s + c * 32, r);
        tmem_ld_wait();
        if (MASK && valid < kBK) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i >= valid) r[i] = __float_as_uint(-INFINITY);
        }
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const uint64_t x2 = ffma2(pack2u(r[i], r[i + 1]), scale2, negm2);
          uint64_t e2;
          const int pr = (i >> 1) & 7;
          if (pr == 2 || pr == 5 || pr == 7) {
            e2 = exp2_poly2(x2);
          } else {
            e2 = pack2(ex2f(lo2(x2)), ex2f(hi2(x2)));
          }
          sum2 = fadd2(sum2, e2);
          packed[i / 2] = pack_bf16(lo2(e2), hi2(e2));
        }
        uint8_t* atom = p_atom(q, c >> 1) + row * 128;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int chunk = ((c & 1) * 4 + qq) ^ (row & 7);
          *reinterpret_cast<uint4*>(atom + chunk * 16) =
              make_uint4(packed[4 * qq], packed[4 * qq + 1], packed[4 * qq + 2], packed[4 * qq + 3]);
        }
      }
      l_run += lo2(sum2) + hi2(sum2);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[q]);
    }
    mbar_wait(&o_done[q], (J - 1) & 1);
    tc_fence_after();
    const int qrow = q0 + q * kBQ + row;
    const float inv = 1.0f / l_run;
    uint32_t o[32];
#pragma unroll
    for (int c = 0; c < kD / 32; ++c) {
      tmem_ld_32x32b_x32(t_o + c * 32, o);
      tmem_ld_wait();
      if (qrow < p.sq) {
        __nv_bfloat16* dst = p.o + ((long long)b * p.sq + qrow) * p.ldo + h * kD + c * 32;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          uint4 u = make_uint4(pack_bf16(__uint_as_float(o[8 * qq]) * inv, __uint_as_float(o[8 * qq + 1]) * inv),
                               pack_bf16(__uint_as_float(o[8 * qq + 2]) * inv, __uint_as_float(o[8 * qq + 3]) * inv),
                               pack_bf16(__uint_as_float(o[8 * qq + 4]) * inv, __uint_as_float(o[8 * qq + 5]) * inv),
                               pack_bf16(__uint_as_float(o[8 * qq + 6]) * inv, __uint_as_float(o[8 * qq + 7]) * inv));
          reinterpret_cast<uint4*>(dst)[qq] = u;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<kCols>(tmem);
}

// ---------------------------------------------------------------------------
// Split-KV CTA: ONE query tile, its key range cut in two halves that the two
// softmax warpgroups ("streams") process concurrently against their own K/V rings,
// S / P buffers and O accumulators; the halves are merged in the CTA at the end
// (m = max(m0, m1), O = sum_h 2^(m_h - m) O_h, l likewise). Units are query tiles,
// twice as many as two-tile CTAs, so the last partial wave on 148 SMs is half as
// long. The split point depends on S_kv only: an image's rows are computed
// identically whatever else is in the batch.
constexpr int kStSplit = 2;

template <bool MASK>             // MASK: S_kv is not a multiple of the 128-key block
__global__ void __launch_bounds__(kThreads, 1)
attn_splitkv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                        // 1 tile
  uint8_t* sK = sQ + kTileBytes;                             // [stream][stage]
  uint8_t* sV = sK + 2 * kStSplit * kTileBytes;              // [stream][stage]
  // P_q lives in TMEM columns [384 + 64 q, 448 + 64 q) (bf16 pairs), read by a TS-MMA
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * kStSplit * kTileBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = q_full + 1;                            // [stream][stage]
  uint64_t* kv_empty = kv_full + 2 * kStSplit;
  uint64_t* s_full = kv_empty + 2 * kStSplit;                // [stream]
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  float* s_ml = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);   // [stream][2][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = blockIdx.x * kBQ;
  const int J = p.n_kv;
  const int jh = (J + 1) / 2;
  const int jb[2] = {0, jh}, nj[2] = {jh, J - jh};

  if (warp == 8 && lane == 0) {
    prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2 * kStSplit; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&p_full[i], 4); mbar_init(&o_done[i], 1); }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  auto k_at = [&](int q, int s) { return sK + (q * kStSplit + s) * kTileBytes; };
  auto v_at = [&](int q, int s) { return sV + (q * kStSplit + s) * kTileBytes; };
  if (warp == 8) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, kTileBytes);
      tma_load_3d(sQ, &tmQ, q_full, p.q_col0 + h * kD, q0, b);
      for (int i = 0; i < jh; ++i) {
        for (int q = 0; q < 2; ++q) {
          if (i >= nj[q]) continue;
          const int s = i % kStSplit, bi = q * kStSplit + s, g = jb[q] + i;
          mbar_wait(&kv_empty[bi], ((i / kStSplit) & 1) ^ 1);
          mbar_arrive_expect_tx(&kv_full[bi], 2 * kTileBytes);
          tma_load_3d(k_at(q, s), &tmK, &kv_full[bi], p.k_col0 + h * kD, g * kBK, b);
          tma_load_3d(v_at(q, s), &tmV, &kv_full[bi], p.v_col0 + h * kD, g * kBK, b);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      mbar_wait(q_full, 0);
      const uint64_t dq = sdesc_sw128_kmajor(sQ);
      auto issue_s = [&](int q, int i) {
        const uint64_t dk = sdesc_sw128_kmajor(k_at(q, i % kStSplit));
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) umma_bf16(tmem + q * kBK, dq + 2 * k, dk + 2 * k, kIdescS, k > 0 ? 1u : 0u);
        umma_commit(&s_full[q]);
      };
      auto issue_pv = [&](int q, int i) {
        const uint8_t* v = v_at(q, i % kStSplit);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint64_t dv = sdesc_sw128_mnmajor(v + k * 2048, 8192);
          umma_bf16_ts(tmem + 256 + q * kD, tmem + 384 + q * 64 + 8 * k, dv, kIdescO, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&o_done[q]);
        umma_commit(&kv_empty[q * kStSplit + i % kStSplit]);
      };
      for (int i = 0; i < jh; ++i) {
        for (int q = 0; q < 2; ++q) {
          if (i >= nj[q]) continue;
          const int bi = q * kStSplit + i % kStSplit;
          mbar_wait(&kv_full[bi], (i / kStSplit) & 1);
          tc_fence_after();
          if (i > 0) {                       // S_q(i) overwrites S_q(i-1): P_q(i-1) is out
            mbar_wait(&p_full[q], (i - 1) & 1);
            tc_fence_after();
          }
          issue_s(q, i);
          if (i > 0) issue_pv(q, i - 1);
        }
      }
      for (int q = 0; q < 2; ++q) {
        mbar_wait(&p_full[q], (nj[q] - 1) & 1);
        tc_fence_after();
        issue_pv(q, nj[q] - 1);
      }
    }
  } else {
    // ------------------------------ softmax: stream q over key blocks jb[q] .. ------------------------------
    const int q = warp >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_s = tmem + lane_base + q * kBK;
    const uint32_t t_o = tmem + lane_base + 256 + q * kD;
    const uint32_t t_p = tmem + lane_base + 384 + q * 64;
    float m_run = -INFINITY, l_run = 0.f;
    const uint64_t scale2 = pack2(p.scale_log2, p.scale_log2);
    const int n = nj[q];
    for (int i = 0; i < n; ++i) {
      mbar_wait(&s_full[q], i & 1);
      tc_fence_after();
      const int valid = min(kBK, p.skv - (jb[q] + i) * kBK);
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kBK / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_s + c * 32, r);
        tmem_ld_wait();
        if (MASK && valid < kBK) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (c * 32 + e >= valid) r[e] = __float_as_uint(-INFINITY);
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) mx = fmaxf(mx, __uint_as_float(r[e]));
      }
      const float m_blk = mx * p.scale_log2;
      const bool grow = (i == 0) || (m_blk > m_run + kRescaleThreshold);
      if (i > 0) {
        mbar_wait(&o_done[q], (i - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, grow)) {
          const float alpha = grow ? ex2f(m_run - fmaxf(m_run, m_blk)) : 1.0f;
          uint32_t o[32];
#pragma unroll
          for (int c = 0; c < kD / 32; ++c) {
            tmem_ld_32x32b_x32(t_o + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st_32x32b_x32(t_o + c * 32, o);
          }
          tmem_st_wait();
          if (grow) l_run *= alpha;
        }
      }
      if (grow) m_run = fmaxf(m_run, m_blk);
      const uint64_t negm2 = pack2(-m_run, -m_run);
      uint64_t sum2 = 0ull;
#pragma unroll
      for (int c = 0; c < kBK / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_s + c * 32, r);
        tmem_ld_wait();
        if (MASK && valid < kBK) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (c * 32 + e >= valid) r[e] = __float_as_uint(-INFINITY);
        }
        uint32_t packed[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const uint64_t x2 = ffma2(pack2u(r[e], r[e + 1]), scale2, negm2);
          uint64_t e2;
          const int pr = (e >> 1) & 7;
          if (pr == 2 || pr == 5 || pr == 7) e2 = exp2_poly2(x2);
          else e2 = pack2(ex2f(lo2(x2)), ex2f(hi2(x2)));
          sum2 = fadd2(sum2, e2);
          packed[e / 2] = pack_bf16(lo2(e2), hi2(e2));
        }
        tmem_st_32x32b_x16(t_p + c * 16, packed);
      }
      l_run += lo2(sum2) + hi2(sum2);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[q]);
    }
    mbar_wait(&o_done[q], (n - 1) & 1);
    tc_fence_after();
    // merge the two halves: both warpgroups reach every O column of their rows
    s_ml[(q * 2 + 0) * kBQ + row] = m_run;
    s_ml[(q * 2 + 1) * kBQ + row] = l_run;
    tc_fence_before();
    asm volatile("bar.sync 1, 256;" ::: "memory");
    tc_fence_after();
    const float m0 = s_ml[0 * kBQ + row], l0 = s_ml[1 * kBQ + row];
    const float m1 = s_ml[2 * kBQ + row], l1 = s_ml[3 * kBQ + row];
    const float m = fmaxf(m0, m1);
    const float a0 = ex2f(m0 - m), a1 = ex2f(m1 - m);
    const float inv = 1.0f / (a0 * l0 + a1 * l1);
    const float w0 = a0 * inv, w1 = a1 * inv;
    const int qrow = q0 + row;
    // warpgroup q writes output columns [32q, 32q + 32)
    uint32_t o0[32], o1[32];
    tmem_ld_32x32b_x32(tmem + lane_base + 256 + q * 32, o0);
    tmem_ld_32x32b_x32(tmem + lane_base + 256 + kD + q * 32, o1);
    tmem_ld_wait();
    if (qrow < p.sq) {
      __nv_bfloat16* dst = p.o + ((long long)b * p.sq + qrow) * p.ldo + h * kD + q * 32;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          v[e] = fmaf(__uint_as_float(o0[8 * qq + e]), w0, __uint_as_float(o1[8 * qq + e]) * w1);
        reinterpret_cast<uint4*>(dst)[qq] = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                                                       pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc<kTmemCols>(tmem);
}

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

// 3-D map over [batch][rows][ld] bf16 with a (64 cols, 128 rows, 1) box
bool map3(CUtensorMap* m, const void* base, long long ld, int rows, int batch) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)ld, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t str[2] = {(cuuint64_t)ld * 2, (cuuint64_t)ld * 2 * rows};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE, bool MASK>
int launch_attn(dim3 grid, cudaStream_t st, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                const AttnParams& p, size_t slack) {
  const size_t smem = AttnCfg<MODE>::kSmem + slack;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_kernel<MODE, MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return HP_ERR_CUDA;
    attr = true;
  }
  return hp_launch_pdl(attn_kernel<MODE, MASK>, grid, dim3(AttnCfg<MODE>::kThr), smem, st, tq, tk, tv, p) ==
                 cudaSuccess
             ? HP_OK : HP_ERR_CUDA;
}

int num_sms_attn() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

bool splitkv_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HP_ATTN_SPLITKV");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

}  // namespace

extern "C" int hp_attention(const hp_attn_desc* d, void* stream) {
  if (!d || !d->q || !d->k || !d->v || !d->o) return HP_ERR_PARAMETER;
  if (d->batch < 1 || d->heads < 1 || d->sq < 1 || d->skv < 1) return HP_ERR_SHAPE;
  if ((d->ldq | d->ldk | d->ldv | d->ldo) % 8) return HP_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(d->q) | reinterpret_cast<uintptr_t>(d->k) | reinterpret_cast<uintptr_t>(d->v) |
       reinterpret_cast<uintptr_t>(d->o)) & 15)
    return HP_ERR_UNSUPPORTED;
  CUtensorMap tq, tk, tv;
  if (!map3(&tq, d->q, d->ldq, d->sq, d->batch) || !map3(&tk, d->k, d->ldk, d->skv, d->batch) ||
      !map3(&tv, d->v, d->ldv, d->skv, d->batch))
    return HP_ERR_CUDA;
  AttnParams p{};
  p.sq = d->sq; p.skv = d->skv; p.heads = d->heads;
  p.causal = d->causal ? 1 : 0;
  if (p.causal && d->skv > kBK) return HP_ERR_UNSUPPORTED;    // single key block only (text encoders)
  p.q_col0 = (int)d->q_col0; p.k_col0 = (int)d->k_col0; p.v_col0 = (int)d->v_col0;
  p.o = static_cast<__nv_bfloat16*>(d->o); p.ldo = d->ldo;
  p.scale_log2 = d->scale * 1.4426950408889634f;
  p.n_kv = (d->skv + kBK - 1) / kBK;
  dim3 grid((d->sq + 2 * kBQ - 1) / (2 * kBQ), d->heads, d->batch);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p.n_kv == 1) return launch_attn<kModeSingle, true>(grid, st, tq, tk, tv, p, 1024);
  const bool mask = (d->skv % kBK) != 0;
  // one query tile per CTA when the two-tile grid would leave a short last wave
  const int pair_ctas = grid.x * grid.y * grid.z;
  const int sms = num_sms_attn();
  const int tail = pair_ctas % sms;
  if (splitkv_enabled() && tail != 0 && tail * 2 < sms) {
    constexpr size_t smem = 1024 + (size_t)kTileBytes * (1 + 4 * kStSplit) + 256 + 4 * kBQ * 4;
    static bool attr_s = false;
    if (!attr_s) {
      if (cudaFuncSetAttribute(attn_splitkv_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
              cudaSuccess ||
          cudaFuncSetAttribute(attn_splitkv_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
              cudaSuccess)
        return HP_ERR_CUDA;
      attr_s = true;
    }
    dim3 g1((d->sq + kBQ - 1) / kBQ, d->heads, d->batch);
    const auto kern = (d->skv % kBK) ? attn_splitkv_kernel<true> : attn_splitkv_kernel<false>;
    return hp_launch_pdl(kern, g1, dim3(kThreads), smem, st, tq, tk, tv, p) == cudaSuccess ? HP_OK : HP_ERR_CUDA;
  }
  return mask ? launch_attn<kModePair, true>(grid, st, tq, tk, tv, p, 1024)
              : launch_attn<kModePair, false>(grid, st, tq, tk, tv, p, 1024);
}
