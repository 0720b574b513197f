// hp_attn.cu — K5: fused multi-head attention (head_dim 64) on tcgen05.
//
// Two kernels (hp_attention picks one):
//   attn_single_kernel   S_kv <= 128 (cross-attention, causal text-encoder
//                        attention): one query tile per CTA, each row's keys
//                        split between two softmax warps, 3 CTAs/SM.
//   attn_stream_kernel   everything else, persistent (one CTA per SM walks the
//                        work units): two softmax "streams" per CTA, each
//                        with its own score-MMA and PV-MMA issuing warp; the
//                        128-score row is pulled into registers in one TMEM
//                        load and S released at once, so S(i+1) = Q K(i+1)^T
//                        runs on the tensor core while the softmax of block i
//                        computes its exponentials. PAIR: stream = query tile
//                        (two per CTA, shared K/V ring); SPLIT (when the PAIR
//                        grid leaves a short last wave): one query tile, key
//                        range halved between the streams (fixed split point:
//                        batch-invariant), halves merged at the end.
// Softmax (per row, fp32, log2 domain): block max, lazy rescale of O in TMEM only
// when the running max grows by more than 2^8 (otherwise the stale max is kept:
// p <= 2^8, exact after the final 1/l), exp2 split between MUFU.EX2 and a degree-3
// polynomial on the FMA pipe (P is rounded to bf16 anyway); P is stored to TMEM as
// bf16 pairs and read by a TS-MMA (O += P V, V MN-major straight from its TMA tile).
// Round-2 measurements (tools/attn_ab.py, tools/micro/attn_trace.cu, profiles/r02):
// S=4096 B=2 H=10: 151 -> 128 us; S=1024 B=2 H=20: 30 -> 25.8 us; SD3 S=4429 B=2
// H=24: 420 -> 307 us. The period per 128-key block pair is ~2500 clk against
// ~1240 clk of tensor work (PV at N=64 runs at 45 clk per K=16 step, not 32) and
// ~1300 clk of MUFU: the softmax's issue/latency chain is the limit.
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
constexpr uint32_t kTileBytes = kBQ * kD * 2;        // 16 KB (Q, K or V tile)
constexpr uint32_t kIdescS = idesc_bf16_f32(kBQ, kBK, 0);
constexpr uint32_t kIdescO = idesc_bf16_f32(kBQ, kD, 1);  // B (= V) MN-major
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;            // log2 units

struct AttnParams {
  int sq, skv, heads, batch;
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

// Single-block kernel: every key fits one 128-key block (cross-attention, skv <=
// 128, and the text encoders' causal attention). One CTA = one 128-query tile, 288
// threads: warps 0-7 softmax (warp w owns TMEM lane quarter w & 3 and key half
// w >> 2, in 16-key units: 3 + 2 units for the 77-token context), warp 8 TMA + MMA
// issue + TMEM allocation. The chain load -> score MMA -> softmax -> PV -> store is
// pure latency at these sizes, so it is kept short: two warps per row halve the
// softmax leg (row max and sum meet in shared memory), and three CTAs share an SM
// so the tiles of a B=2 launch (320 at level 3) are all resident in one wave. P
// overwrites Q (keys 0-63) and K (64-127) once the score MMA has read them; O
// reuses the score columns in TMEM.
#ifdef HP_ATTN_TRACE
__device__ long long g_single_trace[16];
#define HP_STRACE(cond, ev) do { if ((cond) && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) \
                                   g_single_trace[ev] = clock64(); } while (0)
#else
#define HP_STRACE(cond, ev) do {} while (0)
#endif
constexpr int kSingleThreads = 288;
constexpr uint32_t kSingleCols = 128;
constexpr size_t kSingleSmem = (size_t)kTileBytes * 3 + 64 + 4 * 128 * 4;   // Q K V | barriers | max, sum

__device__ __forceinline__ void tmem_ld_x16_at(uint32_t taddr, uint32_t* r, const int base) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : HP_R8(base), HP_R8(base + 8)
      : "r"(taddr));
}

template <bool MASK>     // MASK: the key block is partial (or causal)
__global__ void __launch_bounds__(kSingleThreads, 3)
attn_single_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  constexpr int kIssueWarp = 8;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kTileBytes;
  uint8_t* sV = sK + kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kTileBytes);
  uint64_t* qk_full = bars;
  uint64_t* v_full = bars + 1;
  uint64_t* s_full = bars + 2;
  uint64_t* p_full = bars + 3;               // 8 softmax warps
  uint64_t* o_done = bars + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);
  float* s_max = reinterpret_cast<float*>(bars + 8);     // [half][row]
  float* s_sum = s_max + 2 * kBQ;                        // [half][row]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  HP_STRACE(threadIdx.x == 0, 0);
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = blockIdx.x * kBQ;
  const int ns = min(kBK, (p.skv + 15) & ~15);        // key columns computed (multiple of 16)
  const int nu = ns >> 4;                             // 16-key units

  if (warp == kIssueWarp) {
    if (lane == 0) {
      prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmV);
      mbar_init(qk_full, 1);
      mbar_init(v_full, 1);
      mbar_init(s_full, 1);
      mbar_init(p_full, 8);
      mbar_init(o_done, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc<kSingleCols>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  HP_STRACE(threadIdx.x == 0, 1);
  pdl_trigger();

  if (warp == kIssueWarp) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qk_full, 2 * kTileBytes);
      tma_load_3d(sQ, &tmQ, qk_full, p.q_col0 + h * kD, q0, b);
      tma_load_3d(sK, &tmK, qk_full, p.k_col0 + h * kD, 0, b);
      mbar_arrive_expect_tx(v_full, kTileBytes);
      tma_load_3d(sV, &tmV, v_full, p.v_col0 + h * kD, 0, b);
      mbar_wait(qk_full, 0);
      HP_STRACE(true, 2);
      tc_fence_after();
      const uint64_t dq = sdesc_sw128_kmajor(sQ), dk = sdesc_sw128_kmajor(sK);
      // only the keys that exist: N = S_kv rounded up to 16 (77 -> 80 for the text context)
      const uint32_t idesc_s = idesc_bf16_f32(kBQ, (uint32_t)ns, 0);
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) umma_bf16(tmem, dq + 2 * k, dk + 2 * k, idesc_s, k > 0 ? 1u : 0u);
      umma_commit(s_full);
      HP_STRACE(true, 3);
      mbar_wait(v_full, 0);
      mbar_wait(p_full, 0);
      tc_fence_after();
      for (int k = 0; k < nu; ++k) {
        const uint64_t da = sdesc_sw128_kmajor(k < 4 ? sQ : sK) + 2 * (k & 3);
        const uint64_t dv = sdesc_sw128_mnmajor(sV + k * 2048, 8192);
        umma_bf16(tmem, da, dv, kIdescO, k > 0 ? 1u : 0u);
      }
      umma_commit(o_done);
    }
  } else {
    // ------------------------------ softmax ------------------------------
    const int quarter = warp & 3, half = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t t_s = tmem + ((uint32_t)(quarter * 32) << 16);
    const int u0 = half ? (nu + 1) >> 1 : 0, u1 = half ? nu : (nu + 1) >> 1;
    const uint64_t scale2 = pack2(p.scale_log2, p.scale_log2);
    // keys this row may see: the sequence end and, when causal, the row's own position
    const int valid = p.causal ? min(min(kBK, p.skv), q0 + row + 1) : min(kBK, p.skv);
    mbar_wait(s_full, 0);
    HP_STRACE(threadIdx.x == 0, 4);
    tc_fence_after();
    // pass 1: this half's row max, two units per TMEM round trip
    float mx = -INFINITY;
    for (int u = u0; u < u1; u += 2) {
      uint32_t r[32];
      tmem_ld_x16_at(t_s + u * 16, r, 0);
      if (u + 1 < u1) tmem_ld_x16_at(t_s + u * 16 + 16, r, 16);
      tmem_ld_wait();
      const int n = u + 1 < u1 ? 32 : 16;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < n && (!MASK || u * 16 + i < valid)) mx = fmaxf(mx, __uint_as_float(r[i]));
    }
    s_max[half * kBQ + row] = mx;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    mx = fmaxf(s_max[row], s_max[kBQ + row]);
    const float m = mx * p.scale_log2;
    const uint64_t negm2 = pack2(-m, -m);
    // pass 2: P = 2^(s*scale - m) in packed fp32 pairs, 2 of 8 pairs on the FMA-pipe polynomial;
    // P overwrites Q / K, which the score MMA (complete: s_full) no longer reads
    uint64_t sum2[4] = {0ull, 0ull, 0ull, 0ull};
    for (int u = u0; u < u1; ++u) {
      uint32_t r[16];
      tmem_ld_x16_at(t_s + u * 16, r, 0);
      tmem_ld_wait();
      if (MASK && valid < (u + 1) * 16) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (u * 16 + i >= valid) r[i] = __float_as_uint(-INFINITY);
      }
      uint32_t packed[8];
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const uint64_t x2 = ffma2(pack2u(r[i], r[i + 1]), scale2, negm2);
        uint64_t e2;
        const int pr = i >> 1;
        if (pr == 3 || pr == 7) e2 = exp2_poly2(x2);
        else e2 = pack2(ex2f(lo2(x2)), ex2f(hi2(x2)));
        sum2[pr & 3] = fadd2(sum2[pr & 3], e2);
        packed[pr] = pack_bf16(lo2(e2), hi2(e2));
      }
      uint8_t* atom = (u < 4 ? sQ : sK) + row * 128;
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int chunk = ((u & 3) * 2 + qq) ^ (row & 7);
        *reinterpret_cast<uint4*>(atom + chunk * 16) =
            make_uint4(packed[4 * qq], packed[4 * qq + 1], packed[4 * qq + 2], packed[4 * qq + 3]);
      }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(p_full);
    HP_STRACE(threadIdx.x == 0, 5);
    const uint64_t s01 = fadd2(fadd2(sum2[0], sum2[1]), fadd2(sum2[2], sum2[3]));
    s_sum[half * kBQ + row] = lo2(s01) + hi2(s01);
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const float inv = 1.0f / (s_sum[row] + s_sum[kBQ + row]);
    mbar_wait(o_done, 0);
    HP_STRACE(threadIdx.x == 0, 6);
    tc_fence_after();
    // O (64 columns, over the score columns): this warp stores its half of the row
    uint32_t o[32];
    tmem_ld_32x32b_x32(t_s + half * 32, o);
    tmem_ld_wait();
    const int qrow = q0 + row;
    if (qrow < p.sq) {
      __nv_bfloat16* dst = p.o + ((long long)b * p.sq + qrow) * p.ldo + h * kD + half * 32;
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
  HP_STRACE(threadIdx.x == 0, 7);
  tc_fence_before();
  __syncthreads();
  HP_STRACE(threadIdx.x == 0, 8);
  tc_fence_after();
  if (warp == kIssueWarp) tmem_dealloc<kSingleCols>(tmem);
}

// ---------------------------------------------------------------------------
// Streaming kernel (round 2): two independent softmax "streams" per CTA, each with
// its OWN MMA-issue warp, and the score tile released as soon as the softmax has
// pulled it into registers, so S(i+1) = Q K(i+1)^T runs on the tensor core while
// the softmax of block i is still computing exponentials. (The round-1 kernels
// re-read S from TMEM in a second pass, so S(i+1) could only start after P(i) was
// out: ncu showed the softmax warps parked on the score barrier 1/3 of the time.)
//   PAIR  (SPLIT=false): stream q = query tile q of the CTA (256 queries), K/V
//          ring shared by both streams (a slot is released by both PV commits).
//   SPLIT (SPLIT=true):  one query tile, key range cut in two halves (fixed split
//          point: batch-invariant), one K/V ring per stream, halves merged at the end.
// 512 threads: warps 0-3 / 4-7 softmax of stream 0 / 1 (thread = query row),
// warp 8 TMA (warp 9 the second K/V producer in SPLIT), warps 10 / 11 issue the
// score MMAs of stream 0 / 1, warps 12 / 13 the PV MMAs (tcgen05.mma holds its
// issuing thread until the tensor pipe accepts it, and tcgen05.commit tracks the
// issuing thread's MMAs: one issuer per (stream, kind) keeps S off PV's queue),
// warps 14-15 idle. setmaxnreg moves registers from warpgroups 2-3 (48 each) to
// the softmax warpgroups (208 each: the 128-score row stays in registers).
// TMEM (512 cols): S_q [128 q, +128), O_q [256 + 64 q, +64), P_q [384 + 64 q, +64)
// (P as bf16 pairs, the A operand of the TS-MMA O_q += P_q V).
// Softmax per block: one TMEM load of the 128-score row, s_free arrive, a depth-10
// FMNMX3 tree for the row max, exp2 (6/8 MUFU, 2/8 FMA polynomial) with four
// partial sums, then the O rescale (lazy, > 2^8 only) once PV(i-1) is done, P
// stored to TMEM, p_full arrive.
// Persistent: one CTA per SM walks work units (PAIR: 256 queries of one (head,
// batch); SPLIT: 128) round-robin, so barrier init, TMEM allocation and the launch
// happen once, and the next unit's Q / K / V loads and first score MMA overlap the
// current unit's last blocks and epilogue (Q double-buffered). Every unit is
// computed the same way wherever it runs: batch-invariant.
constexpr int kStrThreads = 512;
constexpr int kStrSplitStages = 2, kStrPairStages = 4;
template <bool SPLIT> struct StrCfg {
  static constexpr int kNq = SPLIT ? 1 : 2;                   // Q tiles per unit
  static constexpr int kSlots = SPLIT ? 2 * kStrSplitStages : kStrPairStages;
  static constexpr size_t kSmem = 1024 + (size_t)kTileBytes * (2 * kNq + 2 * kSlots) + 256 + 4 * kBQ * 4;
};

#ifdef HP_ATTN_TRACE
// event timeline of CTA 0 for tools/micro/attn_trace.cu: [stream][event][block]
__device__ long long g_attn_trace[2][12][256];
#define HP_TRACE(cond, q, ev, i) \
  do { if ((cond) && blockIdx.x == 0 && (i) < 256) g_attn_trace[q][ev][i] = clock64(); } while (0)
#else
#define HP_TRACE(cond, q, ev, i) do {} while (0)
#endif
template <bool SPLIT, bool MASK>   // MASK: S_kv is not a multiple of the 128-key block
__global__ void __launch_bounds__(kStrThreads, 1)
attn_stream_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  using Cfg = StrCfg<SPLIT>;
  constexpr int kSlots = Cfg::kSlots;
  constexpr int kNq = Cfg::kNq;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                          // [2 units][kNq tiles]
  uint8_t* sK = sQ + 2 * kNq * kTileBytes;                     // [slot]
  uint8_t* sV = sK + kSlots * kTileBytes;                      // [slot]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kSlots * kTileBytes);
  uint64_t* q_full = bars;                                     // [2]
  uint64_t* q_empty = q_full + 2;                              // [2]
  uint64_t* kv_full = q_empty + 2;                             // [kSlots]
  uint64_t* kv_empty = kv_full + kSlots;                       // [kSlots]
  uint64_t* s_full = kv_empty + kSlots;                        // [stream]
  uint64_t* s_free = s_full + 2;
  uint64_t* p_full = s_free + 2;
  uint64_t* o_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  float* s_ml = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);   // [stream][2][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int J = p.n_kv;
  const int jh = SPLIT ? (J + 1) / 2 : J;
  const int n_qt = (p.sq + kNq * kBQ - 1) / (kNq * kBQ);
  const int n_units = n_qt * p.heads * p.batch;
  // blocks of stream q within a unit: [jb(q), jb(q) + nj(q))
  auto jb = [&](int q) { return SPLIT ? q * jh : 0; };
  auto nj = [&](int q) { return SPLIT ? (q == 0 ? jh : J - jh) : J; };
  // ring slot / phase of stream q's running block index g (over all units of this CTA)
  auto slot = [&](int q, int g) { return SPLIT ? q * kStrSplitStages + g % kStrSplitStages : g % kStrPairStages; };
  auto phase = [&](int g) { return SPLIT ? (g / kStrSplitStages) & 1 : (g / kStrPairStages) & 1; };
  // unit u -> (query tile, head, batch)
  auto unit_q0 = [&](int u) { return (u % n_qt) * kNq * kBQ; };
  auto unit_h = [&](int u) { return (u / n_qt) % p.heads; };
  auto unit_b = [&](int u) { return u / (n_qt * p.heads); };

  if (warp == 8 && lane == 0) {
    prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmV);
    for (int i = 0; i < 2; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 2); }   // both S issuers
    for (int s = 0; s < kSlots; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], SPLIT ? 2 : 4); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&s_free[i], 4); mbar_init(&p_full[i], 4); mbar_init(&o_done[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 32;" ::: "memory");
  if (warp == 8 || (SPLIT && warp == 9)) {
    // producers: warp 8 loads Q and stream 0's K/V (PAIR: the shared ring), warp 9
    // stream 1's K/V (SPLIT), so one stream's full ring never stalls the other's loads
    if (lane == 0) {
      const int q = warp - 8;
      int g = 0;
      for (int u = blockIdx.x, k = 0; u < n_units; u += gridDim.x, ++k) {
        const int h = unit_h(u), b = unit_b(u);
        if (q == 0) {
          const int qs = k & 1;
          mbar_wait_park(&q_empty[qs], ((k >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[qs], kNq * kTileBytes);
#pragma unroll
          for (int t = 0; t < kNq; ++t)
            tma_load_3d(sQ + (qs * kNq + t) * kTileBytes, &tmQ, &q_full[qs], p.q_col0 + h * kD,
                        unit_q0(u) + t * kBQ, b);
        }
        for (int i = 0; i < nj(q); ++i, ++g) {
          const int s = slot(q, g), j = jb(q) + i;
          mbar_wait_park(&kv_empty[s], phase(g) ^ 1);
          mbar_arrive_expect_tx(&kv_full[s], 2 * kTileBytes);
          tma_load_3d(sK + s * kTileBytes, &tmK, &kv_full[s], p.k_col0 + h * kD, j * kBK, b);
          tma_load_3d(sV + s * kTileBytes, &tmV, &kv_full[s], p.v_col0 + h * kD, j * kBK, b);
        }
      }
    }
  } else if (warp == 10 || warp == 11) {
    // S issuer of stream q: S(g) as soon as K(g) is in and the softmax holds S(g-1)
    // in registers. tcgen05.mma holds the issuing thread until the tensor pipe takes
    // the instruction, so S and PV get separate issuers: a queued PV never delays S.
    const int q = warp - 10;
    if (lane == 0) {
      const uint32_t t_s = tmem + q * kBK;
      int g = 0;
      for (int u = blockIdx.x, k = 0; u < n_units; u += gridDim.x, ++k) {
        const int qs = k & 1;
        mbar_wait(&q_full[qs], (k >> 1) & 1);
        const uint64_t dq = sdesc_sw128_kmajor(sQ + (qs * kNq + (SPLIT ? 0 : q)) * kTileBytes);
        for (int i = 0; i < nj(q); ++i, ++g) {
          mbar_wait(&kv_full[slot(q, g)], phase(g));
          HP_TRACE(true, q, 0, g);
          if (g > 0) mbar_wait(&s_free[q], (g - 1) & 1);
          HP_TRACE(true, q, 1, g);
          tc_fence_after();
          const uint64_t dk = sdesc_sw128_kmajor(sK + slot(q, g) * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) umma_bf16(t_s, dq + 2 * kk, dk + 2 * kk, kIdescS, kk > 0 ? 1u : 0u);
          umma_commit(&s_full[q]);
          umma_commit(&kv_empty[slot(q, g)]);
          if (i == nj(q) - 1) umma_commit(&q_empty[qs]);      // this unit's Q is read
          HP_TRACE(true, q, 2, g);
        }
      }
    }
  } else if (warp == 12 || warp == 13) {
    // PV issuer of stream q: O_q (+)= P_q(g) V(g) once the softmax published P(g)
    const int q = warp - 12;
    if (lane == 0) {
      const uint32_t t_o = tmem + 256 + q * kD, t_p = tmem + 384 + q * 64;
      int g = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        for (int i = 0; i < nj(q); ++i, ++g) {
          mbar_wait(&p_full[q], g & 1);
          HP_TRACE(true, q, 3, g);
          tc_fence_after();
          const uint8_t* v = sV + slot(q, g) * kTileBytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t dv = sdesc_sw128_mnmajor(v + kk * 2048, 8192);
            umma_bf16_ts(t_o, t_p + 8 * kk, dv, kIdescO, (i > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&o_done[q]);
          umma_commit(&kv_empty[slot(q, g)]);
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
    // ------------------------------ softmax of stream q ------------------------------
    const int q = warp >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_s = tmem + lane_base + q * kBK;
    const uint32_t t_o = tmem + lane_base + 256 + q * kD;
    const uint32_t t_p = tmem + lane_base + 384 + q * 64;
    const uint64_t scale2 = pack2(p.scale_log2, p.scale_log2);
    int g = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int h = unit_h(u), b = unit_b(u), q0 = unit_q0(u);
      float m_run = -INFINITY, l_run = 0.f;
      const int n = nj(q);
      for (int i = 0; i < n; ++i, ++g) {
        HP_TRACE(quarter == 0 && lane == 0, q, 4, g);
        mbar_wait(&s_full[q], g & 1);
        HP_TRACE(quarter == 0 && lane == 0, q, 5, g);
        tc_fence_after();
        uint32_t r[128];
        tmem_ld_x32_at(t_s + 0, r, 0);
        tmem_ld_x32_at(t_s + 32, r, 32);
        tmem_ld_x32_at(t_s + 64, r, 64);
        tmem_ld_x32_at(t_s + 96, r, 96);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[q]);           // the S issuer may overwrite S now
        HP_TRACE(quarter == 0 && lane == 0, q, 6, g);
        if (MASK) {
          const int valid = min(kBK, p.skv - (jb(q) + i) * kBK);
          if (valid < kBK) {
#pragma unroll
            for (int e = 0; e < 128; ++e)
              if (e >= valid) r[e] = __float_as_uint(-INFINITY);
          }
        }
        // row max: 8 independent chains (FMNMX3 pairs), then a small tree
        float mx[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) mx[a] = __uint_as_float(r[a]);
#pragma unroll
        for (int e = 8; e < 128; e += 8) {
#pragma unroll
          for (int a = 0; a < 8; ++a) mx[a] = fmaxf(mx[a], __uint_as_float(r[e + a]));
        }
        const float m_blk = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                  fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * p.scale_log2;
        // lazy rescale: move the reference max only when it grows by > 2^8
        const bool grow = (i == 0) || (m_blk > m_run + kRescaleThreshold);
        const float m_new = grow ? fmaxf(m_run, m_blk) : m_run;
        const float alpha = grow ? ex2f(m_run - m_new) : 1.0f;     // i == 0: 2^-inf = 0
        const uint64_t negm2 = pack2(-m_new, -m_new);
        uint64_t sum2[4] = {0ull, 0ull, 0ull, 0ull};
        uint32_t packed[64];
#pragma unroll
        for (int e = 0; e < 128; e += 2) {
          const uint64_t x2 = ffma2(pack2u(r[e], r[e + 1]), scale2, negm2);
          uint64_t e2;
          const int pr = (e >> 1) & 7;
          if (pr == 3 || pr == 7) e2 = exp2_poly2(x2);   // 2 of 8 pairs on the FMA pipe
          else e2 = pack2(ex2f(lo2(x2)), ex2f(hi2(x2)));
          sum2[(e >> 1) & 3] = fadd2(sum2[(e >> 1) & 3], e2);
          packed[e >> 1] = pack_bf16(lo2(e2), hi2(e2));
        }
        HP_TRACE(quarter == 0 && lane == 0, q, 7, g);
        const uint64_t s01 = fadd2(fadd2(sum2[0], sum2[1]), fadd2(sum2[2], sum2[3]));
        l_run = l_run * alpha + (lo2(s01) + hi2(s01));
        m_run = m_new;
        if (i > 0) {
          // PV(g-1) must be complete before O is rescaled or P is overwritten (for
          // i == 0 the previous unit's epilogue already waited for its last PV)
          mbar_wait(&o_done[q], (g - 1) & 1);
          HP_TRACE(quarter == 0 && lane == 0, q, 8, g);
          tc_fence_after();
          if (__any_sync(0xffffffffu, grow)) {
            uint32_t o[32];
#pragma unroll
            for (int c = 0; c < kD / 32; ++c) {
              tmem_ld_32x32b_x32(t_o + c * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st_32x32b_x32(t_o + c * 32, o);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[e] = packed[c * 16 + e];
          tmem_st_32x32b_x16(t_p + c * 16, pk);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[q]);
        HP_TRACE(quarter == 0 && lane == 0, q, 9, g);
      }
      // ---- epilogue of this unit: O / l -> bf16 rows ----
      mbar_wait(&o_done[q], (g - 1) & 1);
      tc_fence_after();
      if constexpr (!SPLIT) {
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
              uint4 w = make_uint4(pack_bf16(__uint_as_float(o[8 * qq]) * inv, __uint_as_float(o[8 * qq + 1]) * inv),
                                   pack_bf16(__uint_as_float(o[8 * qq + 2]) * inv, __uint_as_float(o[8 * qq + 3]) * inv),
                                   pack_bf16(__uint_as_float(o[8 * qq + 4]) * inv, __uint_as_float(o[8 * qq + 5]) * inv),
                                   pack_bf16(__uint_as_float(o[8 * qq + 6]) * inv, __uint_as_float(o[8 * qq + 7]) * inv));
              reinterpret_cast<uint4*>(dst)[qq] = w;
            }
          }
        }
      } else {
        // merge the two halves: warpgroup q writes output columns [32q, 32q + 32) of
        // its rows from both streams' O, so both warpgroups meet before (statistics
        // exchange) and after (neither O may be overwritten while the other reads it)
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
        uint32_t o0[32], o1[32];
        tmem_ld_32x32b_x32(tmem + lane_base + 256 + q * 32, o0);
        tmem_ld_32x32b_x32(tmem + lane_base + 256 + kD + q * 32, o1);
        tmem_ld_wait();
        tc_fence_before();
        asm volatile("bar.sync 1, 256;" ::: "memory");
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

int launch_single(dim3 grid, cudaStream_t st, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                  const AttnParams& p) {
  constexpr size_t smem = kSingleSmem + 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_single_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return HP_ERR_CUDA;
    attr = true;
  }
  return hp_launch_pdl(attn_single_kernel<true>, grid, dim3(kSingleThreads), smem, st, tq, tk, tv, p) == cudaSuccess
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

// HP_ATTN_MODE: 0 auto, 1 two-tile, 2 split-KV (A/B switch)
int attn_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("HP_ATTN_MODE");
    m = (e && (e[0] == '1' || e[0] == '2')) ? e[0] - '0' : 0;
  }
  return m;
}

template <bool SPLIT, bool MASK>
int launch_stream(dim3 grid, cudaStream_t st, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                  const AttnParams& p) {
  constexpr size_t smem = StrCfg<SPLIT>::kSmem;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_stream_kernel<SPLIT, MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return HP_ERR_CUDA;
    attr = true;
  }
  return hp_launch_pdl(attn_stream_kernel<SPLIT, MASK>, grid, dim3(kStrThreads), smem, st, tq, tk, tv, p) ==
                 cudaSuccess ? HP_OK : HP_ERR_CUDA;
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
  p.sq = d->sq; p.skv = d->skv; p.heads = d->heads; p.batch = d->batch;
  p.causal = d->causal ? 1 : 0;
  if (p.causal && d->skv > kBK) return HP_ERR_UNSUPPORTED;    // single key block only (text encoders)
  p.q_col0 = (int)d->q_col0; p.k_col0 = (int)d->k_col0; p.v_col0 = (int)d->v_col0;
  p.o = static_cast<__nv_bfloat16*>(d->o); p.ldo = d->ldo;
  p.scale_log2 = d->scale * 1.4426950408889634f;
  p.n_kv = (d->skv + kBK - 1) / kBK;
  dim3 grid((d->sq + 2 * kBQ - 1) / (2 * kBQ), d->heads, d->batch);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p.n_kv == 1) return launch_single(dim3((d->sq + kBQ - 1) / kBQ, d->heads, d->batch), st, tq, tk, tv, p);
  const bool mask = (d->skv % kBK) != 0;
  // persistent CTAs over work units. The unit kind depends on the key count only, never
  // on batch or heads, so an image's rows are computed the same way whatever else is in
  // the batch (the condition-partitioned B=1 forwards equal the CFG-batched B=2 one):
  // split-KV units (one query tile, half the keys per stream, merged in the CTA) up to
  // 32 key blocks, where the finer units balance the SMs better (S=1024 / 4096), two-tile
  // units with shared K/V beyond (SD3's S=4429, S=16384), where K/V sharing wins.
  const int pair_units = grid.x * grid.y * grid.z;
  const int sms = num_sms_attn();
  const int mode = attn_mode();
  const bool split = mode == 2 || (mode == 0 && p.n_kv <= 32);
  const int units = split ? (int)((d->sq + kBQ - 1) / kBQ) * d->heads * d->batch : pair_units;
  const dim3 g1(units < sms ? units : sms);
  if (split)
    return mask ? launch_stream<true, true>(g1, st, tq, tk, tv, p) : launch_stream<true, false>(g1, st, tq, tk, tv, p);
  return mask ? launch_stream<false, true>(g1, st, tq, tk, tv, p) : launch_stream<false, false>(g1, st, tq, tk, tv, p);
}
