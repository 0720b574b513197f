// hp_attn.cu — K5: fused multi-head attention (head_dim 64) on tcgen05.
//
// One CTA per (128-query tile, head, batch). Warp roles:
//   warp 0      TMA: Q once, then K/V tiles of 128 keys through a 3-stage ring
//   warp 1      MMA: S(j) = Q K(j)^T into a double-buffered TMEM S (2 x 128 cols),
//               O~(j) = P(j) V(j) into a double-buffered TMEM O~ (2 x 64 cols);
//               V is consumed MN-major straight from its [keys][64] tile
//   warp 2      TMEM allocation
//   warps 4..7  softmax: thread i owns query row i; tcgen05.ld of S, online
//               max/exp2/sum in fp32 registers, P as bf16 written to a
//               double-buffered SW128 smem tile (the A operand of the PV MMA),
//               O accumulated in registers with the running rescale.
// S(j+1) is computed on the tensor core while the softmax warps work on S(j).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>
#include <mutex>
#include "hybridpar_b200_denoiser.h"
#include "hp_tc.cuh"

using namespace hptc;

namespace {

constexpr int kBQ = 128, kBK = 128, kD = 64;
constexpr int kStages = 3;
constexpr int kThreads = 256;
constexpr uint32_t kTileBytes = kBQ * kD * 2;        // 16 KB (Q, K or V tile)
constexpr uint32_t kPBytes = kBQ * kBK * 2;          // 32 KB (two 64-key SW128 atoms)
constexpr uint32_t kIdescS = idesc_bf16_f32(kBQ, kBK, 0);
constexpr uint32_t kIdescO = idesc_bf16_f32(kBQ, kD, 1);  // B (= V) MN-major
constexpr uint32_t kTmemCols = 512;                  // S0 S1 (256) + O0 O1 (128)
constexpr uint32_t kColS = 0, kColO = 256;

struct AttnParams {
  int sq, skv, heads;
  int q_col0, k_col0, v_col0;
  __nv_bfloat16* o; long long ldo;
  float scale_log2;
  int n_kv;
};

__global__ void __launch_bounds__(kThreads, 1)
attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kTileBytes;
  uint8_t* sV = sK + kStages * kTileBytes;
  uint8_t* sP = sV + kStages * kTileBytes;  // 2 buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * kPBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = q_full + 1;
  uint64_t* kv_empty = kv_full + kStages;
  uint64_t* s_full = kv_empty + kStages;   // [2]
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* o_full = p_full + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int q0 = qt * kBQ;
  const int J = p.n_kv;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&p_full[i], 4); mbar_init(&o_full[i], 1); }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, kTileBytes);
      tma_load_3d(sQ, &tmQ, q_full, p.q_col0 + h * kD, q0, b);
      for (int j = 0; j < J; ++j) {
        const int s = j % kStages;
        mbar_wait(&kv_empty[s], ((j / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[s], 2 * kTileBytes);
        tma_load_3d(sK + s * kTileBytes, &tmK, &kv_full[s], p.k_col0 + h * kD, j * kBK, b);
        tma_load_3d(sV + s * kTileBytes, &tmV, &kv_full[s], p.v_col0 + h * kD, j * kBK, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(q_full, 0);
      const uint64_t dq = sdesc_sw128_kmajor(sQ);
      auto issue_pv = [&](int j) {
        const int s = j % kStages, pb = j & 1;
        mbar_wait(&p_full[pb], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t d_o = tmem + kColO + pb * kD;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          // A = P: K-major, two 64-key atoms of 16 KB; B = V: MN-major, +16 keys = +2048 B
          const uint64_t da = sdesc_sw128_kmajor(sP + pb * kPBytes + (k >> 2) * (kBQ * 128)) + 2 * (k & 3);
          const uint64_t dv = sdesc_sw128_mnmajor(sV + s * kTileBytes + k * 2048, 8192);
          umma_bf16(d_o, da, dv, kIdescO, k > 0 ? 1u : 0u);
        }
        umma_commit(&o_full[pb]);
        umma_commit(&kv_empty[s]);
      };
      for (int j = 0; j < J; ++j) {
        const int s = j % kStages, sb = j & 1;
        mbar_wait(&kv_full[s], (j / kStages) & 1);
        tc_fence_after();
        const uint64_t dk = sdesc_sw128_kmajor(sK + s * kTileBytes);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) umma_bf16(tmem + kColS + sb * kBK, dq + 2 * k, dk + 2 * k, kIdescS, k > 0 ? 1u : 0u);
        umma_commit(&s_full[sb]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(J - 1);
    }
  } else if (warp >= 4) {
    // ------------------------------ softmax / correction ------------------------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;          // query row inside the tile
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    float o_acc[kD];
#pragma unroll
    for (int i = 0; i < kD; ++i) o_acc[i] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    float m_prev_pv = -INFINITY;    // max the pending O~(j-1) is relative to
    float m_acc = -INFINITY;        // max o_acc is relative to
    for (int j = 0; j < J; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      const int valid = min(kBK, p.skv - j * kBK);
      // pass 1: row max over this block
      uint32_t r[32];
      float blk_max = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < kBK / 32; ++c) {
        tmem_ld_32x32b_x32(tmem + lane_base + kColS + sb * kBK + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float v = (c * 32 + i < valid) ? __uint_as_float(r[i]) : -INFINITY;
          blk_max = fmaxf(blk_max, v);
        }
      }
      const float m_new = fmaxf(m_run, blk_max * p.scale_log2);
      const float corr = exp2f(m_run - m_new);   // 0 on the first block
      float sum = 0.f;
      // pass 2: P = exp2(s*scale - m_new), written bf16 into the SW128 A tile
      uint8_t* pbase = sP + sb * kPBytes;
#pragma unroll 1
      for (int c = 0; c < kBK / 32; ++c) {
        tmem_ld_32x32b_x32(tmem + lane_base + kColS + sb * kBK + c * 32, r);
        tmem_ld_wait();
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const int key = c * 32 + i;
          const float p0 = key < valid ? exp2f(fmaf(__uint_as_float(r[i]), p.scale_log2, -m_new)) : 0.f;
          const float p1 = key + 1 < valid ? exp2f(fmaf(__uint_as_float(r[i + 1]), p.scale_log2, -m_new)) : 0.f;
          sum += p0 + p1;
          packed[i / 2] = pack_bf16(p0, p1);
        }
        // keys c*32 .. c*32+31 live in atom (c>>1), 16-byte chunks 4*(c&1) .. +3
        uint8_t* atom = pbase + (c >> 1) * (kBQ * 128) + row * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = ((c & 1) * 4 + q) ^ (row & 7);
          *reinterpret_cast<uint4*>(atom + chunk * 16) =
              make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
        }
      }
      l_run = l_run * corr + sum;
      m_run = m_new;
      fence_proxy_async_smem();     // generic-proxy smem writes -> visible to the tensor core
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[sb]);
      // fold the previous block's O~ (relative to m_prev_pv) into o_acc
      if (j >= 1) {
        const int ob = (j - 1) & 1;
        mbar_wait(&o_full[ob], ((j - 1) >> 1) & 1);
        tc_fence_after();
        const float a_old = exp2f(m_acc - m_prev_pv);
        uint32_t ro[32];
#pragma unroll
        for (int c = 0; c < kD / 32; ++c) {
          tmem_ld_32x32b_x32(tmem + lane_base + kColO + ob * kD + c * 32, ro);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o_acc[c * 32 + i] = fmaf(o_acc[c * 32 + i], a_old, __uint_as_float(ro[i]));
        }
        m_acc = m_prev_pv;
      }
      m_prev_pv = m_new;
    }
    // last block
    {
      const int ob = (J - 1) & 1;
      mbar_wait(&o_full[ob], ((J - 1) >> 1) & 1);
      tc_fence_after();
      const float a_old = exp2f(m_acc - m_prev_pv);
      uint32_t ro[32];
#pragma unroll
      for (int c = 0; c < kD / 32; ++c) {
        tmem_ld_32x32b_x32(tmem + lane_base + kColO + ob * kD + c * 32, ro);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o_acc[c * 32 + i] = fmaf(o_acc[c * 32 + i], a_old, __uint_as_float(ro[i]));
      }
    }
    const int qrow = q0 + row;
    if (qrow < p.sq) {
      const float inv = 1.0f / l_run;
      __nv_bfloat16* dst = p.o + ((long long)b * p.sq + qrow) * p.ldo + h * kD;
#pragma unroll
      for (int q = 0; q < kD / 8; ++q) {
        uint4 u = make_uint4(pack_bf16(o_acc[8 * q] * inv, o_acc[8 * q + 1] * inv),
                             pack_bf16(o_acc[8 * q + 2] * inv, o_acc[8 * q + 3] * inv),
                             pack_bf16(o_acc[8 * q + 4] * inv, o_acc[8 * q + 5] * inv),
                             pack_bf16(o_acc[8 * q + 6] * inv, o_acc[8 * q + 7] * inv));
        reinterpret_cast<uint4*>(dst)[q] = u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<kTmemCols>(tmem);
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
  p.q_col0 = (int)d->q_col0; p.k_col0 = (int)d->k_col0; p.v_col0 = (int)d->v_col0;
  p.o = static_cast<__nv_bfloat16*>(d->o); p.ldo = d->ldo;
  p.scale_log2 = d->scale * 1.4426950408889634f;
  p.n_kv = (d->skv + kBK - 1) / kBK;
  constexpr size_t smem = 1024 + kTileBytes * (1 + 2 * kStages) + 2 * kPBytes + 256;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return HP_ERR_CUDA;
    attr = true;
  }
  dim3 grid((d->sq + kBQ - 1) / kBQ, d->heads, d->batch);
  attn_kernel<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(tq, tk, tv, p);
  return cudaGetLastError() == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}
