// hp_sampler.cu — K1 (fused exchange + CFG + DDIM/Euler + discrepancy
// partials) with K2 (fixed-order discrepancy finalize + device switch
// controller) in the last-CTA tail.
//
// Reference semantics (hybridpar 0.1.0, /root/reference/pkg/src/hybridpar):
//   cfg_combine   schedules.py:128-133   e = eps_c + w * (eps_c - eps_u)
//   ddim_step     schedules.py:152-168   x0 = (x - sigma_t e)/sqrt(ab_t);
//                                        x' = sqrt(ab_{t-1}) x0 + sqrt(1-ab_{t-1}) e
//   fm_euler_step schedules.py:171-182   x' = x - v dt
//   _check_pair   schedules.py:121-125   non-finite -> NumericError
//   rel_mae       monitor.py:103-118     sum|eps_c-eps_u| / sum|eps_u|
//   record        monitor.py:76-85       descending, finite
//   slope         monitor.py:121-132     (M_t - M_{t+L}) / L
//   update_controller monitor.py:146-189
//
// HBM-bound: 14 B/elem for f32 x + bf16 eps (+bf16 copy of x'), no reuse, so
// the kernel is a grid-stride stream with 16-byte vector accesses where the
// operand alignment allows it. The grid size depends on n only, so the
// discrepancy partial sums (and M_t) are deterministic run to run.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>
#include "hybridpar_b200.h"
#include "hp_common.cuh"

namespace {

constexpr int kThreads = 128;
constexpr int kVec = 4;                     // elements per thread per sweep
constexpr int64_t kMaxBlocks = 148 * 8;     // B200 SM count x 8 (fixed => deterministic)

// ------------------------------------------------------------------------
// exact (non-contracted) arithmetic in the compute type
template <typename C> struct Ar;
template <> struct Ar<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <> struct Ar<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};

template <typename T> struct Ld;
template <> struct Ld<double> {
  template <typename C> static __device__ __forceinline__ void v4(const double* p, C* o) {
    double4 v = *reinterpret_cast<const double4*>(p);  // 32B aligned checked on host
    o[0] = (C)v.x; o[1] = (C)v.y; o[2] = (C)v.z; o[3] = (C)v.w;
  }
  template <typename C> static __device__ __forceinline__ C s(const double* p) { return (C)*p; }
};
template <> struct Ld<float> {
  template <typename C> static __device__ __forceinline__ void v4(const float* p, C* o) {
    float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = (C)v.x; o[1] = (C)v.y; o[2] = (C)v.z; o[3] = (C)v.w;
  }
  template <typename C> static __device__ __forceinline__ C s(const float* p) { return (C)*p; }
};
template <> struct Ld<__nv_bfloat16> {
  template <typename C> static __device__ __forceinline__ void v4(const __nv_bfloat16* p, C* o) {
    uint2 raw = *reinterpret_cast<const uint2*>(p);
    __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&raw.x);
    __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&raw.y);
    float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    o[0] = (C)fa.x; o[1] = (C)fa.y; o[2] = (C)fb.x; o[3] = (C)fb.y;
  }
  template <typename C> static __device__ __forceinline__ C s(const __nv_bfloat16* p) {
    return (C)__bfloat162float(*p);
  }
};

template <typename T> struct St;
template <> struct St<double> {
  template <typename C> static __device__ __forceinline__ void v4(double* p, const C* v) {
    *reinterpret_cast<double4*>(p) = make_double4((double)v[0], (double)v[1], (double)v[2], (double)v[3]);
  }
  template <typename C> static __device__ __forceinline__ void s(double* p, C v) { *p = (double)v; }
};
template <> struct St<float> {
  template <typename C> static __device__ __forceinline__ void v4(float* p, const C* v) {
    *reinterpret_cast<float4*>(p) = make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
  }
  template <typename C> static __device__ __forceinline__ void s(float* p, C v) { *p = (float)v; }
};

__device__ __forceinline__ void st_bf16x4(__nv_bfloat16* p, const float* v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
  __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
  uint2 raw;
  raw.x = *reinterpret_cast<uint32_t*>(&a);
  raw.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = raw;
}

template <typename C> __device__ __forceinline__ bool finite_(C v) { return isfinite(v); }

struct StepScalars {
  double w, c_sigma, c_sqrt_ab, c_sqrt_ab_prev, c_sqrt_1m_ab_prev, dt;
};

// ------------------------------------------------------------------------
// device controller (monitor.py:76-85, 121-132, 146-189), one thread
__device__ void ctrl_record(hp_ctrl* c, int t, double v) {
  if (c->status != HP_OK) return;
  if (t < 0 || t > HP_MAX_T) { c->status = HP_ERR_PARAMETER; return; }
  if (!isfinite(v)) { c->status = HP_ERR_NUMERIC; return; }
  if (c->last_recorded_t >= 0 && t >= c->last_recorded_t) { c->status = HP_ERR_SEQUENCING; return; }
  c->m[t] = v;
  c->has[t] = 1;
  c->last_recorded_t = t;
  c->n_recorded += 1;
}

__device__ void ctrl_update(hp_ctrl* c, int t) {
  if (c->status != HP_OK) return;
  if (t < 0) { c->status = HP_ERR_PARAMETER; return; }
  if (c->last_t >= 0 && t != c->last_t - 1) { c->status = HP_ERR_SEQUENCING; return; }
  const int s = c->steps_done + 1;
  int label;
  if (c->tau1 < 0) {
    bool fired = false;
    const int tl = t + c->L;
    if (tl <= HP_MAX_T && c->has[t] && c->has[tl]) {
      const double g = __ddiv_rn(__dsub_rn(c->m[t], c->m[tl]), (double)c->L);
      fired = (0.0 <= g) && (g < c->g_slope);
    }
    if (fired) {
      c->tau1 = s < c->tau_cap ? s : c->tau_cap;
      c->tau2 = c->tau1 + c->k;
    } else if (s >= c->tau_cap) {
      c->tau1 = c->tau_cap;
      c->tau2 = c->tau1 + c->k;
    }
    label = HP_STAGE_WARM_UP;
  } else if (s <= c->tau1) {
    label = HP_STAGE_WARM_UP;
  } else if (s <= c->tau2) {
    label = HP_STAGE_PARALLELISM;
  } else {
    label = HP_STAGE_FULLY_CONNECTING;
  }
  if (label < c->stage) { c->status = HP_ERR_SEQUENCING; return; }
  c->stage = label;
  c->steps_done = s;
  c->last_t = t;
}

__device__ void mirror_publish(hp_ctrl_mirror* mr, const hp_ctrl* c, int t, double m, int status) {
  if (mr == nullptr) return;
  mr->tau1 = c ? c->tau1 : -1;
  mr->tau2 = c ? c->tau2 : -1;
  mr->stage = c ? c->stage : 0;
  mr->status = status;
  mr->t = t;
  mr->m = m;
  __threadfence_system();
  // seq = HP_MAX_T + 1 - t grows as t descends: the host waits for its step's value
  hp_st_release_sys_u32(reinterpret_cast<uint32_t*>(&mr->seq), (uint32_t)(HP_MAX_T + 1 - t));
}

// deterministic fixed-order finalize of the per-CTA partials (last CTA)
__device__ void finalize_tail(double* partials, int nblocks, uint32_t* nonfinite,
                              double* m_out, hp_ctrl* ctrl, int ctrl_op, int t,
                              hp_ctrl_mirror* mirror, int32_t* status_out, bool has_u) {
  __shared__ double s_num[kThreads];
  __shared__ double s_den[kThreads];
  double num = 0.0, den = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += kThreads) {
    num += partials[2 * i];
    den += partials[2 * i + 1];
  }
  s_num[threadIdx.x] = num;
  s_den[threadIdx.x] = den;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_num[threadIdx.x] += s_num[threadIdx.x + w];
      s_den[threadIdx.x] += s_den[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int status = HP_OK;
    const uint32_t bad = *nonfinite;
    *nonfinite = 0u;
    double m = 0.0;
    if (bad) status = HP_ERR_NUMERIC;
    else if (!has_u) m = NAN;
    else if (s_den[0] == 0.0) status = HP_ERR_DEGENERATE;
    else m = s_num[0] / s_den[0];
    if (m_out) *m_out = m;
    if (status_out) *status_out = status;
    if (ctrl) {
      if (status != HP_OK) {
        if (ctrl->status == HP_OK) ctrl->status = status;
      } else if (ctrl_op >= HP_CTRL_RECORD && has_u) {
        ctrl_record(ctrl, t, m);
        if (ctrl_op == HP_CTRL_RECORD_UPDATE) ctrl_update(ctrl, t);
      }
      status = ctrl->status;
    }
    mirror_publish(mirror, ctrl, t, m, status);
  }
}

template <typename XT, typename ET, typename C, int UPDATE, bool HAS_U, bool BF16_OUT>
__global__ void __launch_bounds__(kThreads)
sampler_step_kernel(const XT* x, const ET* eps_c, const ET* eps_u, XT* x_out,
                    __nv_bfloat16* x_out_bf16, int64_t n, StepScalars sc,
                    double* partials, uint32_t* ticket, uint32_t* nonfinite,
                    double* m_out, hp_ctrl* ctrl, int ctrl_op, int t,
                    hp_ctrl_mirror* mirror, int32_t* status_out,
                    const volatile uint32_t* wait_flag, uint32_t wait_value, bool vec_ok) {
  using A = Ar<C>;
  if (wait_flag != nullptr) {
    // exchange fusion: the partner's eps for this step must have landed. A partner
    // that never arrives (crashed rank) turns into HP_ERR_TIMEOUT after 20 s instead
    // of a hung GPU; the step then completes on stale data and the status is sticky.
    __shared__ int s_timeout;
    if (threadIdx.x == 0) {
      s_timeout = 0;
      const uint64_t t0 = hp_globaltimer();
      // fail fast once a previous wait of this run timed out (sticky status): the run is
      // already lost, do not spend another 20 s per step
      const bool dead = ctrl != nullptr && *reinterpret_cast<volatile int32_t*>(&ctrl->status) == HP_ERR_TIMEOUT;
      while (!dead && hp_ld_acquire_sys_u32(wait_flag) < wait_value) {
        __nanosleep(64);
        if (hp_globaltimer() - t0 > 20000000000ull) { s_timeout = 1; break; }
      }
    }
    __syncthreads();
    if (s_timeout && threadIdx.x == 0) {
      if (status_out) *status_out = HP_ERR_TIMEOUT;
      if (ctrl) ctrl->status = HP_ERR_TIMEOUT;
    }
  }
  const C w = (C)sc.w, c_sigma = (C)sc.c_sigma, c_sab = (C)sc.c_sqrt_ab,
          c_sabp = (C)sc.c_sqrt_ab_prev, c_s1m = (C)sc.c_sqrt_1m_ab_prev, dt = (C)sc.dt;
  double num = 0.0, den = 0.0;
  bool bad = false;

  auto body = [&](const C* xv, const C* ec, const C* eu, C* out, int cnt) {
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      if (j >= cnt) break;
      C e;
      if (HAS_U) {
        const C diff = A::sub(ec[j], eu[j]);
        e = A::add(ec[j], A::mul(w, diff));
        num += (double)fabs(diff);
        den += (double)fabs(eu[j]);
        bad |= !(finite_(eu[j]));
      } else {
        e = ec[j];
      }
      bad |= !(finite_(ec[j]) && finite_(e));
      if (UPDATE != HP_UPDATE_NONE) bad |= !finite_(xv[j]);
      if (UPDATE == HP_UPDATE_DDIM) {
        const C x0 = A::div(A::sub(xv[j], A::mul(c_sigma, e)), c_sab);
        out[j] = A::add(A::mul(c_sabp, x0), A::mul(c_s1m, e));
      } else if (UPDATE == HP_UPDATE_EULER) {
        out[j] = A::sub(xv[j], A::mul(e, dt));
      } else {
        out[j] = e;
      }
    }
  };

  const int64_t stride = (int64_t)gridDim.x * kThreads * kVec;
  for (int64_t base = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * kVec; base < n; base += stride) {
    C xv[kVec], ec[kVec], eu[kVec], out[kVec];
    const int cnt = (n - base) >= kVec ? kVec : (int)(n - base);
    if (UPDATE == HP_UPDATE_NONE) {
#pragma unroll
      for (int j = 0; j < kVec; ++j) xv[j] = (C)0;
    }
    if (vec_ok && cnt == kVec) {
      if (UPDATE != HP_UPDATE_NONE) Ld<XT>::v4(x + base, xv);
      Ld<ET>::v4(eps_c + base, ec);
      if (HAS_U) Ld<ET>::v4(eps_u + base, eu);
    } else {
      for (int j = 0; j < cnt; ++j) {
        if (UPDATE != HP_UPDATE_NONE) xv[j] = Ld<XT>::template s<C>(x + base + j);
        ec[j] = Ld<ET>::template s<C>(eps_c + base + j);
        if (HAS_U) eu[j] = Ld<ET>::template s<C>(eps_u + base + j);
      }
    }
    body(xv, ec, eu, out, cnt);
    if (vec_ok && cnt == kVec) {
      St<XT>::v4(x_out + base, out);
      if (BF16_OUT) {
        float o[4] = {(float)out[0], (float)out[1], (float)out[2], (float)out[3]};
        st_bf16x4(x_out_bf16 + base, o);
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        St<XT>::s(x_out + base + j, out[j]);
        if (BF16_OUT) x_out_bf16[base + j] = __float2bfloat16_rn((float)out[j]);
      }
    }
  }

  // ---- discrepancy partials (fixed order: warp shuffle, then smem) ----
  const int any_bad = __syncthreads_or(bad ? 1 : 0);
  if (partials == nullptr) return;
  num = hp_warp_sum(num);
  den = hp_warp_sum(den);
  __shared__ double s_num[kThreads / 32], s_den[kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_num[warp] = num; s_den[warp] = den; }
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    double bn = 0.0, bd = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) { bn += s_num[i]; bd += s_den[i]; }
    partials[2 * blockIdx.x] = bn;
    partials[2 * blockIdx.x + 1] = bd;
    if (any_bad) atomicAdd(nonfinite, 1u);
    __threadfence();
    const uint32_t prev = atomicAdd(ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) *ticket = 0u;  // self-reset for the next launch / graph replay
  finalize_tail(partials, gridDim.x, nonfinite, m_out, ctrl, ctrl_op, t, mirror, status_out, HAS_U);
}

template <typename XT, typename ET, typename C>
cudaError_t launch_step(const hp_step_desc* d, cudaStream_t st, int blocks, bool vec_ok) {
  StepScalars sc{d->w, d->c_sigma, d->c_sqrt_ab, d->c_sqrt_ab_prev, d->c_sqrt_1m_ab_prev, d->dt};
  const XT* x = static_cast<const XT*>(d->x);
  const ET* ec = static_cast<const ET*>(d->eps_c);
  const ET* eu = static_cast<const ET*>(d->eps_u);
  XT* xo = static_cast<XT*>(d->x_out);
  __nv_bfloat16* xb = static_cast<__nv_bfloat16*>(d->x_out_bf16);
  const bool has_u = eu != nullptr;
  const bool bo = xb != nullptr;
#define HP_LAUNCH(UPD, HU, BO)                                                           \
  sampler_step_kernel<XT, ET, C, UPD, HU, BO><<<blocks, kThreads, 0, st>>>(              \
      x, ec, eu, xo, xb, d->n, sc, d->partials, d->ticket, d->nonfinite, d->m_out,       \
      d->ctrl, d->ctrl_op, d->t, d->mirror, d->status, d->wait_flag, d->wait_value, vec_ok)
  if (d->update == HP_UPDATE_DDIM) {
    if (has_u) { if (bo) HP_LAUNCH(HP_UPDATE_DDIM, true, true); else HP_LAUNCH(HP_UPDATE_DDIM, true, false); }
    else       { if (bo) HP_LAUNCH(HP_UPDATE_DDIM, false, true); else HP_LAUNCH(HP_UPDATE_DDIM, false, false); }
  } else if (d->update == HP_UPDATE_EULER) {
    if (has_u) { if (bo) HP_LAUNCH(HP_UPDATE_EULER, true, true); else HP_LAUNCH(HP_UPDATE_EULER, true, false); }
    else       { if (bo) HP_LAUNCH(HP_UPDATE_EULER, false, true); else HP_LAUNCH(HP_UPDATE_EULER, false, false); }
  } else {
    if (has_u) HP_LAUNCH(HP_UPDATE_NONE, true, false); else HP_LAUNCH(HP_UPDATE_NONE, false, false);
  }
#undef HP_LAUNCH
  return cudaGetLastError();
}

// rel_mae only: reuse the step kernel's reduction path without the update
template <typename ET>
__global__ void __launch_bounds__(kThreads)
rel_mae_kernel(const ET* eps_c, const ET* eps_u, int64_t n, double* partials,
               uint32_t* ticket, uint32_t* nonfinite, double* m_out, int32_t* status_out) {
  using C = typename std::conditional<std::is_same<ET, double>::value, double, float>::type;
  double num = 0.0, den = 0.0;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    const C ec = Ld<ET>::template s<C>(eps_c + i);
    const C eu = Ld<ET>::template s<C>(eps_u + i);
    const C diff = Ar<C>::sub(ec, eu);
    num += (double)fabs(diff);
    den += (double)fabs(eu);
    bad |= !(isfinite(ec) && isfinite(eu));
  }
  const int any_bad = __syncthreads_or(bad ? 1 : 0);
  num = hp_warp_sum(num);
  den = hp_warp_sum(den);
  __shared__ double s_num[kThreads / 32], s_den[kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_num[warp] = num; s_den[warp] = den; }
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    double bn = 0.0, bd = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) { bn += s_num[i]; bd += s_den[i]; }
    partials[2 * blockIdx.x] = bn;
    partials[2 * blockIdx.x + 1] = bd;
    if (any_bad) atomicAdd(nonfinite, 1u);
    __threadfence();
    s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) *ticket = 0u;
  finalize_tail(partials, gridDim.x, nonfinite, m_out, nullptr, HP_CTRL_NONE, 0, nullptr, status_out, true);
}

template <typename AT, typename ET>
__global__ void blend_kernel(AT* acc, const ET* eps, double f, int first, int64_t n) {
  using C = typename std::conditional<std::is_same<AT, double>::value, double, float>::type;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const C e = Ld<ET>::template s<C>(eps + i);
    const C prod = Ar<C>::mul((C)f, e);
    const C base = first ? (C)0 : (C)acc[i];
    acc[i] = (AT)Ar<C>::add(base, prod);
  }
}

__global__ void ctrl_init_kernel(hp_ctrl* c, int L, double g, int tau_cap, int k, int T) {
  for (int i = threadIdx.x; i <= HP_MAX_T; i += blockDim.x) { c->m[i] = 0.0; c->has[i] = 0; }
  if (threadIdx.x == 0) {
    c->L = L; c->g_slope = g; c->tau_cap = tau_cap; c->k = k; c->T = T;
    c->tau1 = -1; c->tau2 = -1; c->stage = HP_STAGE_WARM_UP; c->steps_done = 0;
    c->last_t = -1; c->last_recorded_t = -1; c->status = HP_OK; c->n_recorded = 0;
  }
}

__global__ void ctrl_step_kernel(hp_ctrl* c, int t, const double* m, int op, hp_ctrl_mirror* mirror) {
  double mv = m ? *m : 0.0;
  if (op >= HP_CTRL_RECORD) ctrl_record(c, t, mv);
  ctrl_update(c, t);
  mirror_publish(mirror, c, t, mv, c->status);
}

template <typename ET>
int dispatch_eps(int x_dtype, const hp_step_desc* d, cudaStream_t st, int blocks, bool vec) {
  cudaError_t e;
  if (x_dtype == HP_F64) e = launch_step<double, ET, double>(d, st, blocks, vec);
  else if (std::is_same<ET, double>::value) return HP_ERR_UNSUPPORTED;  // f64 eps needs f64 x
  else e = launch_step<float, ET, float>(d, st, blocks, vec);
  return e == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

inline bool aligned(const void* p, size_t a) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % a) == 0; }
inline size_t esize(int dt) { return dt == HP_F64 ? 8 : dt == HP_F32 ? 4 : 2; }

}  // namespace

extern "C" {

int64_t hp_step_blocks(int64_t n) {
  int64_t b = (n + (int64_t)kThreads * kVec - 1) / ((int64_t)kThreads * kVec);
  if (b < 1) b = 1;
  if (b > kMaxBlocks) b = kMaxBlocks;
  return b;
}

int hp_sampler_step(const hp_step_desc* d, void* stream) {
  if (d == nullptr || d->eps_c == nullptr || d->x_out == nullptr) return HP_ERR_PARAMETER;
  if (d->x == nullptr && d->update != HP_UPDATE_NONE) return HP_ERR_PARAMETER;
  if (d->n < 0) return HP_ERR_SHAPE;
  if (d->update != HP_UPDATE_DDIM && d->update != HP_UPDATE_EULER && d->update != HP_UPDATE_NONE)
    return HP_ERR_PARAMETER;
  if (d->x_dtype != HP_F64 && d->x_dtype != HP_F32) return HP_ERR_UNSUPPORTED;
  if (d->partials != nullptr && (d->ticket == nullptr || d->nonfinite == nullptr)) return HP_ERR_PARAMETER;
  if (d->n == 0) return HP_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = (int)hp_step_blocks(d->n);
  const size_t xa = esize(d->x_dtype) * kVec, ea = esize(d->eps_dtype) * kVec;
  const bool vec = aligned(d->x, xa) && aligned(d->x_out, xa) && aligned(d->eps_c, ea) &&
                   aligned(d->eps_u, ea) && aligned(d->x_out_bf16, 8);
  switch (d->eps_dtype) {
    case HP_F64: return dispatch_eps<double>(d->x_dtype, d, st, blocks, vec);
    case HP_F32: return dispatch_eps<float>(d->x_dtype, d, st, blocks, vec);
    case HP_BF16: return dispatch_eps<__nv_bfloat16>(d->x_dtype, d, st, blocks, vec);
    default: return HP_ERR_UNSUPPORTED;
  }
}

int hp_rel_mae(const void* eps_c, const void* eps_u, int32_t dtype, int64_t n, double* partials,
               uint32_t* ticket, uint32_t* nonfinite, double* m_out, int32_t* status, void* stream) {
  if (!eps_c || !eps_u || !partials || !ticket || !nonfinite || !m_out) return HP_ERR_PARAMETER;
  if (n <= 0) return HP_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = (int)hp_step_blocks(n);
  switch (dtype) {
    case HP_F64: rel_mae_kernel<double><<<blocks, kThreads, 0, st>>>((const double*)eps_c, (const double*)eps_u, n, partials, ticket, nonfinite, m_out, status); break;
    case HP_F32: rel_mae_kernel<float><<<blocks, kThreads, 0, st>>>((const float*)eps_c, (const float*)eps_u, n, partials, ticket, nonfinite, m_out, status); break;
    case HP_BF16: rel_mae_kernel<__nv_bfloat16><<<blocks, kThreads, 0, st>>>((const __nv_bfloat16*)eps_c, (const __nv_bfloat16*)eps_u, n, partials, ticket, nonfinite, m_out, status); break;
    default: return HP_ERR_UNSUPPORTED;
  }
  return cudaGetLastError() == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

int hp_blend_accumulate(void* acc, int32_t acc_dtype, const void* eps, int32_t eps_dtype, double f,
                        int32_t first, int64_t n, void* stream) {
  if (!acc || !eps) return HP_ERR_PARAMETER;
  if (n == 0) return HP_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (acc_dtype == HP_F64 && eps_dtype == HP_F64) blend_kernel<double, double><<<blocks, 256, 0, st>>>((double*)acc, (const double*)eps, f, first, n);
  else if (acc_dtype == HP_F32 && eps_dtype == HP_F32) blend_kernel<float, float><<<blocks, 256, 0, st>>>((float*)acc, (const float*)eps, f, first, n);
  else if (acc_dtype == HP_F32 && eps_dtype == HP_BF16) blend_kernel<float, __nv_bfloat16><<<blocks, 256, 0, st>>>((float*)acc, (const __nv_bfloat16*)eps, f, first, n);
  else return HP_ERR_UNSUPPORTED;
  return cudaGetLastError() == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

int hp_ctrl_init(hp_ctrl* ctrl, int32_t L, double g_slope, int32_t tau_cap, int32_t k, int32_t T, void* stream) {
  if (!ctrl) return HP_ERR_PARAMETER;
  if (L < 1 || !(g_slope > 0) || tau_cap < 0 || k < 0 || T < 1 || T > HP_MAX_T) return HP_ERR_PARAMETER;
  ctrl_init_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(ctrl, L, g_slope, tau_cap, k, T);
  return cudaGetLastError() == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

int hp_ctrl_step(hp_ctrl* ctrl, int32_t t, const double* m, int32_t op, hp_ctrl_mirror* mirror, void* stream) {
  if (!ctrl) return HP_ERR_PARAMETER;
  if (op >= HP_CTRL_RECORD && m == nullptr) return HP_ERR_PARAMETER;
  ctrl_step_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(ctrl, t, m, op, mirror);
  return cudaGetLastError() == cudaSuccess ? HP_OK : HP_ERR_CUDA;
}

}  // extern "C"
