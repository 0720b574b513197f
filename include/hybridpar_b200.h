/*
 * hybridpar_b200.h — C ABI of the B200-native hybrid data/pipeline-parallel
 * denoising loop (sampler, discrepancy monitor, switch controller, pair
 * exchange, pipeline staging).
 *
 * Every entry point takes plain pointers, sizes and a cudaStream_t (passed as
 * void*), never allocates, is stream-ordered and CUDA-graph capturable, and
 * returns an int status (HP_OK = 0; negative values map onto the reference
 * error taxonomy, /root/reference/pkg/src/hybridpar/errors.py:8-50).
 *
 * Reference interfaces replaced (hybridpar 0.1.0, pkg/src/hybridpar/):
 *   hp_sampler_step      schedules.py:128-133  cfg_combine
 *                        schedules.py:152-168  ddim_step
 *                        schedules.py:171-182  fm_euler_step
 *                        schedules.py:121-125  _check_pair (non-finite count)
 *                        monitor.py:103-118    rel_mae (numerator/denominator
 *                                              partials + fixed-order finalize)
 *                        engine.py:187-192     _exact_update (all of the above
 *                                              in one launch)
 *   hp_ctrl_*            monitor.py:65-100     DiscrepancySeries (device copy)
 *                        monitor.py:121-132    slope
 *                        monitor.py:146-189    update_controller
 *   hp_blend_accumulate  engine.py:254-261     _pipelined_estimate blend
 *   hp_ipc_* / hp_signal / hp_flag_*           engine.py:217-231 _measured_step
 *                        and engine.py:307-337 _pipelined_step: the two
 *                        latent messages per measured step and the N-1
 *                        activation messages per pipelined step become NVLink
 *                        peer loads/stores guarded by system-scope flags.
 */
#ifndef HYBRIDPAR_B200_H
#define HYBRIDPAR_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-50) ------------------------------------- */
#define HP_OK                    0
#define HP_ERR_PARAMETER        -1   /* ParameterError        errors.py:8   */
#define HP_ERR_SHAPE            -2   /* ShapeError            errors.py:12  */
#define HP_ERR_NUMERIC          -3   /* NumericError          errors.py:16  */
#define HP_ERR_STEP_UNDERFLOW   -4   /* StepUnderflowError    errors.py:20  */
#define HP_ERR_HISTORY          -5   /* HistoryError          errors.py:24  */
#define HP_ERR_SEQUENCING       -6   /* SequencingError       errors.py:28  */
#define HP_ERR_DEGENERATE       -7   /* DegenerateInputError  errors.py:32  */
#define HP_ERR_PLAN             -8   /* PlanError             errors.py:36  */
#define HP_ERR_CUDA           -100   /* CUDA runtime / launch failure       */
#define HP_ERR_UNSUPPORTED    -101   /* dtype / alignment combination       */
#define HP_ERR_TIMEOUT        -102   /* peer flag never arrived             */

/* ---- element types ------------------------------------------------------ */
#define HP_F64   0
#define HP_F32   1
#define HP_BF16  2

/* ---- update rules -------------------------------------------------------- */
#define HP_UPDATE_DDIM   0   /* schedules.py:152-168 (eta = 0)                */
#define HP_UPDATE_EULER  1   /* schedules.py:171-182 (x - v*dt)               */
#define HP_UPDATE_NONE   2   /* out = e (cfg_combine alone, schedules.py:128) */

/* ---- controller ops performed in the tail of hp_sampler_step ------------- */
#define HP_CTRL_NONE            0  /* compute M_t only (into m_out)           */
#define HP_CTRL_RECORD          1  /* series.record(t, M_t)  monitor.py:76-85 */
#define HP_CTRL_RECORD_UPDATE   2  /* record + update_controller (146-189)    */

#define HP_STAGE_WARM_UP           0
#define HP_STAGE_PARALLELISM       1
#define HP_STAGE_FULLY_CONNECTING  2

#define HP_MAX_T 1024   /* largest schedule length the device series holds */
#define HP_MAX_PEERS 8  /* destinations of one hp_stage_broadcast (one NVLink domain of 8 GPUs) */

/* Device-resident controller state: StageState (monitor.py:135-143) plus the
 * DiscrepancySeries values (monitor.py:65-100) indexed by timestep t, plus the
 * SwitchConfig (monitor.py:35-62). Lives in device memory; 8-byte aligned. */
typedef struct hp_ctrl {
    int32_t L, tau_cap, k, T;      /* SwitchConfig + schedule length        */
    double  g_slope;
    int32_t tau1, tau2;            /* -1 = None                             */
    int32_t stage;                 /* HP_STAGE_*                            */
    int32_t steps_done;
    int32_t last_t;                /* -1 = None                             */
    int32_t last_recorded_t;       /* -1 = None (series descending check)   */
    int32_t status;                /* first error seen (HP_ERR_*), sticky   */
    int32_t n_recorded;
    double  m[HP_MAX_T + 1];       /* series value at key t                 */
    uint8_t has[HP_MAX_T + 1];     /* 1 if recorded                         */
} hp_ctrl;

/* Small mirror the sampler tail writes into mapped pinned host memory so the
 * host can poll the switch decision without a stream synchronize. */
typedef struct hp_ctrl_mirror {
    int32_t seq;                   /* step counter written last (release)   */
    int32_t tau1, tau2, stage, status, t;
    double  m;
} hp_ctrl_mirror;

/* One fused sampler step (kernel K1, with K2 in its last-block tail):
 *   e      = eps_c + w * (eps_c - eps_u)          (eps_u == NULL: e = eps_c)
 *   DDIM:  x0  = (x - c_sigma * e) / c_sqrt_ab
 *          out = c_sqrt_ab_prev * x0 + c_sqrt_1m_ab_prev * e
 *   EULER: out = x - e * dt
 *   NONE:  out = e                                 (x may be NULL)
 *   num   += |eps_c - eps_u|,  den += |eps_u|,  nonfinite += !isfinite(x,eps)
 * Every scalar is the exact fp64 value the reference computes on the host
 * (sched.sigma(t), np.sqrt(sched.alpha_bar(t)), ...), and the per-element
 * arithmetic keeps the reference operation order with no FMA contraction, so
 * the f64 instantiation reproduces numpy bit for bit.
 *
 * Optional exchange fusion: when wait_flag != NULL one thread per CTA spins
 * (system-scope acquire) until *wait_flag >= wait_value before any CTA reads
 * eps_u, which may then be a peer-mapped NVLink pointer (hp_ipc_open).
 */
typedef struct hp_step_desc {
    const void* x;          int32_t x_dtype;     /* HP_F64 | HP_F32          */
    const void* eps_c;
    const void* eps_u;      int32_t eps_dtype;   /* HP_F64 | HP_F32 | HP_BF16 */
    void*       x_out;                           /* x_dtype                  */
    void*       x_out_bf16;                      /* optional bf16 copy       */
    int64_t     n;
    int32_t     update;                          /* HP_UPDATE_*              */
    int32_t     t;                               /* timestep of x            */
    double      w;
    double      c_sigma, c_sqrt_ab, c_sqrt_ab_prev, c_sqrt_1m_ab_prev, dt;
    /* discrepancy + controller (partials may be NULL: no discrepancy)      */
    double*     partials;                        /* >= 2*hp_step_blocks(n)   */
    uint32_t*   ticket;                          /* zero-initialised once    */
    uint32_t*   nonfinite;                       /* zero-initialised once    */
    double*     m_out;                           /* optional M_t (device)    */
    int32_t*    status;                          /* optional step status     */
    hp_ctrl*    ctrl;                            /* optional                 */
    int32_t     ctrl_op;                         /* HP_CTRL_*                */
    hp_ctrl_mirror* mirror;                      /* optional, mapped pinned  */
    /* exchange fusion                                                       */
    const volatile uint32_t* wait_flag;          /* optional                 */
    uint32_t    wait_value;
} hp_step_desc;

/* number of CTAs (and partial pairs) hp_sampler_step uses for n elements */
int64_t hp_step_blocks(int64_t n);
int hp_sampler_step(const hp_step_desc* d, void* stream);

/* Reference-shaped primitives over device buffers (one launch each).      */
/* rel_mae (monitor.py:103-118): writes M to *m_out, status to *status.     */
int hp_rel_mae(const void* eps_c, const void* eps_u, int32_t dtype, int64_t n,
               double* partials, uint32_t* ticket, uint32_t* nonfinite,
               double* m_out, int32_t* status, void* stream);

/* Pipelined-window blend (engine.py:254-261): acc = (first ? 0 : acc) + f*eps,
 * computed as the reference does (zeros + f0*e0 + f1*e1 ...). */
int hp_blend_accumulate(void* acc, int32_t acc_dtype, const void* eps,
                        int32_t eps_dtype, double f, int32_t first, int64_t n,
                        void* stream);

/* Controller (monitor.py:135-205) on device. */
int hp_ctrl_init(hp_ctrl* ctrl, int32_t L, double g_slope, int32_t tau_cap,
                 int32_t k, int32_t T, void* stream);
/* record (optional) then update_controller at timestep t, one thread. */
int hp_ctrl_step(hp_ctrl* ctrl, int32_t t, const double* m, int32_t op,
                 hp_ctrl_mirror* mirror, void* stream);

/* ---- pair exchange / pipeline staging over NVLink peer memory ----------- */
#define HP_IPC_HANDLE_BYTES 64
/* cudaIpcGetMemHandle of a device allocation base pointer. */
int hp_ipc_get_handle(void* dev_ptr, uint8_t out_handle[HP_IPC_HANDLE_BYTES]);
/* cudaIpcOpenMemHandle (lazy peer access); returns the mapped pointer. */
int hp_ipc_open(const uint8_t handle[HP_IPC_HANDLE_BYTES], void** out_ptr);
int hp_ipc_close(void* mapped_ptr);
/* cudaDeviceCanAccessPeer + cudaDeviceEnablePeerAccess. */
int hp_enable_peer(int32_t peer_device);

/* Stream-ordered system-scope release store of `value` to *flag (flag may be
 * a peer-mapped pointer): the message "my buffer for step `value` is ready". */
int hp_signal(uint32_t* flag, uint32_t value, void* stream);
/* Stream-ordered wait until *flag >= value (spin with acquire; gives up with
 * HP_ERR_TIMEOUT written to *status after timeout_ns). */
int hp_flag_wait(const volatile uint32_t* flag, uint32_t value,
                 int32_t* status, uint64_t timeout_ns, void* stream);

/* HOST-side wait: poll *flag (device memory, local or peer-mapped) with small
 * D2H reads on a private non-blocking stream until *flag >= value; the value
 * read is stored in *observed (may be NULL). No kernel waits, so ranks that
 * share one GPU (tests) cannot stall each other's contexts; also used by
 * passive ranks to learn the window's first step. HP_ERR_TIMEOUT after
 * timeout_ns (0 = never). */
int hp_flag_poll(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, uint32_t* observed);

/* K3: copy nbytes from src (local) to dst (peer-mapped or local) with 16-byte
 * vector stores, then release-signal *flag = value (flag may be NULL).
 * engine.py:322-337 activation hand-off. */
int hp_stage_send(void* dst, const void* src, int64_t nbytes, uint32_t* flag,
                  uint32_t value, void* stream);

/* K3 fan-out: copy nbytes from src (local) to each of n_dst <= HP_MAX_PEERS
 * destinations (peer-mapped pointers; `dsts` and `flags` are HOST arrays read
 * at call time), then release *flags[i] = value for every non-NULL flag
 * (flags itself may be NULL; with nbytes == 0 only the flags are released and
 * dsts/src may be NULL). One launch per step for the layer-wise window,
 * where every segment rank hands its contribution to all ranks
 * (engine.py:330-337; the reference sends N-1 activations to device 0). */
int hp_stage_broadcast(void* const* dsts, uint32_t* const* flags, int32_t n_dst, const void* src,
                       int64_t nbytes, uint32_t value, void* stream);

/* Zero-filled device allocation with an exact base pointer (IPC-exportable
 * exchange buffers and flag words); hp_free releases it. Not for the hot loop. */
int hp_alloc(int64_t nbytes, void** out_ptr);
int hp_free(void* ptr);

/* library version / build info */
const char* hp_version(void);
int hp_device_sm_count(int32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* HYBRIDPAR_B200_H */
