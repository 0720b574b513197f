/*
 * hybridpar_b200_denoiser.h — C ABI of the denoiser kernels behind the seam.
 *
 * The reference has no neural network: its only denoiser is the analytic
 * Gaussian mixture eps_prediction (/root/reference/pkg/src/hybridpar/
 * mixture.py:152-158), reached from engine.py:171-184 (_branches /
 * _conditional_branch). These entry points are what a random-init
 * SDXL-shaped U-Net or SD3-shaped MMDiT needs to stand in at that seam on
 * B200: tcgen05/TMA GEMM and implicit-GEMM 3x3 convolution with fused
 * epilogues, fused multi-head attention, and the memory-bound norm /
 * resampling ops. All tensors are bf16 NHWC / row-major unless noted, all
 * calls are stream-ordered, never allocate, and are CUDA-graph capturable.
 */
#ifndef HYBRIDPAR_B200_DENOISER_H
#define HYBRIDPAR_B200_DENOISER_H

#include <stdint.h>
#include "hybridpar_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- GEMM / implicit-GEMM convolution (tcgen05 + TMA, TMEM accumulators) --- */
#define HP_A_PLAIN        0   /* A is [M, K] row-major (lda elements)            */
#define HP_A_CONV3X3      1   /* A is NHWC [n, h, w, c]; K = 9*c; pad 1, stride 1  */
#define HP_A_CONV3X3_S2   2   /* same, stride 2 (output h/2 x w/2)                 */
/* HP_A_UPCONV: nearest 2x upsample then 3x3 conv (pad 1), computed as four
 * sub-pixel 2x2 convs on the LOW-res NHWC input [n, h, w, c] (one per output
 * phase (py, px), all in one launch): b = [4 * N, 4 * c], phase-major, tap
 * (ty, tx) of a phase = the sum of the 3x3 taps that read the same input
 * pixel; K = 4 * c; M = n * h * w; d = the 2x output [n, 2h, 2w, N] with row
 * stride ldd. 16 instead of 36 taps of MMA work per output pixel.          */
#define HP_A_UPCONV       3

#define HP_ACT_NONE   0
#define HP_ACT_GELU   1       /* exact erf GELU                                     */
#define HP_ACT_SILU   2
#define HP_ACT_GEGLU  3       /* weight rows interleaved per 2*BN/2 tile: out = a*gelu(b) */

typedef struct hp_gemm_desc {
    const void* a;     int64_t lda;            /* bf16                           */
    int32_t a_mode;                            /* HP_A_*                         */
    int32_t img_n, img_h, img_w, img_c;        /* conv input geometry            */
    const void* b;     int64_t ldb;            /* bf16 weights [N, K] (K-major)  */
    void* d;           int64_t ldd;            /* bf16 output [M, N_out]         */
    int64_t M, N, K;
    const float* bias;                         /* [N] or NULL                    */
    const float* bias2; int64_t bias2_div;     /* bias2[(row/div)*N + col]       */
    const void* residual; int64_t ldr;         /* bf16 [M, N_out] or NULL        */
    int32_t act;                               /* HP_ACT_*                       */
    int32_t block_n;                           /* 0 = auto                       */
    float alpha;                               /* acc scale before bias          */
    const float* colscale;                     /* [N] or NULL: d = residual + colscale[col] *
                                                  act(alpha*acc + bias)  (adaLN-Zero gate) */
    /* batched plain GEMM (a_mode HP_A_PLAIN only): `batch` independent row
     * blocks of M rows each; element strides between consecutive blocks of A,
     * D, residual and colscale (0 = shared). batch <= 1 = ordinary GEMM.    */
    int32_t batch;
    int64_t a_bstride, d_bstride, r_bstride, cs_bstride;
    int64_t bias2_ld;                          /* row stride of bias2 (0 = N)    */
    /* fused LayerNorm of the output rows (ln_y != NULL): also writes
     * ln_y = LayerNorm(d) with gamma/beta [N] fp32; the N tiles of each
     * 128-row block run as one thread-block cluster and combine their
     * row partial sums through distributed shared memory (N/block_n <= 8). */
    const float* ln_gamma; const float* ln_beta; float ln_eps;
    void* ln_y; int64_t ldy;
    /* LayerNorm folded into the next GEMM (no normalised tensor is written).
     * Producer side, stats_out != NULL: the epilogue also writes, for every
     * output row and N tile, (mean, M2) of the STORED bf16 row segment as two
     * floats at stats_out[2 * (row * (N / block_n) + tile)] (plain, batch 1,
     * not GEGLU, N % block_n == 0).
     * Consumer side, ln_stats != NULL: A holds the raw rows, B = W * gamma
     * (columns scaled), ln_colsum[n] = sum_k B[n, k] (fp32 of the bf16 B),
     * bias = b + W beta. The epilogue combines the ln_parts partials of
     * ln_part_n columns each (Chan's formula, fixed order; ln_parts *
     * ln_part_n == K) into mean / rstd per row and forms
     *   LN(A) W^T + b = rstd * (acc - mean * ln_colsum[n]) + bias[n]
     * before the activation. */
    float* stats_out;
    const float* ln_stats; int32_t ln_parts; int32_t ln_part_n;
    const float* ln_colsum; float ln_fold_eps;
    /* GroupNorm partials of the output (gn_part != NULL): for every 128-row block
     * and 10-column segment, (sum, sum of squares) of the STORED bf16 values as two
     * floats at gn_part[2 * (idx * (N / 10) + segment)], idx = image * gn_parts +
     * block within the image, images of gn_rows rows (HP_A_UPCONV: gn_rows = input
     * pixels per image, blocks phase-major). Requires N % 160 == 0, M % 128 == 0,
     * no activation; consumed by hp_group_norm_parts. */
    float* gn_part; int64_t gn_rows; int32_t gn_parts;
} hp_gemm_desc;

int hp_gemm(const hp_gemm_desc* d, void* stream);
/* block_n the auto heuristic would choose (0 if unsupported shape) */
int32_t hp_gemm_pick_block_n(int64_t M, int64_t N, int64_t K, int32_t act);
/* block_n for a GEMM that writes LayerNorm row statistics (stats_out): chosen so the
 * statistics segment width (160 when N % 160 == 0) and the split-K decision depend on
 * N and K only, never on M (batch invariance of the folded LayerNorm). */
int32_t hp_gemm_stats_block_n(int64_t M, int64_t N, int64_t K);

/* ---- fused multi-head attention (tcgen05 S = QK^T and O = PV) -------------- */
/* q: [B, Sq, ldq] with head h at column h*64 (+q_col0); k/v likewise with
 * Skv rows; o: [B, Sq, ldo]. head_dim = 64. scale applied to QK^T.          */
typedef struct hp_attn_desc {
    const void* q; int64_t ldq; int64_t q_col0;
    const void* k; int64_t ldk; int64_t k_col0;
    const void* v; int64_t ldv; int64_t v_col0;
    void* o;       int64_t ldo;
    int32_t batch, heads, sq, skv;
    float scale;
    int32_t causal;    /* 1: key j masked for query i when j > i (text encoders; skv <= 128) */
} hp_attn_desc;
int hp_attention(const hp_attn_desc* d, void* stream);

/* ---- norms, activations, resampling (HBM-bound) --------------------------- */
/* GroupNorm over NHWC bf16 (x1 channels c1, optional x2 concat channels c2),
 * affine gamma/beta fp32, optional SiLU, writes y [n, hw, c1+c2] bf16.
 * stats: workspace of >= 2*n*groups floats.                                  */
int hp_group_norm(const void* x1, int32_t c1, const void* x2, int32_t c2, int32_t n, int64_t hw,
                  int32_t groups, float eps, const float* gamma, const float* beta, int32_t silu,
                  void* y, float* stats, void* stream);
/* GroupNorm(+SiLU) of x [n, hw, c] (bf16) whose statistics the producing GEMMs
 * left as hp_gemm_desc.gn_part partials: channels [0, c1) from part1 (c1 / 10
 * segments per partial row), channels [c1, c) from part2 (the second operand of
 * a channel concat; NULL when c1 == c). hw / 128 partial rows per image. Folds
 * the partials in fixed order (fp64), writes y [n, hw, c]. One launch, no
 * grid-wide barrier. Group width c / groups must be a multiple of 10. */
int hp_group_norm_parts(const void* x, int32_t c, int32_t n, int64_t hw, const float* part1, int32_t c1,
                        const float* part2, int32_t groups, float eps, const float* gamma,
                        const float* beta, int32_t silu, void* y, void* stream);
/* LayerNorm over rows of bf16 [rows, c]; optional gamma/beta (fp32);
 * optional adaLN modulation y = norm*(1+scale[b]) + shift[b] with
 * b = row / rows_per_batch, scale/shift fp32 rows of length c (stride ldm). */
int hp_layer_norm(const void* x, int64_t rows, int32_t c, float eps, const float* gamma,
                  const float* beta, const void* shift, const void* scale, int64_t ldm,
                  int64_t rows_per_batch, void* y, void* stream);
/* Joint (two-stream) modulated LayerNorm for MMDiT token buffers laid out
 * [batch][rows_per_batch][c]: row i of a batch uses (shift, scale) when
 * i < split and (shift2, scale2) otherwise (each fp32, batch stride ldm). */
int hp_layer_norm_joint(const void* x, int64_t rows, int32_t c, float eps, const float* shift,
                        const float* scale, const float* shift2, const float* scale2, int64_t ldm,
                        int64_t rows_per_batch, int64_t split, void* y, void* stream);
/* y = silu(x) elementwise, bf16 */
int hp_silu(const void* x, void* y, int64_t n, void* stream);
/* y = x * sigmoid(1.702 x) (quick GELU, CLIP ViT-L MLP) elementwise, bf16; kept out
 * of the GEMM epilogue, whose unrolled code every denoiser GEMM shares */
int hp_quick_gelu(const void* x, void* y, int64_t n, void* stream);
/* nearest 2x upsample NHWC bf16: [n, h, w, c] -> [n, 2h, 2w, c] */
int hp_upsample2x(const void* x, int32_t n, int32_t h, int32_t w, int32_t c, void* y, void* stream);
/* channel concat NHWC: y[..., 0:c1] = a, y[..., c1:c1+c2] = b */
int hp_concat_channels(const void* a, int32_t c1, const void* b, int32_t c2, int64_t pixels,
                       void* y, void* stream);
/* token + position embedding: y[r, :] = tok[ids[r], :] + pos[r % seq, :] (fp32
 * tables, bf16 out), the text encoders' input layer.                        */
int hp_embed_tokens(const int64_t* ids, int64_t rows, int32_t seq, const float* tok, const float* pos, int32_t dim,
                    void* y, void* stream);
/* row softmax, bf16 in / bf16 out: y[r, :] = softmax(scale * x[r, :]) over `cols`
 * values, fp32 math, fixed-order reductions (the VAE decoder's single-head
 * 512-dim attention runs as GEMM -> this -> GEMM; cols <= 32768).            */
int hp_softmax_rows(const void* x, int64_t ldx, int64_t rows, int32_t cols, float scale, void* y, int64_t ldy,
                    void* stream);
/* per-row channel window copy, bf16: y[r, j] = j < c_src ? x[r, j] : 0 for j < c_dst
 * (zero-pads conv_in's 4 latent channels to the 64 the implicit-GEMM conv needs,
 * and slices conv_out's 4 channels out of its 64-wide padded GEMM output).     */
int hp_copy_cols(const void* x, int64_t ldx, int32_t c_src, int64_t rows, void* y, int64_t ldy, int32_t c_dst,
                 void* stream);
/* direct 3x3 conv for tiny channel counts (conv_in / conv_out): NHWC bf16 in,
 * weights fp32 [cout, 3, 3, cin], bias fp32; out either bf16 NHWC or fp32  */
int hp_conv3x3_small(const void* x, int32_t n, int32_t h, int32_t w, int32_t cin,
                     const float* wgt, const float* bias, int32_t cout, void* y,
                     int32_t y_is_f32, void* stream);
/* sinusoidal timestep embedding (flip_sin_to_cos, shift 0): out[b, dim] fp32 */
int hp_timestep_embedding(const float* t, int32_t b, int32_t dim, float max_period, float* out,
                          void* stream);
/* small-M linear for embeddings: y[M, N] = act_out(act_in(x)[M, K] W[N, K]^T + bias), fp32 io,
 * bf16 weights; act_* in {HP_ACT_NONE, HP_ACT_SILU}; M <= 8, K % 8 == 0,
 * M * K <= 40960 (x is staged in shared memory, act_in applied once)       */
int hp_linear_small(const float* x, int32_t M, int32_t K, const void* w, const float* bias,
                    int32_t N, int32_t act_in, int32_t act_out, float* y, void* stream);
/* patchify (inverse = 0): NHWC latent [n,h,w,c] -> tokens [n, (h/p)(w/p), p*p*c]
 * ordered (py, px, c); inverse = 1 maps tokens back to the latent.           */
int hp_patchify(const void* x, int32_t n, int32_t h, int32_t w, int32_t c, int32_t p,
                int32_t inverse, void* y, void* stream);
/* y[row, :] = x[row, :] + add[row % add_rows, :]  (positional embedding), bf16 */
int hp_add_rows(const void* x, const void* add, int64_t rows, int64_t add_rows, int32_t c,
                void* y, void* stream);
/* gated residual for adaLN-Zero: x[row, :] += gate[b, :] * y[row, :]        */
int hp_gated_residual(void* x, const void* y, const void* gate, int64_t ldg, int64_t rows,
                      int32_t c, int64_t rows_per_batch, void* stream);
/* bf16 -> fp32 copy with layout change NHWC(c) -> flat latent (same order) */
int hp_cast_bf16_f32(const void* x, float* y, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HYBRIDPAR_B200_DENOISER_H */
