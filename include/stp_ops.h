/*
 * stp_ops.h — kernel-level entry points of libstp.so.
 *
 * These are the hot-path operations every STP unit is made of (SURVEY §8a
 * rows a3-a10), exported individually so each kernel can be checked against
 * the CPU oracle on its own.  The executor behind stp_train_step (stp.h)
 * launches exactly these kernels.
 *
 * Conventions (all entry points):
 *  - Tensors are row-major DEVICE pointers; `dtype` (stp_dtype) selects fp32
 *    or bf16 storage for activations/weights; statistics (rstd, LSE, CE
 *    stats) and gradient accumulators are always fp32.  Arithmetic is fp32
 *    (fp32 accumulation in bf16 mode).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous on `stream`; errors from the launch are returned, errors
 *    during execution surface at the caller's next synchronisation.
 *  - Returns STP_EINVAL for bad sizes/alignment (message in stp_last_error),
 *    STP_ECUDA for launch failures.
 */
#ifndef STP_OPS_H_
#define STP_OPS_H_

#include <stdint.h>
#include "stp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ----------------------------------------------------------------- GEMM
 * The TP-sharded column/row-parallel linear layers (the
 * paper's Column/RowParallelLinear GEMMs):
 *   STP_GEMM_NT: C[M,N] = A[M,K] . B[N,K]^T   forward  Y = X W^T
 *   STP_GEMM_NN: C[M,N] = A[M,K] . B[K,N]     dgrad    dX = dY W
 *   STP_GEMM_TN: C[M,N] = A[K,M]^T . B[K,N]   wgrad    dW = dY^T X
 * lda/ldb/ldc are row strides in elements.  bf16: tcgen05 (TMEM accumulator,
 * TMA 128B-swizzled operands); requires lda, ldb, ldc % 8 == 0 and 16-byte
 * aligned bases.  fp32: true-fp32 SIMT FMA (no TF32).
 * Epilogues:
 *   STP_EPI_STORE:     C(dtype) = acc
 *   STP_EPI_BIAS:      C(dtype) = acc + bias[n]            (bias dtype)
 *   STP_EPI_ACCUM_F32: C(fp32) += acc                      (gradient accumulation)
 *   STP_EPI_RESID:     C(dtype) = acc + R[m*ldr + n]       (residual add, R dtype)
 *   STP_EPI_SWIGLU_BWD: C is the [M, 2N] tensor [G | U] (ldc >= 2N) of the MLP unit's
 *                      gate / up projections; with dH = acc, IN PLACE:
 *                      C[m, n]   = dH * U * s(G) * (1 + G * (1 - s(G)))   (dG)
 *                      C[m, N+n] = dH * G * s(G)                         (dU)
 *                      s = logistic: the SwiGLU backward (P:L70 MLP unit,
 *                      SURVEY §8c.1) fused into the FC2 activation-gradient GEMM
 * `max_ctas` caps the persistent grid (0 = all SMs) so TP communication
 * kernels can run beside the GEMM. */
typedef enum { STP_GEMM_NT = 0, STP_GEMM_NN = 1, STP_GEMM_TN = 2 } stp_gemm_layout;
typedef enum { STP_EPI_STORE = 0, STP_EPI_BIAS = 1, STP_EPI_ACCUM_F32 = 2, STP_EPI_RESID = 3,
               STP_EPI_SWIGLU_BWD = 4,
               STP_EPI_STORE_CE = 5  /* internal: LM head store + fp32 CE row statistics (stp_op_lm_head_ce) */
} stp_epilogue;

stp_status stp_op_gemm(int32_t dtype, int32_t layout, int32_t epilogue,
                       int64_t M, int64_t N, int64_t K,
                       const void* A, int64_t lda, const void* B, int64_t ldb,
                       void* C, int64_t ldc, const void* bias, const void* R, int64_t ldr,
                       int32_t max_ctas, void* stream);

/* -------------------------------------------------------------- RMSNorm
 * y = gamma * x * rstd, rstd = (mean_h x^2 + eps)^(-1/2)  (Pre-Attn/Pre-MLP
 * units; RMSNorm reading Q9).  rows x h; rstd_out fp32 [rows]
 * (nullable).  If resid != NULL the input is x + resid and the sum is written
 * to x_out (fused residual add of Eq. 1, SP form Q10); else x_out may be NULL. */
stp_status stp_op_rmsnorm_fwd(int32_t dtype, int64_t rows, int64_t h,
                              const void* x, const void* resid, void* x_out,
                              const void* gamma, float eps, void* y, float* rstd_out,
                              void* stream);
/* dx = rstd*(g*dy) - x*rstd^3*mean_h(g*dy*x) (+ dres if non-NULL: the "+1"
 * residual term of Eq. 2); dgamma_acc (fp32 [h], nullable) += sum_rows
 * dy*x*rstd. */
stp_status stp_op_rmsnorm_bwd(int32_t dtype, int64_t rows, int64_t h,
                              const void* dy, const void* x, const void* gamma,
                              const float* rstd, const void* dres, void* dx,
                              float* dgamma_acc, void* stream);

/* ------------------------------------------------------------------ RoPE
 * Rotate-half RoPE (theta, positions pos0..pos0+s-1) applied in place to
 * n_heads heads of width d starting at column col0 of a [s, ld] buffer:
 * x' = x*cos + rot(x)*sin; backward: dx = dx'*cos - rot(dx'*sin). */
stp_status stp_op_rope(int32_t dtype, int32_t backward, int64_t s, int64_t ld, int64_t col0,
                       int32_t n_heads, int32_t d, float theta, int64_t pos0,
                       void* x, void* stream);

/* --------------------------------------------------------------- SwiGLU
 * gu = [G | U] (s x 2I, ld_gu); H = silu(G)*U (s x I).  Backward writes
 * dGU = [dG | dU] from dH, G, U. */
stp_status stp_op_swiglu_fwd(int32_t dtype, int64_t s, int64_t I, const void* gu, void* H,
                             void* stream);
stp_status stp_op_swiglu_bwd(int32_t dtype, int64_t s, int64_t I, const void* dH,
                             const void* gu, void* dgu, void* stream);

/* ------------------------------------------------------------ attention
 * Causal GQA attention, scale 1/sqrt(d) (FlashAttention-2's role in the
 * paper; math SURVEY §8c.1).  q/k/v point at the first q/k/v column
 * of row 0; rows have stride ld_qkv (elements); head i of q uses kv head
 * i / (nq/nkv).  o: [s, nq*d] (ld_o); lse: fp32 [nq, s] (natural-log
 * log-sum-exp of the scaled, masked scores). */
stp_status stp_op_attn_fwd(int32_t dtype, int64_t s, int32_t nq, int32_t nkv, int32_t d,
                           const void* q, const void* k, const void* v, int64_t ld_qkv,
                           void* o, int64_t ld_o, float* lse, void* stream);
/* dO -> dQ, dK, dV (written, not accumulated; dK/dV summed over each kv
 * head's query heads).  dq/dk/dv have the q/k/v layout (ld_dqkv). `ws` is an
 * fp32 workspace of stp_op_attn_bwd_ws_bytes(...) bytes. */
int64_t stp_op_attn_bwd_ws_bytes(int64_t s, int32_t nq, int32_t nkv, int32_t d);
stp_status stp_op_attn_bwd(int32_t dtype, int64_t s, int32_t nq, int32_t nkv, int32_t d,
                           const void* q, const void* k, const void* v, int64_t ld_qkv,
                           const void* o, int64_t ld_o, const void* dout, const float* lse,
                           void* dq, void* dk, void* dv, int64_t ld_dqkv,
                           void* ws, void* stream);

/* ------------------------------------------- ViT first chunk (MLLM, cfg5)
 * The heterogeneous first virtual stage of the MLLM workload: "the ViT encoder
 * is assigned to the first virtual stage on device 0" (§5 P:L171;
 * Table 3).  Model: Qwen2-VL's vision tower + 2x2 merger as
 * oracle/vit.py restates it (readings V1-V4 in DESIGN.md).
 *
 * Bidirectional multi-head attention (no GQA: nh q, k and v heads) over the
 * fused [q | k | v] row layout of the QKV projection: qkv [s, ld_qkv] holds
 * q heads at columns [0, nh d), k at [nh d, 2 nh d), v at [2 nh d, 3 nh d).
 * O = softmax(Q K^T / sqrt(d)) V per head; lse fp32 [nh, s].  bf16 needs
 * d in {80, 128} (tcgen05 kernels; d = 80 heads are zero-padded to 128 in
 * shared memory by TMA) and ld_qkv = 3 nh d; fp32 runs SIMT kernels (d <= 128).
 * Backward writes dqkv in the same layout (ld_dqkv = 3 nh d for bf16); ws is
 * stp_op_attn_bwd_ws_bytes(s, nh, nh, d) bytes. */
stp_status stp_op_attn_full_fwd(int32_t dtype, int64_t s, int32_t nh, int32_t d, const void* qkv, int64_t ld_qkv,
                                void* o, int64_t ld_o, float* lse, void* stream);
stp_status stp_op_attn_full_bwd(int32_t dtype, int64_t s, int32_t nh, int32_t d, const void* qkv, int64_t ld_qkv,
                                const void* o, int64_t ld_o, const void* dout, const float* lse, void* dqkv,
                                int64_t ld_dqkv, void* ws, void* stream);
/* LayerNorm y = gamma (x - mu) r + beta, r = (var + eps)^(-1/2) over h
 * (biased variance), rows x h row-major.  If resid != NULL the input is
 * x + resid and the sum is written to x_out (the residual add of the SP comm
 * phase).  mean_out / rstd_out fp32 [rows] (nullable).  h % 8 == 0,
 * h <= 4096 (bf16) / 2048 (fp32), 16-byte aligned rows. */
stp_status stp_op_layernorm_fwd(int32_t dtype, int64_t rows, int64_t h, const void* x, const void* resid, void* x_out,
                                const void* gamma, const void* beta, float eps, void* y, float* mean_out,
                                float* rstd_out, void* stream);
/* dx = r (gamma dy - mean_h(gamma dy) - xhat mean_h(gamma dy xhat)) (+ dres),
 * xhat = (x - mu) r; dgamma_acc += sum_rows dy xhat, dbeta_acc += sum_rows dy
 * (fp32 [h], nullable).  x is the LayerNorm input; dx may alias dres. */
stp_status stp_op_layernorm_bwd(int32_t dtype, int64_t rows, int64_t h, const void* dy, const void* x,
                                const void* gamma, const float* mean, const float* rstd, const void* dres, void* dx,
                                float* dgamma_acc, float* dbeta_acc, void* stream);
/* Elementwise activation over n elements (n % 8 == 0, 16-byte aligned):
 * kind 0 QuickGELU y = a sigmoid(1.702 a) (ViT MLP); kind 1 GELU
 * y = a Phi(a), erf form (merger MLP).  Backward: da = dy act'(a) (da may
 * alias dy). */
stp_status stp_op_act_fwd(int32_t dtype, int32_t kind, int64_t n, const void* a, void* y, void* stream);
stp_status stp_op_act_bwd(int32_t dtype, int32_t kind, int64_t n, const void* dy, const void* a, void* da,
                          void* stream);
/* 2-D vision RoPE (rotate-half) in place on n_heads heads of width d at
 * column col0 of a [s, ld] buffer whose rows are the patches of a
 * (s / grid_w) x grid_w image in 2x2 merge-window order: angle j < d/4 is
 * h_pos inv_j, d/4 <= j < d/2 is w_pos inv_{j-d/4}, inv_j = theta^(-2j/(d/2))
 * (oracle/vit.py vit_rope_tables).  grid_w and s / grid_w even. */
stp_status stp_op_rope2d(int32_t dtype, int32_t backward, int64_t s, int64_t ld, int64_t col0, int32_t n_heads,
                         int32_t d, int32_t grid_w, float theta, void* x, void* stream);

/* ------------------------------------------------- vocab-parallel pieces
 * Embedding (vocab rows [v0, v0+Vl) on this rank): out[i] = E[tok_i - v0] if
 * tok_i in range else 0 (the TP partial summed by the reduce-scatter). */
stp_status stp_op_embed_fwd(int32_t dtype, int64_t s, int64_t h, const int32_t* tok,
                            int64_t v0, int64_t Vl, const void* E, void* out, void* stream);
/* dE_acc (fp32 [Vl, h]) += rows of dX for tokens in range (scatter-add). */
stp_status stp_op_embed_bwd(int32_t dtype, int64_t s, int64_t h, const int32_t* tok,
                            int64_t v0, int64_t Vl, const void* dX, float* dE_acc, void* stream);
/* Local cross-entropy statistics of logits [s, Vl] (ld): stats fp32 [s, 3] =
 * (row max, sum exp(z - max), target logit or 0 if target not in range). */
stp_status stp_op_ce_stats(int32_t dtype, int64_t s, int64_t Vl, const void* logits, int64_t ld,
                           const int32_t* tgt, int64_t v0, float* stats, void* stream);
/* Combine t ranks' stats (fp32 [t, s, 3], gathered) -> lse fp32 [s] and
 * loss_acc (fp32 scalar) += loss_scale * sum_i (lse_i - target_logit_i). */
stp_status stp_op_ce_combine(int64_t s, int32_t t, const float* stats_all, float* lse,
                             float* loss_acc, float loss_scale, void* stream);
/* LM head fused with the local CE statistics (F_HEAD unit; reading Q18, fp32
 * statistics): logits[s, Vl] = xf[s, h] W[Vl, h]^T stored in dtype (for the
 * backward), and stats fp32 [s, 3] computed from the fp32 accumulators in the
 * GEMM epilogue (bf16) before rounding: (row max, sum exp(z - max), target
 * logit or 0).  ws: stp_op_lm_head_ce_ws_bytes(s, Vl) bytes of device scratch. */
int64_t stp_op_lm_head_ce_ws_bytes(int64_t s, int64_t Vl);
stp_status stp_op_lm_head_ce(int32_t dtype, int64_t s, int64_t Vl, int64_t h, const void* xf, const void* W,
                             void* logits, const int32_t* tgt, int64_t v0, void* ws, float* stats, void* stream);
/* dlogits = grad_scale * (softmax - onehot) written in place over logits. */
stp_status stp_op_ce_grad(int32_t dtype, int64_t s, int64_t Vl, void* logits, int64_t ld,
                          const int32_t* tgt, int64_t v0, const float* lse, float grad_scale,
                          void* stream);

/* Column sum (bias gradient): acc fp32 [n] += sum_rows X[rows, n] (ld). */
stp_status stp_op_colsum_acc(int32_t dtype, int64_t rows, int64_t n, const void* X, int64_t ld,
                             float* acc, void* stream);
/* dst = src (elementwise dtype conversion fp32 <-> bf16 or copy), n elements. */
stp_status stp_op_convert(int32_t src_dtype, int32_t dst_dtype, int64_t n, const void* src,
                          void* dst, void* stream);
/* Number of SMs of the current device (for launch sizing / roofline). */
int32_t stp_num_sms(void);
/* Kernels launched by this library on the calling thread since load. */
int64_t stp_kernel_launches(void);

/* Runtime tuning knobs (process-wide; STP_EINVAL for unknown keys / values):
 *   "gemm_mc"  0 = 1-SM tcgen05 GEMM, 1 = automatic 1-SM / 2-SM choice per
 *              shape (default), 3 = always the 2-SM (cta_group::2) kernel
 * Kernel-variant environment switches (read once per process; the defaults
 * are the measured-faster variants, the alternatives exist for A/B runs,
 * DESIGN.md §7c):
 *   STP_GEMM_RASTER=0       m-block-fastest GEMM tile order
 *   STP_ATTN_BWD_ORDER=0    attention backward CTAs key-tile major over all heads
 *                           (default: grouped by kv head)
 *   STP_ATTN_DQ_BULK=0      attention backward dQ drained with per-element
 *                           red.add (default for d = 128: smem + bulk reductions)
 *   STP_LN_ROWBLOCK=0       warp-per-row LayerNorm kernels (default: a row per
 *                           128-thread CTA for h <= 4096)
 *   STP_DGAMMA_VEC=1        vectorised RMSNorm dgamma column reduction
 *   STP_ATTN_MMA_SYNC=1     d = 128 attention on the mma.sync kernels instead
 *                           of tcgen05 (the recompiled-baseline comparison)
 *   STP_GEMM_MC=n           initial value of "gemm_mc" */
stp_status stp_set_option(const char* key, int64_t value);

/* ------------------------------------------------------------ profiling
 * Kernel-class profiler (calling thread): when enabled, each launch of class
 * cls (0 GEMM, 1 attention fwd, 2 attention bwd) is bracketed by CUDA events
 * on its own stream and tagged with its algorithmic FLOPs and bytes.
 * stp_prof_read synchronises on the recorded events and returns the launch
 * count and the sums (ms = summed per-launch event time). */
stp_status stp_prof_enable(int32_t on);
stp_status stp_prof_reset(void);
stp_status stp_prof_read(int32_t cls, int64_t* count, double* flops, double* bytes, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* STP_OPS_H_ */
