/*
 * stp.h — C ABI of the B200 STP library (libstp.so).
 *
 * Synergistic Tensor + Pipeline parallel schedule (STP), arXiv 2510.27257:
 * "decouples the forward and backward passes in PP into fine-grained
 * computation units, which are then braided to form a composite computation
 * sequence" (PAPER.md abstract, P:L8), units = Pre-Attn/Attn/Pre-MLP/MLP with
 * backward split into activation-gradient B and weight-gradient W (§3,
 * P:L66-70), under a V-shape PP schedule (§4).
 *
 * Conventions
 *  - Every call returns stp_status; STP_OK = 0, negative = error.  The
 *    message of the last failing call on this thread is stp_last_error().
 *  - No exceptions cross the ABI.  No torch types: plain pointers and sizes.
 *  - "device" pointers are CUDA global-memory pointers of the current device;
 *    "host" pointers are ordinary CPU memory.
 *  - Microbatch indices are 1-based (Fig. 5 numbering); -1 = absent.
 *  - Handles (stp_schedule, stp_stage) are library-owned; the caller frees
 *    them with the matching stp_free_ / stp_destroy_ call.
 */
#ifndef STP_H_
#define STP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
typedef enum {
  STP_OK = 0,
  STP_EINVAL = -1,        /* bad argument / config (message says which) */
  STP_EUNSUPPORTED = -2,  /* valid but unsupported combination */
  STP_ENOMEM = -3,        /* device or host allocation failed */
  STP_ECUDA = -4,         /* a CUDA runtime / driver call failed */
  STP_ENCCL = -5,         /* an NCCL call failed */
  STP_ESCHEDULE = -6,     /* schedule construction failed (e.g. deadlock) */
  STP_ESTATE = -7,        /* handle poisoned by an earlier CUDA/NCCL error */
  STP_ECAPACITY = -8      /* caller buffer too small; *n_out holds the need */
} stp_status;

/* Thread-local message of the last failing stp_* call on this thread; valid
 * until the next stp_* call on the same thread.  Never NULL. */
const char* stp_last_error(void);
/* Library version string, e.g. "stp-b200 0.1 (sm_100a)". */
const char* stp_version(void);

/* ------------------------------------------------------------- schedule */
/* Schedule kinds.  STP = the R-STP reading of §4.2 with the
 * App. A warm-up rule; 1F1B_I = Megatron interleaved 1F1B with two
 * virtual stages; ZB = ZB-V-style greedy (V-shape, B/W split, 2p
 * memory cap); STP_NOBRAID = STP actions expanded without interleaving;
 * STP_NOSEP = STP slot grid without W separation; 1F1B_I_NAIVE = 1F1B-I with
 * every backward TP communication synchronous; 1F1B = PipeDream 1F1B (v=1).
 * Exact definitions: DESIGN.md "Schedules". */
typedef enum {
  STP_SCHED_STP = 0,
  STP_SCHED_1F1B_I = 1,
  STP_SCHED_ZB = 2,
  STP_SCHED_STP_NOBRAID = 3,
  STP_SCHED_STP_NOSEP = 4,
  STP_SCHED_1F1B_I_NAIVE = 5,
  STP_SCHED_1F1B = 6,
  STP_SCHED_STP_MEM = 7   /* Ours^: memory-efficient warm-up (App. A Fig. 8b, App. B (d); reading R4) */
} stp_sched_kind;

/* Action kinds (Fig. 5 caption P:L112 and §4.2: F, B, W, F&B, F&W). */
typedef enum {
  STP_A_F = 0,      /* lone forward of (chunk, f_mb) */
  STP_A_BFULL = 1,  /* lone full backward (B+W) of (chunk, b_mb) */
  STP_A_B = 2,      /* lone activation backward; W deferred */
  STP_A_W = 3,      /* lone weight backward of (w_chunk, w_mb) */
  STP_A_FB = 4,     /* braided F(f_mb) & full backward(b_mb), same chunk (Fig. 3a) */
  STP_A_FBS = 5,    /* braided F(f_mb) & activation backward(b_mb) (Fig. 3b) */
  STP_A_FW = 6      /* braided F(f_mb) & deferred W(w_mb, w_chunk) */
} stp_act_kind;

typedef struct {
  int32_t kind, chunk, f_mb, b_mb, w_mb, w_chunk; /* -1 = absent */
} stp_action;

/* Unit ops of the expansion. */
typedef enum {
  STP_U_F_ATTN = 0, STP_U_F_MLP = 1, STP_U_B_MLP = 2, STP_U_B_ATTN = 3,
  STP_U_W_MLP = 4, STP_U_W_ATTN = 5,
  STP_U_CF = 6,      /* forward TP comm phase (RS + residual + RMSNorm + AG) */
  STP_U_CB = 7,      /* backward TP comm phase (RS + RMSNorm-bwd + residual grad + AG) */
  STP_U_F_EMB = 8, STP_U_W_EMB = 9,
  STP_U_F_HEAD = 10, STP_U_B_HEAD = 11, STP_U_W_HEAD = 12,
  STP_U_PP_SEND = 13, STP_U_PP_RECV = 14,
  /* MLLM first virtual stage (stp_schedule_units_mllm): 2x2 merger + text
   * embedding producing the LM input (F), its activation gradient (B) and
   * its weight gradients (W) */
  STP_U_F_MERGE = 15, STP_U_B_MERGE = 16, STP_U_W_MERGE = 17
} stp_unit_op;

typedef struct {
  int32_t action;   /* index into the rank's action list */
  int32_t stream;   /* 0 compute, 1 TP-comm, 2 PP */
  int32_t op;       /* stp_unit_op */
  int32_t layer;    /* global layer (F/B/W units); phase index k (CF/CB); peer device (PP); else -1 */
  int32_t chunk, mb;
  int32_t dep0, dep1; /* indices of units this one waits on across streams; -1 = none */
} stp_unit;

typedef struct stp_schedule stp_schedule;

/* Build the per-PP-rank action lists for `kind` (pure, host-only,
 * deterministic).  pp >= 1, vpp = 2 (1 for STP_SCHED_1F1B), tp >= 1 (recorded
 * only), n_micro >= 1; 1F1B_I needs n_micro % pp == 0 (else STP_EUNSUPPORTED).
 * *out receives a new handle (free with stp_free_schedule). */
stp_status stp_build_schedule(int32_t pp, int32_t vpp, int32_t tp, int32_t n_micro,
                              int32_t kind, stp_schedule** out);
/* Copy rank pp_rank's actions into buf[0..cap).  *n_out is always set to the
 * number of actions; STP_ECAPACITY if cap < *n_out (nothing partial is
 * guaranteed). */
stp_status stp_schedule_actions(const stp_schedule* s, int32_t pp_rank,
                                stp_action* buf, int32_t cap, int32_t* n_out);
/* Unit-level expansion of rank pp_rank's actions (braid pairing, comm phases,
 * PP send/recv, cross-stream deps).  layers_per_vstage: host array of
 * pp*vpp layer counts in virtual-stage order (vs 0 holds layers 0..).  Same
 * capacity protocol as stp_schedule_actions. */
stp_status stp_schedule_units(const stp_schedule* s, int32_t pp_rank,
                              const int32_t* layers_per_vstage,
                              stp_unit* buf, int32_t cap, int32_t* n_out);
/* MLLM variant (§5: "the ViT encoder is assigned to the first
 * virtual stage on device 0"): layers_per_vstage[0] is the number of ViT
 * layers on virtual stage 0 (global layers 0..n_vit-1; the LM layers follow),
 * whose forward lane is F_EMB (patch embedding), the ViT layers' F_ATTN /
 * F_MLP and F_MERGE; its backward lane starts with B_MERGE, its W list with
 * W_MERGE (reading V5). */
stp_status stp_schedule_units_mllm(const stp_schedule* s, int32_t pp_rank,
                                   const int32_t* layers_per_vstage,
                                   stp_unit* buf, int32_t cap, int32_t* n_out);
/* Canonical text: header, then per rank "rank d", A lines and
 * (if layers_per_vstage != NULL) U lines.  Writes at most cap bytes incl. the
 * terminating NUL; *n_out = length without NUL; STP_ECAPACITY if too small. */
stp_status stp_schedule_serialize(const stp_schedule* s, const int32_t* layers_per_vstage,
                                  char* buf, int64_t cap, int64_t* n_out);
/* Same for the MLLM expansion (header line ends with " mllm"). */
stp_status stp_schedule_serialize_mllm(const stp_schedule* s, const int32_t* layers_per_vstage,
                                       char* buf, int64_t cap, int64_t* n_out);
/* Max number of chunk-microbatches whose forward was issued and whose weight
 * gradient was not, walking rank pp_rank's list in order (= stash slots). */
stp_status stp_schedule_stash_slots(const stp_schedule* s, int32_t pp_rank, int32_t* n_out);
void stp_free_schedule(stp_schedule* s);

/* Paper's layer split (reading Q17): L+2 spread evenly over n_slots,
 * remainder to the earliest slots, then 2 taken from the last slot.
 * STP_EINVAL ("IndivisibleLayers") if a slot would be empty. */
stp_status stp_layer_split(int32_t n_layers, int32_t n_slots, int32_t* out);

/* ---------------------------------------------------------------- stage */
typedef enum { STP_DTYPE_F32 = 0, STP_DTYPE_BF16 = 1 } stp_dtype;

typedef struct {
  int32_t vocab, hidden, n_layers, n_q_heads, n_kv_heads, head_dim, ffn, seq;
  float rms_eps, rope_theta;
  int32_t qkv_bias;   /* 1 = Qwen2 QKV bias (reading Q11) */
  int32_t dtype;      /* stp_dtype of params/activations; grads are always fp32 */
} stp_model_cfg;

typedef struct {
  int32_t tp, pp, vpp, n_micro, tp_rank, pp_rank;
  const int32_t* layers_per_vstage; /* host [pp*vpp], vs order; NULL = stp_layer_split */
  int32_t sched_kind;               /* stp_sched_kind used by stp_train_step */
} stp_parallel_cfg;

typedef struct stp_stage stp_stage;

/* Size of the opaque NCCL unique id blob (ncclUniqueId). */
int32_t stp_nccl_id_bytes(void);
/* Create a new NCCL unique id into buf (stp_nccl_id_bytes() bytes). */
stp_status stp_nccl_get_id(void* buf);

/* Create rank (pp_rank, tp_rank)'s stage on CUDA device cuda_device.
 * world_nccl_id: the world communicator's ncclUniqueId bytes (rank
 * pp_rank*tp + tp_rank of tp*pp), identical on all ranks (broadcast by the
 * caller, e.g. with torch.distributed); NULL allowed only when tp*pp == 1.
 * The library derives the TP and PP communicators with ncclCommSplit.
 * Streams are created internally.  Parameters are bound separately.
 * TP transport (env STP_TP_TRANSPORT, read here): "p2p" maps the TP peers'
 * stash slots / partial buffers / flag words with CUDA IPC (all TP ranks on
 * one node, peer access over NVLink) and runs each comm phase as one fused
 * NVLink kernel; "ce" pulls the rows with the copy engines over the same
 * mappings and reduces / normalises in one local kernel; "nccl" uses NCCL
 * reduce-scatter / all-gather.  Default: "ce" for the braided schedules (STP,
 * STP-NOSEP), "p2p" for the others, "nccl" for MLLM stages.  An IPC or peer-access failure returns
 * STP_ECUDA with the CUDA error text.  Multi-rank stages require
 * CUDA_DEVICE_MAX_CONNECTIONS >= 16 (STP_EUNSUPPORTED otherwise).
 * Other environment knobs read here (all optional):
 *   STP_OFFLOAD_ALPHA  activation offloading (§4.3, R5):
 *                      fraction in [0, 1] of chunk 0's layers whose MLP
 *                      activations live in pinned host memory between their
 *                      forward and backward; needs page-locked host memory
 *   STP_GRAPH=1        replay each step as one CUDA graph once the device
 *                      inputs repeat (TP = 1 or STP_TP_TRANSPORT=nccl)
 *   STP_P2P_PUSH=1     p2p transport, bf16: the row-parallel GEMMs store
 *                      their partial rows straight into the TP peers' buffers
 *   STP_P2P_CTAS, STP_COMM_SMEM, STP_GEMM_MAX_CTAS   CTA caps / SM
 *                      partitioning between the comm kernels and the GEMMs
 *   STP_NCCL_TP_CTAS, STP_NCCL_PP_CTAS   NCCL maxCTAs of the TP (16) and PP
 *                      (4) communicators; STP_NCCL_REGISTER=1 registers the
 *                      stash with the TP communicator (NCCL transport)
 *   STP_CE_WAIT=spin   ce transport: spin-wait kernels instead of
 *                      cuStreamWaitValue32 for the peer flags
 *   STP_DEBUG=1        synchronise and log every unit */
stp_status stp_init_stage(const stp_model_cfg* model, const stp_parallel_cfg* par,
                          const void* world_nccl_id, int32_t cuda_device,
                          stp_stage** out);

/* ---- MLLM: the ViT encoder as the heterogeneous first virtual stage ----
 * PAPER.md §5: "In MLLM scenarios, the ViT encoder is assigned to the
 * first virtual stage on device 0, and the LM model is uniformly distributed
 * across the remaining virtual stages"; Table 3 P:L231-263.  Vision tower =
 * Qwen2-VL's (LayerNorm, bidirectional attention with 2-D RoPE, QuickGELU
 * MLP, biases) + 2x2 patch merger (LayerNorm, GELU MLP) as oracle/vit.py
 * restates it (readings V1-V5). */
typedef struct {
  int32_t hidden, n_layers, n_heads, head_dim, mlp, patch_dim;
  int32_t grid_h, grid_w;   /* image of grid_h x grid_w patches (both even),
                               rows in 2x2 merge-window order */
  float ln_eps, rope_theta; /* 1e-6, 10000 for Qwen2-VL */
} stp_vit_cfg;

/* As stp_init_stage, with virtual stage 0 = ViT + merger and the LM on
 * virtual stages 1..pp*vpp-1.  model->seq is the LM sequence: the first
 * n_img = grid_h*grid_w/4 rows are the merged image tokens, the rest text;
 * model->n_layers counts LM layers only.  par->layers_per_vstage (if given)
 * = [n_vit, LM layers of vs 1, ...]; NULL = [vit->n_layers, stp_layer_split(
 * n_layers, pp*vpp-1)] ("the last virtual stage also contains two
 * fewer layers").  TP shards the ViT like the LM (heads, MLP and merger
 * columns; sequence-parallel residual shards of grid_h*grid_w/tp rows).
 * Requires STP_TP_TRANSPORT=nccl when tp > 1 (STP_EUNSUPPORTED otherwise),
 * n_heads, mlp, 4*hidden % tp == 0, grid_h*grid_w % (4*tp) == 0, n_img <
 * model->seq, head_dim in {80, 128} for bf16. */
stp_status stp_init_stage_mllm(const stp_model_cfg* model, const stp_vit_cfg* vit,
                               const stp_parallel_cfg* par, const void* world_nccl_id,
                               int32_t cuda_device, stp_stage** out);
/* Bind the image patches for the next steps: DEVICE [n_micro, grid_h*grid_w,
 * patch_dim] in the model dtype (caller-owned, borrowed until rebound).  Only
 * the rank holding virtual stage 0 reads them.  For an MLLM stage the token
 * rows [n_micro, seq] of stp_train_step carry the text tokens at positions
 * n_img..seq-1 (positions 0..n_img-1 are ignored); targets cover all seq
 * positions. */
stp_status stp_stage_bind_images(stp_stage* st, const void* d_patches);

/* Parameter layout of a stage: for every layer held
 * by this rank (virtual stages of chunk 0 then chunk 1; layers ascending):
 *   ln1[h], wqkv[(nq/t+2*nkv/t)*d, h], bqkv[(nq/t+2*nkv/t)*d] (if qkv_bias),
 *   wo[h, nq/t*d], ln2[h], wgu[2*I/t, h], wd[h, I/t]
 * then, on the rank holding vs 0: embed[V/t, h]; on the rank holding the last
 * vs: final_ln[h], lm_head[V/t, h].  wqkv rows = [q heads of rank | k heads |
 * v heads]; wgu rows = [gate rows of rank | up rows]; V, I, heads split in
 * contiguous blocks by tp_rank.  Row-major, PyTorch Linear [out, in].
 * stp_stage_param_count gives the number of tensors; stp_stage_param_info
 * gives tensor i's name (static string), element count and dims. */
stp_status stp_stage_param_count(const stp_stage* st, int32_t* n_out);
stp_status stp_stage_param_info(const stp_stage* st, int32_t i, const char** name,
                                int64_t* numel, int64_t* dim0, int64_t* dim1);
/* Bind caller-owned device buffers: params (dtype of the model cfg) and fp32
 * gradient accumulators (same element counts), n = stp_stage_param_count.
 * Pointers stay borrowed for the stage's lifetime.  Gradients are ADDED to
 * (the caller zeroes them); replicated gammas receive the TP-summed grad. */
stp_status stp_bind_params(stp_stage* st, int32_t n, void* const* param_ptrs,
                           void* const* grad_ptrs);

typedef struct {
  double step_ms;         /* device time of the step on this rank (events) */
  double exposed_tp_ms;   /* compute-stream idle time waiting on TP comm */
  double pp_bubble_ms;    /* remaining compute-stream idle time */
  double compute_busy_ms; /* sum of compute-unit durations (if timed) */
  int64_t peak_act_bytes; /* stash bytes of the peak in-flight count */
  int32_t n_units;        /* units executed on this rank */
  int32_t n_kernels;      /* kernels this library launched in the step */
} stp_step_stats;

/* Timing mode of stp_train_step: 0 = none (fastest), 1 = per-unit CUDA events
 * (exposed-TP / PP-bubble accounting). */
stp_status stp_stage_set_timing(stp_stage* st, int32_t mode);

/* One synchronous training step (PAPER.md P:L119-122 over n_micro
 * microbatches, no optimizer): tokens/targets are DEVICE int32 [n_micro, seq]
 * (only the rank holding vs 0 reads tokens; only the rank holding the last
 * vs reads targets; others may pass NULL).  Gradients are accumulated into
 * the bound fp32 buffers with the 1/(seq*n_micro) loss scale (reading Q19).
 * *h_loss (host, nullable) = mean loss on the rank holding the last vs, 0
 * elsewhere.  Returns after the step's last event (synchronous).
 * Stream ordering: `stream` is the caller's cudaStream_t (NULL = the legacy
 * default stream).  The step's first kernel runs after everything the caller
 * enqueued on `stream` before the call (parameter writes, zeroed gradients,
 * token uploads); work the caller enqueues on `stream` afterwards is ordered
 * after the step.  The step itself runs on the stage's own streams. */
stp_status stp_train_step(stp_stage* st, const int32_t* d_tokens, const int32_t* d_targets,
                          float* h_loss, stp_step_stats* stats, void* stream);
/* Same, but tokens/targets are HOST int32 arrays copied to the device inside
 * the call (end-to-end path; the copies also wait for `stream`); *h_loss read
 * back to the host. */
stp_status stp_train_step_host(stp_stage* st, const int32_t* h_tokens, const int32_t* h_targets,
                               float* h_loss, stp_step_stats* stats, void* stream);

/* Executed unit trace of the last step: the unit ops in host-enqueue order,
 * same layout as stp_schedule_units (capacity protocol as above). */
stp_status stp_stage_trace(const stp_stage* st, stp_unit* buf, int32_t cap, int32_t* n_out);
/* Per-unit event times of the last timed step (ms from step start): start and
 * end per unit, n = n_units.  Requires timing mode 1. */
stp_status stp_stage_unit_times(const stp_stage* st, float* start_ms, float* end_ms,
                                int32_t cap, int32_t* n_out);
void stp_destroy_stage(stp_stage* st);

#ifdef __cplusplus
}
#endif
#endif /* STP_H_ */
