// Stream/event unit executor of one TP x PP rank.
//
// One stp_stage per rank process.  It owns three kinds of CUDA streams:
//   compute   F/B/W units (GEMMs, attention, SwiGLU, embedding, LM head)
//   tp-comm   the TP communication phases of the units (reduce-scatter ->
//             residual add + RMSNorm (fwd) / RMSNorm-bwd + residual grad
//             (bwd) -> all-gather), i.e. the Pre-Attn / Pre-MLP units placed
//             "according to their computational dependencies" (PAPER.md
//             P:L70) in the sequence-parallel form (reading Q10).  Transport
//             (STP_TP_TRANSPORT): p2p (default) = one fused NVLink kernel per
//             phase over IPC-mapped peer buffers (tpcomm.cu, ce_* / p2p_*
//             below), ce = copy-engine pulls, nccl = NCCL RS / AG
//   pp        one stream per (peer, direction) NCCL communicator for the PP
//             activation / gradient send-recv
// and executes its rank's unit list (stp_schedule_units) in order: every unit
// waits on the events of its dep0/dep1 units, runs, and records its own
// event.  A braided action therefore overlaps each TP comm phase of one
// microbatch with the next compute unit of the other microbatch (Fig. 3,
// P:L55-70) without any host synchronisation.
//
// Memory: per chunk a pool of stash slots (one per in-flight
// chunk-microbatch, count = the program-order peak), each holding every
// tensor the backward and the deferred weight-gradient units need; a slot is
// reacquired only after the events of its last readers (its last W unit and
// its PP sends).
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.h"
#include "schedule.h"

namespace stp {

// launchers from the other translation units
stp_status gemm_dispatch(int dtype, int layout, int epi, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                         const void* B, int64_t ldb, void* C, int64_t ldc, const void* bias, const void* R,
                         int64_t ldr, int max_ctas, cudaStream_t st);
stp_status rmsnorm_fwd(int dtype, int64_t rows, int64_t h, const void* x, const void* resid, void* x_out,
                       const void* g, float eps, void* y, float* rstd, cudaStream_t st);
stp_status rmsnorm_bwd(int dtype, int64_t rows, int64_t h, const void* dy, const void* x, const void* g,
                       const float* rstd, const void* dres, void* dx, float* dgamma, cudaStream_t st);
stp_status rope(int dtype, int backward, int64_t s, int64_t ld, int64_t col0, int nh, int d, float theta,
                int64_t pos0, void* x, cudaStream_t st);
stp_status swiglu_fwd(int dtype, int64_t s, int64_t I, const void* gu, void* H, cudaStream_t st);
stp_status swiglu_bwd(int dtype, int64_t s, int64_t I, const void* dH, const void* gu, void* dgu, cudaStream_t st);
stp_status embed_fwd(int dtype, int64_t s, int64_t h, const int32_t* tok, int64_t v0, int64_t Vl, const void* E,
                     void* out, cudaStream_t st);
stp_status embed_bwd(int dtype, int64_t s, int64_t h, const int32_t* tok, int64_t v0, int64_t Vl, const void* dX,
                     float* dE, cudaStream_t st);
stp_status ce_stats(int dtype, int64_t s, int64_t Vl, const void* logits, int64_t ld, const int32_t* tgt, int64_t v0,
                    float* stats, cudaStream_t st);
stp_status ce_combine(int64_t s, int t, const float* stats_all, float* lse, float* loss_acc, float scale,
                      cudaStream_t st);
stp_status ce_grad(int dtype, int64_t s, int64_t Vl, void* logits, int64_t ld, const int32_t* tgt, int64_t v0,
                   const float* lse, float scale, cudaStream_t st);
stp_status colsum_acc(int dtype, int64_t rows, int64_t n, const void* X, int64_t ld, float* acc, cudaStream_t st);
stp_status add(int dtype, int64_t n, const void* a, const void* b, void* out, cudaStream_t st);
stp_status attn_fwd(int dtype, int64_t s, int nq, int nkv, int d, int causal, const void* q, const void* k,
                    const void* v, int64_t ld, void* o, int64_t ldo, float* lse, cudaStream_t st);
stp_status attn_bwd(int dtype, int64_t s, int nq, int nkv, int d, int causal, const void* q, const void* k,
                    const void* v, int64_t ld, const void* o, int64_t ldo, const void* dout, const float* lse,
                    void* dq, void* dk, void* dv, int64_t ldd, void* ws, cudaStream_t st);
int64_t attn_bwd_ws_bytes(int64_t s, int nq, int nkv, int d);
// copy-engine TP transport (tpcomm.cu)
stp_status tp_signal(uint32_t* const* dst, int n, uint32_t val, cudaStream_t st);
stp_status tp_wait(const uint32_t* flag, uint32_t val, bool spin, cudaStream_t st);
stp_status tp_fused_fwd(int dtype, int64_t rows, int64_t h, const void* const* pieces, int np, const void* resid,
                        void* x_out, const void* g, float eps, float* rstd, void* const* dsts, int nd,
                        cudaStream_t st);
stp_status tp_fused_bwd(int dtype, int64_t rows, int64_t h, const void* const* pieces, int np, const void* x,
                        const void* g, const float* rstd, const void* dres, void* dx, void* dy_out,
                        void* const* dsts, int nd, cudaStream_t st);
stp_status rmsnorm_dgamma(int dtype, int64_t rows, int64_t h, const void* dy, const void* x, const float* rstd,
                          float* dgamma, cudaStream_t st);
stp_status convert(int sd, int dd, int64_t n, const void* src, void* dst, cudaStream_t st);
int64_t lm_head_ce_ws_bytes(int64_t s, int64_t Vl);
void gemm_push_targets(void* const* ptrs, int n, int64_t rows, int64_t off);
stp_status lm_head_ce(int dtype, int64_t s, int64_t Vl, int64_t h, const void* xf, const void* W, void* logits,
                      const int32_t* tgt, int64_t v0, void* ws, float* stats, int max_ctas, cudaStream_t st);
// ViT first chunk (vit.cu)
stp_status layernorm_fwd(int dtype, int64_t rows, int64_t h, const void* x, const void* resid, void* x_out,
                         const void* g, const void* b, float eps, void* y, float* mean, float* rstd, cudaStream_t st);
stp_status layernorm_bwd(int dtype, int64_t rows, int64_t h, const void* dy, const void* x, const void* g,
                         const float* mean, const float* rstd, const void* dres, void* dx, float* dg, float* db,
                         cudaStream_t st);
stp_status act_fwd(int dtype, int kind, int64_t n, const void* a, void* y, cudaStream_t st);
stp_status act_bwd(int dtype, int kind, int64_t n, const void* dy, const void* a, void* da, cudaStream_t st);
stp_status rope2d(int dtype, int backward, int64_t s, int64_t ld, int64_t col0, int nh, int d, int gw, float theta,
                  void* x, cudaStream_t st);

#define STP_NCCL_TRY(expr)                                                     \
  do {                                                                         \
    ncclResult_t r_ = (expr);                                                  \
    if (r_ != ncclSuccess) {                                                   \
      ::stp::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,              \
                       ncclGetErrorString(r_));                                \
      return STP_ENCCL;                                                        \
    }                                                                          \
  } while (0)

namespace {

struct Param {
  std::string name;
  int64_t d0 = 0, d1 = 1;
  void* p = nullptr;
  float* g = nullptr;
  int64_t numel() const { return d0 * d1; }
};

struct LayerIdx {
  int ln1 = -1, wqkv = -1, bqkv = -1, wo = -1, ln2 = -1, wgu = -1, wd = -1;
};

// ViT layer parameters (oracle/vit.py names; TP shards as the LM's)
struct VitIdx {
  int ln1_g = -1, ln1_b = -1, wqkv = -1, bqkv = -1, wo = -1, bo = -1, ln2_g = -1, ln2_b = -1, w1 = -1, b1 = -1,
      w2 = -1, b2 = -1;
};

// ViT layer stash: full-sequence [sv, .] buffers (after the all-gather) and
// [sv/t, hv] residual shards, with the LayerNorm statistics of the shard rows
struct VitSlotLayer {
  void *xn = nullptr, *qkv = nullptr, *o = nullptr, *x1 = nullptr, *xn2 = nullptr, *a = nullptr, *hh = nullptr,
       *xres = nullptr, *dy_attn = nullptr, *dqkv = nullptr, *dy_mlp = nullptr;
  float *lse = nullptr, *mean1 = nullptr, *rstd1 = nullptr, *mean2 = nullptr, *rstd2 = nullptr;
};

struct SlotLayer {
  void *xn = nullptr, *qkv = nullptr, *o = nullptr, *x1 = nullptr, *xn2 = nullptr, *gu = nullptr, *hh = nullptr,
       *xres = nullptr, *dy_attn = nullptr, *dqkv = nullptr, *dy_mlp = nullptr;
  float *lse = nullptr, *rstd1 = nullptr, *rstd2 = nullptr;
  // activation offloading (§4.3): [gu | hh] of an offloaded layer lives in a
  // pool block from F_MLP until its D2H copy, in host memory until the reload
  // before the backward, and in a pool block again until W_MLP
  int blk = -1;
  void* host = nullptr;
  cudaEvent_t ev_d2h = nullptr, ev_h2d = nullptr;
};

struct OffBlock {
  void* dev = nullptr;
  cudaEvent_t ev = nullptr;  // the last reader / writer of the previous occupant
  bool ev_valid = false, busy = false;
};

struct Slot {
  void* mem = nullptr;
  void *x_in = nullptr, *dx_in = nullptr;
  std::vector<SlotLayer> L;
  void *xf = nullptr, *logits = nullptr, *dx0 = nullptr;
  float *rstdf = nullptr, *stats = nullptr, *stats_all = nullptr, *lse_ce = nullptr;
  // ViT chunk (MLLM vs 0): layers, merger input / pre-activation / activation,
  // the LM-input shard it produces, the all-gathered LM-input gradient and the
  // running ViT residual gradient shard
  std::vector<VitSlotLayer> V;
  void *yq = nullptr, *z = nullptr, *gz = nullptr, *x_out = nullptr, *dylm = nullptr, *vdx = nullptr;
  float *meanq = nullptr, *rstdq = nullptr;
  bool busy = false;
  int mb = -1;
  std::vector<cudaEvent_t> free_events;  // readers of the previous occupant
};

struct Chunk {
  int c = 0, vs = 0, l0 = 0, nl = 0;
  bool first = false, last = false;
  bool vit = false;  // MLLM: virtual stage 0 = ViT + merger (layers l0..l0+nl-1 are ViT layers)
  std::vector<Slot> slots;
  std::map<int, int> mb2slot;
  size_t slot_bytes = 0;
};

}  // namespace
}  // namespace stp

struct stp_stage {
  // config
  stp_model_cfg mc{};
  int t = 1, p = 1, vpp = 2, m = 1, tp_rank = 0, pp_rank = 0, kind = 0, dtype = 1;
  int dev = 0;
  int64_t s = 0, sl = 0, h = 0, qh = 0, kh = 0, d = 0, qkv_w = 0, o_w = 0, fi = 0, Vl = 0;
  size_t es = 2;
  std::vector<int> lay;
  stp::Schedule sched;
  std::vector<stp_unit> units;
  // params
  std::vector<stp::Param> params;
  std::map<int, stp::LayerIdx> lidx;  // global layer -> indices
  int p_embed = -1, p_final = -1, p_lm = -1;
  bool bound = false;
  // MLLM (stp_init_stage_mllm): ViT dims, per rank
  bool mllm = false;
  stp_vit_cfg vc{};
  int64_t nvit = 0, sv = 0, svl = 0, hv = 0, vnh = 0, vd = 0, vqkv_w = 0, vo_w = 0, vml = 0, vpd = 0, n_img = 0,
          m4 = 0, m4l = 0;
  std::map<int, stp::VitIdx> vidx;
  int p_patch = -1, p_mln_g = -1, p_mln_b = -1, p_mw1 = -1, p_mb1 = -1, p_mw2 = -1, p_mb2 = -1;
  const void* patches = nullptr;
  void *vrtmp = nullptr, *vntmp = nullptr, *vdtmp_h = nullptr, *vdtmp_o = nullptr, *vdtmp_m = nullptr,
       *vattn_ws = nullptr;
  // activation offloading (§4.3, STP_OFFLOAD_ALPHA): the MLP
  // activations [gu | hh] of the first off_n layers of chunk 0 go to pinned
  // host memory after their forward and come back before their backward
  float off_alpha = 0.f;
  int off_n = 0;
  size_t off_bytes = 0;
  std::vector<stp::OffBlock> off_pool;
  cudaStream_t s_d2h = nullptr, s_h2d = nullptr;
  std::vector<void*> host_allocs;
  std::map<std::pair<int, int>, bool> off_reloaded;  // (chunk, mb) -> reload issued this pass
  int64_t off_d2h_bytes = 0, off_h2d_bytes = 0;
  // chunks
  std::vector<stp::Chunk> chunks;
  // streams / comms
  cudaStream_t s_comp = nullptr, s_comm = nullptr;
  // PP channels: one NCCL communicator + stream per virtual-stage edge
  // (src vs, dst vs) this rank sends or receives on (per-edge FIFO; a single
  // channel per device pair is not FIFO for ZB / 1F1B-I).
  std::map<std::pair<int, int>, cudaStream_t> s_send, s_recv;
  ncclComm_t world = nullptr, tpc = nullptr;
  std::map<std::pair<int, int>, ncclComm_t> c_send, c_recv;
  std::vector<std::pair<int, int>> unit_edge;  // per unit: PP edge (src vs, dst vs)
  std::vector<char> unit_fwd;                  // per unit: PP message belongs to a forward pass
  std::vector<std::pair<int, int>> edges_sorted;  // all PP edges of the grid, global order
  std::vector<ncclComm_t> owned;
  std::vector<std::pair<ncclComm_t, void*>> nccl_regs;  // ncclCommRegister handles
  // buffers
  void *pf = nullptr, *pb = nullptr;               // partial outputs (forward / backward lanes)
  void *rtmp = nullptr, *ntmp = nullptr;           // comm-stream temps [sl, h]
  void *dtmp_h = nullptr, *dtmp_o = nullptr;       // compute temps dH [s, fi], dO [s, o_w]
  void* attn_ws = nullptr;
  void* ce_ws = nullptr;                           // LM-head CE statistics partials
  float* dgamma = nullptr;                         // internal gamma grads (per layer ln1, ln2, + final)
  std::map<int, int> dgamma_off;                   // param index -> offset into dgamma
  int64_t dgamma_n = 0;
  float* loss_acc = nullptr;
  int32_t *tok_buf = nullptr, *tgt_buf = nullptr;  // for the host-input path
  std::vector<void*> allocs;
  // events
  std::vector<cudaEvent_t> ev_done;
  std::vector<cudaEvent_t> ev_t0, ev_t1;  // timing
  cudaEvent_t ev_base = nullptr, ev_end = nullptr, ev_caller = nullptr, ev_join = nullptr;
  cudaEvent_t ev_gstart = nullptr, ev_gend = nullptr;  // timing of a graph launch
  cudaEvent_t ev_last = nullptr;  // the step's last event the caller's stream waits on (ev_end / ev_gend)
  float* h_loss_pin = nullptr;  // pinned: the step's loss read-back (a fixed address for graph replay)
  // CUDA-graph replay of the step (STP_GRAPH=1)
  bool use_graph = false;
  cudaGraphExec_t graph_exec = nullptr;
  std::array<const void*, 3> graph_key{};
  int64_t graph_launches = 0, steps_done = 0;
  // partial buffers: one per lane with NCCL (the collective copies it out
  // before it completes), two per lane with the copy-engine transport (peers
  // pull from them; see ce_* below).  ev_*b[i]: the comm phase that last read
  // buffer i has finished on this rank.
  void *pfb[2] = {nullptr, nullptr}, *pbb[2] = {nullptr, nullptr};
  int pfi = 0, pbi = 0;
  cudaEvent_t ev_pfb[2] = {nullptr, nullptr}, ev_pbb[2] = {nullptr, nullptr};
  bool pfb_pending[2] = {false, false}, pbb_pending[2] = {false, false};
  bool pf_pending = false, pb_pending = false;  // the current comm phase read pf / pb
  // p2p push mode (STP_P2P_PUSH): the row-parallel GEMM of a unit writes row
  // block q of its partial into TP peer q's partial buffer at this rank's slice
  // (the reduce-scatter's NVLink transfer in the GEMM epilogue); pf_push /
  // pb_push: the current partial was pushed (the comm phase then reads t local
  // slices instead of pulling the peers' rows)
  bool p2p_push = false, pf_push = false, pb_push = false;
  // copy-engine TP transport (STP_TP_TRANSPORT=ce; tpcomm.cu)
  bool ce = false, ce_spin = false;
  bool p2p = false;              // STP_TP_TRANSPORT=p2p: fused NVLink load/store kernels instead of copy engines
  uint32_t* flags = nullptr;     // [2][16]: A (partials ready), B (shard ready), one word per peer
  uint32_t phase = 0, open_phase = 0;
  void* stage_buf = nullptr;     // [t, sl, h]: rows pulled from the peers' partials
  std::vector<std::pair<uint8_t*, size_t>> sym;  // symmetric allocations, same order on every TP rank
  std::vector<std::vector<uint8_t*>> sym_peer;   // [q][i]: IPC mapping of peer q's allocation i
  std::vector<cudaStream_t> s_pull;              // one per peer: concurrent copy-engine pulls
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_pool_next = 0;
  int timing = 0;
  bool poisoned = false;
  // per-step
  const int32_t* tokens = nullptr;
  const int32_t* targets = nullptr;
  std::vector<stp_unit> trace;
  std::vector<float> t_start, t_end;
  int gemm_max_ctas = 0;
  bool debug = false;
  int64_t launches_step = 0;
  int64_t peak_bytes = 0;
};

namespace stp {
namespace {

int ncdt(int dtype) { return dtype == STP_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32; }

stp_status dalloc(stp_stage* S, void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) return STP_OK;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
    return STP_ENOMEM;
  }
  S->allocs.push_back(*p);
  return STP_OK;
}

cudaEvent_t pool_event(stp_stage* S) {
  if (S->ev_pool_next >= S->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    S->ev_pool.push_back(e);
  }
  return S->ev_pool[S->ev_pool_next++];
}

// Carve a slot's buffers out of one allocation (256-byte aligned pieces).
struct Carver {
  uint8_t* base;
  size_t off = 0;
  bool dry;
  void* take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    void* p = dry ? nullptr : base + off;
    off += bytes;
    return p;
  }
};

void carve_vit_slot(stp_stage* S, const Chunk& C, Slot& sl, Carver& cv) {
  const size_t es = S->es;
  const int64_t sv = S->sv, hv = S->hv, vsh = S->svl * S->hv;
  sl.x_in = cv.take(vsh * es);
  sl.dx_in = cv.take(S->sl * S->h * es);
  sl.V.resize(C.nl);
  for (int j = 0; j < C.nl; ++j) {
    VitSlotLayer& L = sl.V[j];
    L.xn = cv.take(sv * hv * es);
    L.qkv = cv.take(sv * S->vqkv_w * es);
    L.o = cv.take(sv * S->vo_w * es);
    L.lse = (float*)cv.take(S->vnh * sv * 4);
    L.mean1 = (float*)cv.take(S->svl * 4);
    L.rstd1 = (float*)cv.take(S->svl * 4);
    L.mean2 = (float*)cv.take(S->svl * 4);
    L.rstd2 = (float*)cv.take(S->svl * 4);
    L.x1 = cv.take(vsh * es);
    L.xn2 = cv.take(sv * hv * es);
    L.a = cv.take(sv * S->vml * es);  // backward overwrites it with dA
    L.hh = cv.take(sv * S->vml * es);
    L.xres = cv.take(vsh * es);
    L.dy_attn = cv.take(sv * hv * es);
    L.dqkv = cv.take(sv * S->vqkv_w * es);
    L.dy_mlp = cv.take(sv * hv * es);
  }
  sl.yq = cv.take(sv * hv * es);                // = [n_img, 4 hv] merger input
  sl.meanq = (float*)cv.take(S->svl * 4);
  sl.rstdq = (float*)cv.take(S->svl * 4);
  sl.z = cv.take(S->n_img * S->m4l * es);        // backward overwrites it with dZ
  sl.gz = cv.take(S->n_img * S->m4l * es);
  sl.x_out = cv.take(S->sl * S->h * es);
  sl.dylm = cv.take(S->s * S->h * es);
  sl.vdx = cv.take(vsh * es);
}

void carve_slot(stp_stage* S, const Chunk& C, Slot& sl, Carver& cv) {
  if (C.vit) return carve_vit_slot(S, C, sl, cv);
  const size_t es = S->es;
  const int64_t s = S->s, h = S->h, shard = S->sl * S->h;
  sl.x_in = cv.take(shard * es);
  sl.dx_in = cv.take(shard * es);
  sl.L.resize(C.nl);
  for (int j = 0; j < C.nl; ++j) {
    SlotLayer& L = sl.L[j];
    L.xn = cv.take(s * h * es);
    L.qkv = cv.take(s * S->qkv_w * es);
    L.o = cv.take(s * S->o_w * es);
    L.lse = (float*)cv.take(S->qh * s * 4);
    L.rstd1 = (float*)cv.take(S->sl * 4);
    L.rstd2 = (float*)cv.take(S->sl * 4);
    L.x1 = cv.take(shard * es);
    L.xn2 = cv.take(s * h * es);
    if (C.c == 0 && !C.vit && j < S->off_n) {
      L.gu = L.hh = nullptr;  // pool block while on the device (offloaded layer)
    } else {
      L.gu = cv.take(s * 2 * S->fi * es);  // backward overwrites it with dGU
      L.hh = cv.take(s * S->fi * es);
    }
    L.xres = cv.take(shard * es);
    L.dy_attn = cv.take(s * h * es);
    L.dqkv = cv.take(s * S->qkv_w * es);
    L.dy_mlp = cv.take(s * h * es);
  }
  if (C.last) {
    sl.xf = cv.take(s * h * es);
    sl.rstdf = (float*)cv.take(S->sl * 4);
    sl.logits = cv.take(s * S->Vl * es);
    sl.stats = (float*)cv.take(s * 3 * 4);
    sl.stats_all = (float*)cv.take((size_t)S->t * s * 3 * 4);
    sl.lse_ce = (float*)cv.take(s * 4);
  }
  if (C.first) sl.dx0 = cv.take(s * h * es);
}

// ----------------------------------------------------------- collectives
stp_status reduce_scatter(stp_stage* S, const void* src, void* dst) {
  STP_NCCL_TRY(ncclReduceScatter(src, dst, (size_t)(S->sl * S->h), (ncclDataType_t)ncdt(S->dtype), ncclSum, S->tpc,
                                 S->s_comm));
  return STP_OK;
}
stp_status all_gather(stp_stage* S, const void* src, void* dst, size_t count) {
  if (S->t == 1) {
    if (src != dst) STP_CUDA_TRY(cudaMemcpyAsync(dst, src, count * S->es, cudaMemcpyDeviceToDevice, S->s_comm));
    return STP_OK;
  }
  STP_NCCL_TRY(ncclAllGather(src, dst, count, (ncclDataType_t)ncdt(S->dtype), S->tpc, S->s_comm));
  return STP_OK;
}

Chunk& chunk_of(stp_stage* S, int c) { return S->chunks[c]; }

// --------------------------------------------- copy-engine TP transport
// STP_TP_TRANSPORT=ce.  Every TP rank maps its peers' stash slots, partial
// buffers and flag words (CUDA IPC, exchanged once at init), and each comm
// phase c (numbered identically on all TP ranks: they run the same unit
// list) becomes
//   A(c): signal "my partial for c is ready and phase c-1 is done", wait for
//         the peers' A(c); pull this rank's rows of every peer's partial
//         (cudaMemcpyAsync over NVLink: copy engines, no SMs);
//         tp_fused_fwd: sum + residual (+ RMSNorm into this rank's rows of
//         the all-gather destination);
//   B(c): signal "my rows of the destination are written", wait for the
//         peers' B(c); pull every peer's rows of the destination.
// Safety without "consumed" flags: a rank completes phase c only after all
// peers signalled A(c) or B(c), i.e. finished phase c-1.  So when a rank
// overwrites a buffer peers pull from, every peer has finished the phases
// before the current one: partials alternate between two buffers per lane
// (two partial writes of a lane are separated by a phase that consumes the
// all-gather of the first), and a destination / dx_in region is rewritten
// only phases after its last pull.  See DESIGN.md "Copy-engine TP transport".
uint8_t* sym_peer_ptr(stp_stage* S, int q, const void* p) {
  const uint8_t* b = (const uint8_t*)p;
  for (size_t i = 0; i < S->sym.size(); ++i)
    if (b >= S->sym[i].first && b < S->sym[i].first + S->sym[i].second)
      return S->sym_peer[q][i] + (b - S->sym[i].first);
  return nullptr;
}

stp_status ce_handshake(stp_stage* S, int which, uint32_t c) {
  uint32_t* dst[16];
  int n = 0;
  for (int q = 0; q < S->t; ++q)
    if (q != S->tp_rank) {
      uint8_t* pf = sym_peer_ptr(S, q, S->flags);
      if (!pf) return fail(STP_ESTATE, "flag words not mapped");
      dst[n++] = (uint32_t*)pf + which * 16 + S->tp_rank;
    }
  STP_TRY(tp_signal(dst, n, c, S->s_comm));
  for (int q = 0; q < S->t; ++q)
    if (q != S->tp_rank) STP_TRY(tp_wait(S->flags + which * 16 + q, c, S->ce_spin, S->s_comm));
  return STP_OK;
}

// rows [q*sl, (q+1)*sl) of `dst` <- peer q's copy, for every peer q (ag), or
// stage[q] <- rows of this rank from peer q's `src` (rs); one copy-engine
// transfer per peer, concurrent on the per-peer pull streams.
stp_status ce_pull(stp_stage* S, bool rs, const void* src, void* dst) {
  const size_t bytes = (size_t)(S->sl * S->h) * S->es;
  cudaEvent_t fork = pool_event(S);
  STP_CUDA_TRY(cudaEventRecord(fork, S->s_comm));
  int k = 0;
  for (int q = 0; q < S->t; ++q) {
    if (q == S->tp_rank) continue;
    cudaStream_t ps = S->s_pull[k++];
    STP_CUDA_TRY(cudaStreamWaitEvent(ps, fork, 0));
    uint8_t* from = sym_peer_ptr(S, q, rs ? src : dst);
    if (!from) return fail(STP_ESTATE, "buffer not in the symmetric set");
    if (rs)
      STP_CUDA_TRY(cudaMemcpyAsync((uint8_t*)S->stage_buf + q * bytes, from + S->tp_rank * bytes, bytes,
                                   cudaMemcpyDeviceToDevice, ps));
    else
      STP_CUDA_TRY(cudaMemcpyAsync((uint8_t*)dst + q * bytes, from + q * bytes, bytes, cudaMemcpyDeviceToDevice, ps));
    cudaEvent_t e = pool_event(S);
    STP_CUDA_TRY(cudaEventRecord(e, ps));
    STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comm, e, 0));
  }
  return STP_OK;
}

// Reduce-scatter of `partial` (+ resid) into x_out; with g: RMSNorm into this
// rank's rows of `dst` and the all-gather of dst.  Opens phase c (kept in
// open_phase for a following ce_ag when dst is null).
stp_status ce_rs(stp_stage* S, const void* partial, const void* resid, void* x_out, const void* g, float* rstd,
                 void* dst);
stp_status ce_ag(stp_stage* S, void* dst) {
  const uint32_t c = S->open_phase ? S->open_phase : ++S->phase;
  S->open_phase = 0;
  STP_TRY(ce_handshake(S, 1, c));
  return ce_pull(S, false, nullptr, dst);
}
stp_status p2p_rs(stp_stage* S, const void* partial, const void* resid, void* x_out, const void* g, float* rstd,
                  void* dst);
stp_status ce_rs(stp_stage* S, const void* partial, const void* resid, void* x_out, const void* g, float* rstd,
                 void* dst) {
  if (S->p2p) return p2p_rs(S, partial, resid, x_out, g, rstd, dst);
  const uint32_t c = ++S->phase;
  STP_TRY(ce_handshake(S, 0, c));
  STP_TRY(ce_pull(S, true, partial, nullptr));
  const size_t bytes = (size_t)(S->sl * S->h) * S->es;
  const void* pieces[16];
  int n = 0;
  for (int q = 0; q < S->t; ++q)
    pieces[n++] = q == S->tp_rank ? (const uint8_t*)partial + q * bytes : (const uint8_t*)S->stage_buf + q * bytes;
  void* y = dst ? (uint8_t*)dst + S->tp_rank * bytes : nullptr;
  STP_TRY(tp_fused_fwd(S->dtype, S->sl, S->h, pieces, n, resid, x_out, g, S->mc.rms_eps, rstd, &y, y ? 1 : 0,
                       S->s_comm));
  S->open_phase = c;
  if (dst) return ce_ag(S, dst);
  return STP_OK;
}
// all-gather of a shard held elsewhere: copy it into this rank's rows of dst
stp_status ce_ag_shard(stp_stage* S, const void* shard, void* dst) {
  const size_t bytes = (size_t)(S->sl * S->h) * S->es;
  STP_CUDA_TRY(cudaMemcpyAsync((uint8_t*)dst + S->tp_rank * bytes, shard, bytes, cudaMemcpyDeviceToDevice,
                               S->s_comm));
  return ce_ag(S, dst);
}

// ---- p2p variant (STP_TP_TRANSPORT=p2p): one fused kernel per phase reads
// this rank's rows of every peer's partial over NVLink, reduces, applies the
// residual + RMSNorm (fwd) or RMSNorm-bwd + residual grad (bwd), and stores
// the result into this rank's rows of every rank's all-gather destination.
// Handshakes: A(c) before the kernel (peers' partials ready, destinations
// free), B(c) after it (every peer's rows have landed here).
int p2p_pieces(stp_stage* S, const void* partial, const void** pieces) {
  const size_t bytes = (size_t)(S->sl * S->h) * S->es;
  if ((partial == S->pf && S->pf_push) || (partial == S->pb && S->pb_push)) {
    for (int q = 0; q < S->t; ++q) pieces[q] = (const uint8_t*)partial + q * bytes;  // slice q: rank q's rows
    return S->t;
  }
  for (int q = 0; q < S->t; ++q) {
    const uint8_t* b = q == S->tp_rank ? (const uint8_t*)partial : sym_peer_ptr(S, q, partial);
    pieces[q] = b ? b + S->tp_rank * bytes : nullptr;
    if (!b) return -1;
  }
  return S->t;
}
int p2p_dsts(stp_stage* S, void* dst, void** dsts) {
  if (!dst) return 0;
  const size_t bytes = (size_t)(S->sl * S->h) * S->es;
  int n = 0;
  dsts[n++] = (uint8_t*)dst + S->tp_rank * bytes;  // local rows first (the kernel's scratch)
  for (int q = 0; q < S->t; ++q) {
    if (q == S->tp_rank) continue;
    uint8_t* b = sym_peer_ptr(S, q, dst);
    if (!b) return -1;
    dsts[n++] = b + S->tp_rank * bytes;
  }
  return n;
}
stp_status p2p_rs(stp_stage* S, const void* partial, const void* resid, void* x_out, const void* g, float* rstd,
                  void* dst) {
  const uint32_t c = ++S->phase;
  const void* pieces[16];
  void* dsts[16];
  const int np = p2p_pieces(S, partial, pieces), nd = p2p_dsts(S, dst, dsts);
  if (np < 0 || nd < 0) return fail(STP_ESTATE, "buffer not in the symmetric set");
  STP_TRY(ce_handshake(S, 0, c));
  STP_TRY(tp_fused_fwd(S->dtype, S->sl, S->h, pieces, np, resid, x_out, g, S->mc.rms_eps, rstd, dsts, nd,
                       S->s_comm));
  // nd == 0 (no all-gather): peers' reuse of this partial buffer is ordered by
  // the alternate-buffer argument (§8c); STP_DEBUG=1 adds the B handshake anyway
  // (every TP rank takes the same branch: same unit list, same environment)
  if (nd || S->debug) STP_TRY(ce_handshake(S, 1, c));
  return STP_OK;
}
// all-gather of a local shard (optionally RMSNorm-ed on the way)
stp_status p2p_ag(stp_stage* S, const void* shard, const void* g, float* rstd, void* dst) {
  const uint32_t c = ++S->phase;
  void* dsts[16];
  const int nd = p2p_dsts(S, dst, dsts);
  if (nd <= 0) return fail(STP_ESTATE, "buffer not in the symmetric set");
  STP_TRY(ce_handshake(S, 0, c));
  STP_TRY(tp_fused_fwd(S->dtype, S->sl, S->h, &shard, 1, nullptr, nullptr, g, S->mc.rms_eps, rstd, dsts, nd,
                       S->s_comm));
  return ce_handshake(S, 1, c);
}
// RS of the backward partial -> RMSNorm-bwd + residual grad -> AG (dst may be
// null); the dgamma partials follow, off the critical path.
stp_status p2p_bwd(stp_stage* S, const void* x, const void* g, const float* rstd, const void* dres, void* dx,
                   float* dgamma, void* dst) {
  const uint32_t c = ++S->phase;
  const void* pieces[16];
  void* dsts[16];
  const int np = p2p_pieces(S, S->pb, pieces), nd = p2p_dsts(S, dst, dsts);
  if (np < 0 || nd < 0) return fail(STP_ESTATE, "buffer not in the symmetric set");
  STP_TRY(ce_handshake(S, 0, c));
  STP_TRY(tp_fused_bwd(S->dtype, S->sl, S->h, pieces, np, x, g, rstd, dres, dx, S->rtmp, dsts, nd, S->s_comm));
  if (nd || S->debug) STP_TRY(ce_handshake(S, 1, c));
  return rmsnorm_dgamma(S->dtype, S->sl, S->h, S->rtmp, x, rstd, dgamma, S->s_comm);
}

// Copy-engine variant of p2p_bwd: pull this rank's rows of every peer's
// backward partial (copy engines), one fused kernel for the sum + RMSNorm-bwd +
// residual grad writing this rank's rows of dst, then the all-gather pulls.
// (Round 2: the separate RS-sum / RMSNorm-bwd / shard-copy kernels of the
// generic path made the copy-engine CB phase 1.7x the CF phase.)
stp_status ce_bwd(stp_stage* S, const void* x, const void* g, const float* rstd, const void* dres, void* dx,
                  float* dgamma, void* dst) {
  const uint32_t c = ++S->phase;
  STP_TRY(ce_handshake(S, 0, c));
  STP_TRY(ce_pull(S, true, S->pb, nullptr));
  const size_t bytes = (size_t)(S->sl * S->h) * S->es;
  const void* pieces[16];
  for (int q = 0; q < S->t; ++q)
    pieces[q] = q == S->tp_rank ? (const uint8_t*)S->pb + q * bytes : (const uint8_t*)S->stage_buf + q * bytes;
  void* y = dst ? (uint8_t*)dst + S->tp_rank * bytes : nullptr;
  STP_TRY(tp_fused_bwd(S->dtype, S->sl, S->h, pieces, S->t, x, g, rstd, dres, dx, S->rtmp, &y, y ? 1 : 0,
                       S->s_comm));
  S->open_phase = c;
  if (dst) STP_TRY(ce_ag(S, dst));
  return rmsnorm_dgamma(S->dtype, S->sl, S->h, S->rtmp, x, rstd, dgamma, S->s_comm);
}
stp_status fused_bwd(stp_stage* S, const void* x, const void* g, const float* rstd, const void* dres, void* dx,
                     float* dgamma, void* dst) {
  if (S->p2p) return p2p_bwd(S, x, g, rstd, dres, dx, dgamma, dst);
  return ce_bwd(S, x, g, rstd, dres, dx, dgamma, dst);
}

stp_status ag_dx(stp_stage* S, const void* shard_src, void* dst, size_t count) {
  if (S->p2p) return p2p_ag(S, shard_src, nullptr, nullptr, dst);
  if (S->ce) return ce_ag_shard(S, shard_src, dst);
  return all_gather(S, shard_src, dst, count);
}

// Map the peers' symmetric allocations (same order on every TP rank: every
// stash slot, both partial buffers of both lanes, the flag words).
stp_status ce_init(stp_stage* S) {
  S->sym.clear();
  for (auto& C : S->chunks)
    for (auto& sl : C.slots) S->sym.push_back({(uint8_t*)sl.mem, C.slot_bytes});
  const size_t pbytes = (size_t)(S->s * S->h) * S->es;
  for (int i = 0; i < 2; ++i) {
    S->sym.push_back({(uint8_t*)S->pfb[i], pbytes});
    S->sym.push_back({(uint8_t*)S->pbb[i], pbytes});
  }
  S->sym.push_back({(uint8_t*)S->flags, 4096});
  const int n = (int)S->sym.size();
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  std::vector<uint8_t> mine(n * hb), all((size_t)S->t * n * hb);
  for (int i = 0; i < n; ++i)
    STP_CUDA_TRY(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(mine.data() + i * hb), S->sym[i].first));
  void *dm = nullptr, *da = nullptr;
  STP_CUDA_TRY(cudaMalloc(&dm, mine.size()));
  STP_CUDA_TRY(cudaMalloc(&da, all.size()));
  STP_CUDA_TRY(cudaMemcpy(dm, mine.data(), mine.size(), cudaMemcpyHostToDevice));
  STP_NCCL_TRY(ncclAllGather(dm, da, mine.size(), ncclUint8, S->tpc, S->s_comm));
  STP_CUDA_TRY(cudaStreamSynchronize(S->s_comm));
  STP_CUDA_TRY(cudaMemcpy(all.data(), da, all.size(), cudaMemcpyDeviceToHost));
  cudaFree(dm);
  cudaFree(da);
  S->sym_peer.assign(S->t, std::vector<uint8_t*>(n, nullptr));
  for (int q = 0; q < S->t; ++q) {
    if (q == S->tp_rank) continue;
    for (int i = 0; i < n; ++i) {
      cudaIpcMemHandle_t hdl;
      memcpy(&hdl, all.data() + ((size_t)q * n + i) * hb, hb);
      void* p = nullptr;
      STP_CUDA_TRY(cudaIpcOpenMemHandle(&p, hdl, cudaIpcMemLazyEnablePeerAccess));
      S->sym_peer[q][i] = (uint8_t*)p;
    }
  }
  int lo = 0, hi = 0;
  STP_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  for (int q = 0; q + 1 < S->t; ++q) {
    cudaStream_t st;
    STP_CUDA_TRY(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
    S->s_pull.push_back(st);
  }
  // every rank has mapped everything before any phase signals
  STP_NCCL_TRY(ncclAllReduce(S->flags + 1000, S->flags + 1000, 1, ncclUint32, ncclMax, S->tpc, S->s_comm));
  STP_CUDA_TRY(cudaStreamSynchronize(S->s_comm));
  return STP_OK;
}


stp_status acquire(stp_stage* S, int c, int mb, Slot** out) {
  Chunk& C = chunk_of(S, c);
  auto it = C.mb2slot.find(mb);
  if (it != C.mb2slot.end()) {
    *out = &C.slots[it->second];
    return STP_OK;
  }
  for (size_t i = 0; i < C.slots.size(); ++i) {
    Slot& sl = C.slots[i];
    if (sl.busy) continue;
    sl.busy = true;
    sl.mb = mb;
    C.mb2slot[mb] = (int)i;
    // every stream that may write this slot waits for the previous readers
    for (cudaEvent_t e : sl.free_events) {
      STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comp, e, 0));
      STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comm, e, 0));
      for (auto& kv : S->s_recv) STP_CUDA_TRY(cudaStreamWaitEvent(kv.second, e, 0));
    }
    sl.free_events.clear();
    *out = &sl;
    return STP_OK;
  }
  return fail(STP_ESTATE, "no free stash slot (schedule / slot-count mismatch)");
}

Slot* find_slot(stp_stage* S, int c, int mb) {
  Chunk& C = chunk_of(S, c);
  auto it = C.mb2slot.find(mb);
  return it == C.mb2slot.end() ? nullptr : &C.slots[it->second];
}

void release(stp_stage* S, int c, int mb, cudaEvent_t comp_ev) {
  Chunk& C = chunk_of(S, c);
  auto it = C.mb2slot.find(mb);
  if (it == C.mb2slot.end()) return;
  Slot& sl = C.slots[it->second];
  sl.free_events.push_back(comp_ev);
  sl.busy = false;
  sl.mb = -1;
  C.mb2slot.erase(it);
}

int dev_of_vs(stp_stage* S, int vs) { return sched_vstage_device(S->kind, S->p, vs); }

const stp::LayerIdx& LI(stp_stage* S, int l) { return S->lidx.at(l); }
void* P(stp_stage* S, int i) { return S->params[i].p; }
float* G(stp_stage* S, int i) { return S->params[i].g; }
float* DG(stp_stage* S, int i) { return S->dgamma + S->dgamma_off.at(i); }

int64_t vocab0(stp_stage* S) { return (int64_t)S->tp_rank * S->Vl; }

// ------------------------------------------------------------ ViT units
// The MLLM's first virtual stage (math oracle/vit.py).
// Same unit / comm-phase structure as the LM chunk (Fig. 3 reading R2):
// F_EMB = patch embedding of this rank's sequence-parallel shard rows;
// F_ATTN / F_MLP per ViT layer; F_MERGE = 2x2 merger (the [sv, hv] LayerNorm
// output read as [sv/4, 4 hv]) + vocab-parallel text embedding, one [S, h]
// LM-input partial.  Row-parallel biases (wo, w2, merger w2) are added by TP
// rank 0's GEMM epilogue only, so the reduce-scatter sums them once; their
// gradients are column sums of the all-gathered dY (identical on every rank).
stp_status vit_compute(stp_stage* S, const stp_unit& u, Slot* sl) {
  const int dt = S->dtype, mc = S->gemm_max_ctas;
  cudaStream_t st = S->s_comp;
  const int64_t sv = S->sv, hv = S->hv, qw = S->vqkv_w, ow = S->vo_w, ml = S->vml, h = S->h, es = S->es;
  const int epi_rp = S->tp_rank == 0 ? STP_EPI_BIAS : STP_EPI_STORE;  // row-parallel bias: once, on rank 0
  const int gw = S->vc.grid_w;
  const float theta = S->vc.rope_theta;
  auto patches_of = [&](int mb) {
    return (const uint8_t*)S->patches + ((int64_t)(mb - 1) * sv + (int64_t)S->tp_rank * S->svl) * S->vpd * es;
  };
  switch (u.op) {
    case STP_U_F_EMB:
      if (!S->patches) return fail(STP_ESTATE, "MLLM stage: stp_stage_bind_images not called");
      return gemm_dispatch(dt, STP_GEMM_NT, STP_EPI_STORE, S->svl, hv, S->vpd, patches_of(u.mb), S->vpd,
                           P(S, S->p_patch), S->vpd, sl->x_in, hv, nullptr, nullptr, 0, mc, st);
    case STP_U_F_ATTN: {
      VitSlotLayer& L = sl->V[u.layer];
      const VitIdx& I = S->vidx.at(u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NT, STP_EPI_BIAS, sv, qw, hv, L.xn, hv, P(S, I.wqkv), hv, L.qkv, qw,
                            P(S, I.bqkv), nullptr, 0, mc, st));
      STP_TRY(rope2d(dt, 0, sv, qw, 0, (int)(2 * S->vnh), (int)S->vd, gw, theta, L.qkv, st));
      const uint8_t* q = (const uint8_t*)L.qkv;
      const int64_t hs = S->vnh * S->vd * es;
      STP_TRY(attn_fwd(dt, sv, (int)S->vnh, (int)S->vnh, (int)S->vd, 0, q, q + hs, q + 2 * hs, qw, L.o, ow, L.lse,
                       st));
      return gemm_dispatch(dt, STP_GEMM_NT, epi_rp, sv, hv, ow, L.o, ow, P(S, I.wo), ow, S->pf, hv, P(S, I.bo),
                           nullptr, 0, mc, st);
    }
    case STP_U_F_MLP: {
      VitSlotLayer& L = sl->V[u.layer];
      const VitIdx& I = S->vidx.at(u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NT, STP_EPI_BIAS, sv, ml, hv, L.xn2, hv, P(S, I.w1), hv, L.a, ml, P(S, I.b1),
                            nullptr, 0, mc, st));
      STP_TRY(act_fwd(dt, 0, sv * ml, L.a, L.hh, st));
      return gemm_dispatch(dt, STP_GEMM_NT, epi_rp, sv, hv, ml, L.hh, ml, P(S, I.w2), ml, S->pf, hv, P(S, I.b2),
                           nullptr, 0, mc, st);
    }
    case STP_U_F_MERGE: {
      const int64_t ni = S->n_img;
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NT, STP_EPI_BIAS, ni, S->m4l, S->m4, sl->yq, S->m4, P(S, S->p_mw1), S->m4,
                            sl->z, S->m4l, P(S, S->p_mb1), nullptr, 0, mc, st));
      STP_TRY(act_fwd(dt, 1, ni * S->m4l, sl->z, sl->gz, st));
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NT, epi_rp, ni, h, S->m4l, sl->gz, S->m4l, P(S, S->p_mw2), S->m4l, S->pf, h,
                            P(S, S->p_mb2), nullptr, 0, mc, st));
      const int32_t* tok = S->tokens + (int64_t)(u.mb - 1) * S->s + ni;
      return embed_fwd(dt, S->s - ni, h, tok, vocab0(S), S->Vl, P(S, S->p_embed), (uint8_t*)S->pf + ni * h * es, st);
    }
    case STP_U_B_MERGE: {
      const int64_t ni = S->n_img;
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, ni, S->m4l, h, sl->dylm, h, P(S, S->p_mw2), S->m4l,
                            S->vdtmp_m, S->m4l, nullptr, nullptr, 0, mc, st));
      STP_TRY(act_bwd(dt, 1, ni * S->m4l, S->vdtmp_m, sl->z, sl->z, st));  // dZ over Z
      return gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, ni, S->m4, S->m4l, sl->z, S->m4l, P(S, S->p_mw1), S->m4,
                           S->pb, S->m4, nullptr, nullptr, 0, mc, st);
    }
    case STP_U_W_MERGE: {
      const int64_t ni = S->n_img;
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, h, S->m4l, ni, sl->dylm, h, sl->gz, S->m4l,
                            G(S, S->p_mw2), S->m4l, nullptr, nullptr, 0, mc, st));
      STP_TRY(colsum_acc(dt, ni, h, sl->dylm, h, G(S, S->p_mb2), st));
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, S->m4l, S->m4, ni, sl->z, S->m4l, sl->yq, S->m4,
                            G(S, S->p_mw1), S->m4, nullptr, nullptr, 0, mc, st));
      return colsum_acc(dt, ni, S->m4l, sl->z, S->m4l, G(S, S->p_mb1), st);
    }
    case STP_U_B_MLP: {
      VitSlotLayer& L = sl->V[u.layer];
      const VitIdx& I = S->vidx.at(u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, sv, ml, hv, L.dy_mlp, hv, P(S, I.w2), ml, S->vdtmp_h, ml,
                            nullptr, nullptr, 0, mc, st));
      STP_TRY(act_bwd(dt, 0, sv * ml, S->vdtmp_h, L.a, L.a, st));  // dA over A
      return gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, sv, hv, ml, L.a, ml, P(S, I.w1), hv, S->pb, hv, nullptr,
                           nullptr, 0, mc, st);
    }
    case STP_U_W_MLP: {
      VitSlotLayer& L = sl->V[u.layer];
      const VitIdx& I = S->vidx.at(u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, hv, ml, sv, L.dy_mlp, hv, L.hh, ml, G(S, I.w2), ml,
                            nullptr, nullptr, 0, mc, st));
      STP_TRY(colsum_acc(dt, sv, hv, L.dy_mlp, hv, G(S, I.b2), st));
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, ml, hv, sv, L.a, ml, L.xn2, hv, G(S, I.w1), hv,
                            nullptr, nullptr, 0, mc, st));
      return colsum_acc(dt, sv, ml, L.a, ml, G(S, I.b1), st);
    }
    case STP_U_B_ATTN: {
      VitSlotLayer& L = sl->V[u.layer];
      const VitIdx& I = S->vidx.at(u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, sv, ow, hv, L.dy_attn, hv, P(S, I.wo), ow, S->vdtmp_o, ow,
                            nullptr, nullptr, 0, mc, st));
      const uint8_t* q = (const uint8_t*)L.qkv;
      uint8_t* dq = (uint8_t*)L.dqkv;
      const int64_t hs = S->vnh * S->vd * es;
      STP_TRY(attn_bwd(dt, sv, (int)S->vnh, (int)S->vnh, (int)S->vd, 0, q, q + hs, q + 2 * hs, qw, L.o, ow,
                       S->vdtmp_o, L.lse, dq, dq + hs, dq + 2 * hs, qw, S->vattn_ws, st));
      STP_TRY(rope2d(dt, 1, sv, qw, 0, (int)(2 * S->vnh), (int)S->vd, gw, theta, L.dqkv, st));
      return gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, sv, hv, qw, L.dqkv, qw, P(S, I.wqkv), hv, S->pb, hv,
                           nullptr, nullptr, 0, mc, st);
    }
    case STP_U_W_ATTN: {
      VitSlotLayer& L = sl->V[u.layer];
      const VitIdx& I = S->vidx.at(u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, hv, ow, sv, L.dy_attn, hv, L.o, ow, G(S, I.wo), ow,
                            nullptr, nullptr, 0, mc, st));
      STP_TRY(colsum_acc(dt, sv, hv, L.dy_attn, hv, G(S, I.bo), st));
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, qw, hv, sv, L.dqkv, qw, L.xn, hv, G(S, I.wqkv), hv,
                            nullptr, nullptr, 0, mc, st));
      return colsum_acc(dt, sv, qw, L.dqkv, qw, G(S, I.bqkv), st);
    }
    case STP_U_W_EMB: {
      // text rows: vocab-parallel embedding gradient from the all-gathered
      // LM-input gradient; image rows: patch-embedding weight partial of this
      // rank's shard rows (summed over TP at the end of the step)
      const int64_t ni = S->n_img;
      const int32_t* tok = S->tokens + (int64_t)(u.mb - 1) * S->s + ni;
      STP_TRY(embed_bwd(dt, S->s - ni, h, tok, vocab0(S), S->Vl, (const uint8_t*)sl->dylm + ni * h * es,
                        G(S, S->p_embed), st));
      return gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, hv, S->vpd, S->svl, sl->vdx, hv, patches_of(u.mb),
                           S->vpd, DG(S, S->p_patch), S->vpd, nullptr, nullptr, 0, mc, st);
    }
  }
  return fail(STP_ESTATE, "unknown ViT compute unit");
}

// ViT comm phases (NCCL reduce-scatter / all-gather over the [sv, hv]
// residual stream, LayerNorm in place of RMSNorm):
//   cf 1                after F_EMB: ln1(0) -> AG
//   cf 2 + 2j           after F_ATTN(j): RS + residual -> x1; ln2(j) -> AG
//   cf 3 + 2j           after F_MLP(j): RS + x1 -> xres; ln1(j+1) (or the
//                       merger LayerNorm after the last layer) -> AG
//   cf 2 + 2 nv         after F_MERGE: RS of the [S, h] LM-input partial
//   cb 0                AG of the incoming LM-input gradient shard
//   cb 1                after B_MERGE: RS; merger-LN bwd -> AG
//   cb 2 + 2jj (+1)     after B_MLP / B_ATTN of layer nv-1-jj: RS; ln2 / ln1
//                       bwd + residual gradient -> AG for the next B unit
stp_status vit_ln_ag(stp_stage* S, const void* x, const void* resid, void* x_out, int g, int b, float* mean,
                     float* rstd, void* dst) {
  const int dt = S->dtype;
  void* y = S->t == 1 ? dst : S->vntmp;
  STP_TRY(layernorm_fwd(dt, S->svl, S->hv, x, resid, x_out, P(S, g), P(S, b), S->vc.ln_eps, y, mean, rstd, S->s_comm));
  if (S->t > 1) STP_TRY(all_gather(S, S->vntmp, dst, (size_t)(S->svl * S->hv)));
  return STP_OK;
}

stp_status vit_rs(stp_stage* S, const void* partial, const void** out) {
  if (S->t == 1) {
    *out = partial;
    return STP_OK;
  }
  STP_NCCL_TRY(ncclReduceScatter(partial, S->vrtmp, (size_t)(S->svl * S->hv), (ncclDataType_t)ncdt(S->dtype), ncclSum,
                                 S->tpc, S->s_comm));
  *out = S->vrtmp;
  return STP_OK;
}

stp_status vit_cf(stp_stage* S, const Chunk& C, const stp_unit& u, Slot* sl) {
  const int k = u.layer, nv = C.nl;
  if (k == 1) {
    const VitIdx& I = S->vidx.at(0);
    return vit_ln_ag(S, sl->x_in, nullptr, nullptr, I.ln1_g, I.ln1_b, sl->V[0].mean1, sl->V[0].rstd1, sl->V[0].xn);
  }
  if (k == 2 + 2 * nv) {  // LM-input partial [S, h] -> this rank's shard
    S->pf_pending = true;
    if (S->t == 1) {
      STP_CUDA_TRY(cudaMemcpyAsync(sl->x_out, S->pf, S->sl * S->h * S->es, cudaMemcpyDeviceToDevice, S->s_comm));
      return STP_OK;
    }
    return reduce_scatter(S, S->pf, sl->x_out);
  }
  const int idx = k - 2, j = idx / 2;
  if (j < 0 || j >= nv) return fail(STP_ESTATE, "ViT forward comm phase out of range");
  VitSlotLayer& L = sl->V[j];
  const VitIdx& I = S->vidx.at(j);
  const void* src = nullptr;
  STP_TRY(vit_rs(S, S->pf, &src));
  S->pf_pending = true;
  if (idx % 2 == 0)
    return vit_ln_ag(S, src, j == 0 ? sl->x_in : sl->V[j - 1].xres, L.x1, I.ln2_g, I.ln2_b, L.mean2, L.rstd2, L.xn2);
  if (j + 1 < nv) {
    const VitIdx& I2 = S->vidx.at(j + 1);
    return vit_ln_ag(S, src, L.x1, L.xres, I2.ln1_g, I2.ln1_b, sl->V[j + 1].mean1, sl->V[j + 1].rstd1,
                     sl->V[j + 1].xn);
  }
  return vit_ln_ag(S, src, L.x1, L.xres, S->p_mln_g, S->p_mln_b, sl->meanq, sl->rstdq, sl->yq);
}

stp_status vit_cb(stp_stage* S, const Chunk& C, const stp_unit& u, Slot* sl) {
  const int dt = S->dtype, k = u.layer, nv = C.nl;
  const int64_t vsh = S->svl * S->hv;
  cudaStream_t st = S->s_comm;
  if (k == 0) return all_gather(S, sl->dx_in, sl->dylm, (size_t)(S->sl * S->h));
  const void* src = nullptr;
  STP_TRY(vit_rs(S, S->pb, &src));
  S->pb_pending = true;
  if (k == 1) {  // after B_MERGE: merger LayerNorm backward (no residual) -> AG for B_MLP(nv-1)
    STP_TRY(layernorm_bwd(dt, S->svl, S->hv, src, sl->V[nv - 1].xres, P(S, S->p_mln_g), sl->meanq, sl->rstdq, nullptr,
                          sl->vdx, DG(S, S->p_mln_g), DG(S, S->p_mln_b), st));
    return all_gather(S, sl->vdx, sl->V[nv - 1].dy_mlp, (size_t)vsh);
  }
  const int idx = k - 2, jj = idx / 2, j = nv - 1 - jj;
  if (j < 0 || j >= nv) return fail(STP_ESTATE, "ViT backward comm phase out of range");
  VitSlotLayer& L = sl->V[j];
  const VitIdx& I = S->vidx.at(j);
  if (idx % 2 == 0) {  // after B_MLP(j): ln2 bwd + residual grad -> AG for B_ATTN(j)
    STP_TRY(layernorm_bwd(dt, S->svl, S->hv, src, L.x1, P(S, I.ln2_g), L.mean2, L.rstd2, sl->vdx, sl->vdx,
                          DG(S, I.ln2_g), DG(S, I.ln2_b), st));
    return all_gather(S, sl->vdx, L.dy_attn, (size_t)vsh);
  }
  // after B_ATTN(j): ln1 bwd + residual grad -> AG for B_MLP(j-1); at j = 0
  // vdx is the gradient of the patch embedding output (W_EMB reads it)
  STP_TRY(layernorm_bwd(dt, S->svl, S->hv, src, j == 0 ? sl->x_in : sl->V[j - 1].xres, P(S, I.ln1_g), L.mean1,
                        L.rstd1, sl->vdx, sl->vdx, DG(S, I.ln1_g), DG(S, I.ln1_b), st));
  if (j > 0) return all_gather(S, sl->vdx, sl->V[j - 1].dy_mlp, (size_t)vsh);
  return STP_OK;
}

// ------------------------------------------------------ activation offload
// PAPER.md §4.3: "the saved activations required for the weight
// gradients are offloaded to the CPU in parallel with the computation streams
// and reloaded when necessary"; chunk-0 activations, whose lifespan is long,
// are the target, chunk 1 is never offloaded.  reading R5:
// alpha = the fraction of chunk 0's layers whose MLP activations [gu | hh]
// (60% of a layer's stash) are offloaded, the earliest layers first (their
// backward comes last); D2H right after the layer's F_MLP, H2D for all of a
// microbatch's offloaded layers when its backward lane opens (CB 0), each
// B_MLP waits for its own reload.  Separate copy streams per direction (PCIe
// is full duplex); device memory of the offloaded tensors comes from a pool
// sized by a dry run of the unit list.
bool off_layer(const stp_stage* S, const Chunk& C, int j) { return S->off_n > 0 && C.c == 0 && !C.vit && j < S->off_n; }

stp_status off_acquire(stp_stage* S, cudaStream_t st, int* out) {
  for (size_t i = 0; i < S->off_pool.size(); ++i) {
    OffBlock& b = S->off_pool[i];
    if (b.busy) continue;
    b.busy = true;
    if (b.ev_valid) STP_CUDA_TRY(cudaStreamWaitEvent(st, b.ev, 0));
    *out = (int)i;
    return STP_OK;
  }
  return fail(STP_ESTATE, "offload pool exhausted (pool sizing / schedule mismatch)");
}

stp_status off_release(stp_stage* S, int blk, cudaStream_t st) {
  OffBlock& b = S->off_pool[blk];
  STP_CUDA_TRY(cudaEventRecord(b.ev, st));
  b.ev_valid = true;
  b.busy = false;
  return STP_OK;
}

void off_bind(stp_stage* S, SlotLayer& L, int blk) {
  L.blk = blk;
  L.gu = S->off_pool[blk].dev;
  L.hh = (uint8_t*)L.gu + S->s * 2 * S->fi * S->es;
}

// after F_MLP(j) of an offloaded layer: D2H of [gu | hh], block back to the pool
stp_status off_store(stp_stage* S, Slot* sl, int j, cudaEvent_t fwd_done) {
  SlotLayer& L = sl->L[j];
  STP_CUDA_TRY(cudaStreamWaitEvent(S->s_d2h, fwd_done, 0));
  STP_CUDA_TRY(cudaMemcpyAsync(L.host, L.gu, S->off_bytes, cudaMemcpyDeviceToHost, S->s_d2h));
  STP_CUDA_TRY(cudaEventRecord(L.ev_d2h, S->s_d2h));
  STP_TRY(off_release(S, L.blk, S->s_d2h));
  L.blk = -1;
  L.gu = L.hh = nullptr;
  S->off_d2h_bytes += (int64_t)S->off_bytes;
  return STP_OK;
}

// the backward lane of (chunk 0, mb) opens: reload every offloaded layer, the
// last layer (first needed) first
stp_status off_reload(stp_stage* S, Chunk& C, Slot* sl) {
  for (int j = std::min(S->off_n, C.nl) - 1; j >= 0; --j) {
    SlotLayer& L = sl->L[j];
    int blk = -1;
    STP_TRY(off_acquire(S, S->s_h2d, &blk));
    off_bind(S, L, blk);
    STP_CUDA_TRY(cudaStreamWaitEvent(S->s_h2d, L.ev_d2h, 0));
    STP_CUDA_TRY(cudaMemcpyAsync(L.gu, L.host, S->off_bytes, cudaMemcpyHostToDevice, S->s_h2d));
    STP_CUDA_TRY(cudaEventRecord(L.ev_h2d, S->s_h2d));
    S->off_h2d_bytes += (int64_t)S->off_bytes;
  }
  return STP_OK;
}

// ------------------------------------------------------------ units

// Before a unit's row-parallel GEMM: in push mode, target every TP rank's copy
// of the partial buffer (row block q -> rank q, at this rank's slice).
stp_status push_partial(stp_stage* S, void* partial, bool* pushed) {
  *pushed = false;
  if (!S->p2p_push) return STP_OK;
  void* ptrs[8];
  for (int q = 0; q < S->t; ++q) {
    ptrs[q] = q == S->tp_rank ? partial : sym_peer_ptr(S, q, partial);
    if (!ptrs[q]) return fail(STP_ESTATE, "push target not in the symmetric set");
  }
  gemm_push_targets(ptrs, S->t, S->sl, (int64_t)S->tp_rank * S->sl);
  *pushed = true;
  return STP_OK;
}
stp_status push_done(stp_stage* S, stp_status r) {
  if (S->p2p_push) gemm_push_targets(nullptr, 0, 0, 0);  // never leak targets into a later GEMM
  return r;
}

stp_status vit_compute(stp_stage* S, const stp_unit& u, Slot* sl);
stp_status unit_compute(stp_stage* S, const stp_unit& u) {
  Chunk& C = chunk_of(S, u.chunk);
  const int dt = S->dtype;
  const int64_t s = S->s, h = S->h;
  const int mc = S->gemm_max_ctas;
  cudaStream_t st = S->s_comp;
  Slot* sl = nullptr;
  const bool fwd = u.op == STP_U_F_ATTN || u.op == STP_U_F_MLP || u.op == STP_U_F_EMB || u.op == STP_U_F_HEAD ||
                   u.op == STP_U_F_MERGE;
  if (fwd) {
    STP_TRY(acquire(S, u.chunk, u.mb, &sl));
  } else {
    sl = find_slot(S, u.chunk, u.mb);
    if (!sl) return fail(STP_ESTATE, "backward/W unit without a forward stash");
  }
  const bool writes_pf = u.op == STP_U_F_ATTN || u.op == STP_U_F_MLP || u.op == STP_U_F_EMB || u.op == STP_U_F_MERGE;
  const bool writes_pb = u.op == STP_U_B_ATTN || u.op == STP_U_B_MLP || u.op == STP_U_B_HEAD || u.op == STP_U_B_MERGE;
  if (writes_pf) {
    if (S->ce) S->pfi ^= 1;
    S->pf = S->pfb[S->pfi];
    if (S->pfb_pending[S->pfi]) STP_CUDA_TRY(cudaStreamWaitEvent(st, S->ev_pfb[S->pfi], 0));
  }
  if (writes_pb) {
    if (S->ce) S->pbi ^= 1;
    S->pb = S->pbb[S->pbi];
    if (S->pbb_pending[S->pbi]) STP_CUDA_TRY(cudaStreamWaitEvent(st, S->ev_pbb[S->pbi], 0));
  }
  if (C.vit) return vit_compute(S, u, sl);
  const int j = u.layer - C.l0;
  switch (u.op) {
    case STP_U_F_EMB: {
      S->pf_push = false;
      const int32_t* tok = S->tokens + (int64_t)(u.mb - 1) * s;
      return embed_fwd(dt, s, h, tok, vocab0(S), S->Vl, P(S, S->p_embed), S->pf, st);
    }
    case STP_U_F_ATTN: {
      SlotLayer& L = sl->L[j];
      const LayerIdx& I = LI(S, u.layer);
      const bool bias = I.bqkv >= 0;
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NT, bias ? STP_EPI_BIAS : STP_EPI_STORE, s, S->qkv_w, h, L.xn, h,
                            P(S, I.wqkv), h, L.qkv, S->qkv_w, bias ? P(S, I.bqkv) : nullptr, nullptr, 0, mc, st));
      STP_TRY(rope(dt, 0, s, S->qkv_w, 0, (int)(S->qh + S->kh), (int)S->d, S->mc.rope_theta, 0, L.qkv, st));
      const uint8_t* q = (const uint8_t*)L.qkv;
      STP_TRY(attn_fwd(dt, s, (int)S->qh, (int)S->kh, (int)S->d, 1, q, q + S->qh * S->d * S->es,
                       q + (S->qh + S->kh) * S->d * S->es, S->qkv_w, L.o, S->o_w, L.lse, st));
      STP_TRY(push_partial(S, S->pf, &S->pf_push));
      return push_done(S, gemm_dispatch(dt, STP_GEMM_NT, STP_EPI_STORE, s, h, S->o_w, L.o, S->o_w, P(S, I.wo), S->o_w, S->pf, h,
                           nullptr, nullptr, 0, mc, st));
    }
    case STP_U_F_MLP: {
      SlotLayer& L = sl->L[j];
      const LayerIdx& I = LI(S, u.layer);
      if (off_layer(S, C, j)) {
        int blk = -1;
        STP_TRY(off_acquire(S, st, &blk));
        off_bind(S, L, blk);
      }
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NT, STP_EPI_STORE, s, 2 * S->fi, h, L.xn2, h, P(S, I.wgu), h, L.gu,
                            2 * S->fi, nullptr, nullptr, 0, mc, st));
      STP_TRY(swiglu_fwd(dt, s, S->fi, L.gu, L.hh, st));
      STP_TRY(push_partial(S, S->pf, &S->pf_push));
      return push_done(S, gemm_dispatch(dt, STP_GEMM_NT, STP_EPI_STORE, s, h, S->fi, L.hh, S->fi, P(S, I.wd), S->fi, S->pf, h,
                           nullptr, nullptr, 0, mc, st));
    }
    case STP_U_F_HEAD: {
      // LM head + local CE statistics from the fp32 accumulators (GEMM epilogue)
      const int32_t* tgt = S->targets + (int64_t)(u.mb - 1) * s;
      return lm_head_ce(dt, s, S->Vl, h, sl->xf, P(S, S->p_lm), sl->logits, tgt, vocab0(S), S->ce_ws, sl->stats, mc,
                        st);
    }
    case STP_U_B_HEAD: {
      const float scale = 1.f / ((float)s * (float)S->m);
      const int32_t* tgt = S->targets + (int64_t)(u.mb - 1) * s;
      STP_TRY(ce_combine(s, S->t, sl->stats_all, sl->lse_ce, S->loss_acc, scale, st));
      STP_TRY(ce_grad(dt, s, S->Vl, sl->logits, S->Vl, tgt, vocab0(S), sl->lse_ce, scale, st));
      STP_TRY(push_partial(S, S->pb, &S->pb_push));
      return push_done(S, gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, s, h, S->Vl, sl->logits, S->Vl, P(S, S->p_lm), h, S->pb,
                           h, nullptr, nullptr, 0, mc, st));
    }
    case STP_U_W_HEAD:
      return gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, S->Vl, h, s, sl->logits, S->Vl, sl->xf, h,
                           G(S, S->p_lm), h, nullptr, nullptr, 0, mc, st);
    case STP_U_B_MLP: {
      SlotLayer& L = sl->L[j];
      const LayerIdx& I = LI(S, u.layer);
      // (STP_EPI_SWIGLU_BWD would fuse the SwiGLU backward into this GEMM's
      // epilogue; measured slower: the epilogue's [G | U] reads stall the 2-SM
      // kernel, GEMM average 1321 -> 1187 TFLOP/s in round 1; re-measured after
      // the epilogue stopped spilling: GEMM 1576 -> 1688 ms per N = 1 step for
      // the ~40 ms the separate kernel costs, profiles/r02x_*.  Kept separate.)
      if (off_layer(S, C, j)) {
        if (L.blk < 0) return fail(STP_ESTATE, "offloaded layer not reloaded before its backward");
        STP_CUDA_TRY(cudaStreamWaitEvent(st, L.ev_h2d, 0));
      }
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, s, S->fi, h, L.dy_mlp, h, P(S, I.wd), S->fi, S->dtmp_h,
                            S->fi, nullptr, nullptr, 0, mc, st));
      STP_TRY(swiglu_bwd(dt, s, S->fi, S->dtmp_h, L.gu, L.gu, st));  // dGU overwrites GU
      STP_TRY(push_partial(S, S->pb, &S->pb_push));
      return push_done(S, gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, s, h, 2 * S->fi, L.gu, 2 * S->fi, P(S, I.wgu), h, S->pb,
                           h, nullptr, nullptr, 0, mc, st));
    }
    case STP_U_W_MLP: {
      SlotLayer& L = sl->L[j];
      const LayerIdx& I = LI(S, u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, h, S->fi, s, L.dy_mlp, h, L.hh, S->fi, G(S, I.wd),
                            S->fi, nullptr, nullptr, 0, mc, st));
      return gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, 2 * S->fi, h, s, L.gu, 2 * S->fi, L.xn2, h,
                           G(S, I.wgu), h, nullptr, nullptr, 0, mc, st);
    }
    case STP_U_B_ATTN: {
      SlotLayer& L = sl->L[j];
      const LayerIdx& I = LI(S, u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, s, S->o_w, h, L.dy_attn, h, P(S, I.wo), S->o_w,
                            S->dtmp_o, S->o_w, nullptr, nullptr, 0, mc, st));
      const uint8_t* q = (const uint8_t*)L.qkv;
      uint8_t* dq = (uint8_t*)L.dqkv;
      const int64_t ko = S->qh * S->d * S->es, vo = (S->qh + S->kh) * S->d * S->es;
      STP_TRY(attn_bwd(dt, s, (int)S->qh, (int)S->kh, (int)S->d, 1, q, q + ko, q + vo, S->qkv_w, L.o, S->o_w,
                       S->dtmp_o, L.lse, dq, dq + ko, dq + vo, S->qkv_w, S->attn_ws, st));
      STP_TRY(rope(dt, 1, s, S->qkv_w, 0, (int)(S->qh + S->kh), (int)S->d, S->mc.rope_theta, 0, L.dqkv, st));
      STP_TRY(push_partial(S, S->pb, &S->pb_push));
      return push_done(S, gemm_dispatch(dt, STP_GEMM_NN, STP_EPI_STORE, s, h, S->qkv_w, L.dqkv, S->qkv_w, P(S, I.wqkv), h, S->pb,
                           h, nullptr, nullptr, 0, mc, st));
    }
    case STP_U_W_ATTN: {
      SlotLayer& L = sl->L[j];
      const LayerIdx& I = LI(S, u.layer);
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, h, S->o_w, s, L.dy_attn, h, L.o, S->o_w, G(S, I.wo),
                            S->o_w, nullptr, nullptr, 0, mc, st));
      STP_TRY(gemm_dispatch(dt, STP_GEMM_TN, STP_EPI_ACCUM_F32, S->qkv_w, h, s, L.dqkv, S->qkv_w, L.xn, h,
                            G(S, I.wqkv), h, nullptr, nullptr, 0, mc, st));
      if (I.bqkv >= 0) STP_TRY(colsum_acc(dt, s, S->qkv_w, L.dqkv, S->qkv_w, G(S, I.bqkv), st));
      return STP_OK;
    }
    case STP_U_W_EMB: {
      const int32_t* tok = S->tokens + (int64_t)(u.mb - 1) * s;
      return embed_bwd(dt, s, h, tok, vocab0(S), S->Vl, sl->dx0, G(S, S->p_embed), st);
    }
  }
  return fail(STP_ESTATE, "unknown compute unit");
}

// Forward comm phase k of pass (chunk, mb): see DESIGN.md "Comm phases".
stp_status unit_cf(stp_stage* S, const stp_unit& u) {
  Chunk& C = chunk_of(S, u.chunk);
  Slot* sl = nullptr;
  STP_TRY(acquire(S, u.chunk, u.mb, &sl));
  if (C.vit) {
    S->open_phase = 0;
    return vit_cf(S, C, u, sl);
  }
  const int dt = S->dtype;
  const int64_t h = S->h, shard = S->sl * S->h;
  const float eps = S->mc.rms_eps;
  cudaStream_t st = S->s_comm;
  const int k = u.layer;
  S->open_phase = 0;
  // normalise `x` (shard) with gamma into the all-gathered destination `dst`
  auto norm_ag = [&](const void* x, const void* resid, void* x_out, const void* g, float* rstd, void* dst) {
    if (S->p2p && !resid) return p2p_ag(S, x, g, rstd, dst);
    if (S->ce) {
      STP_TRY(rmsnorm_fwd(dt, S->sl, h, x, resid, x_out, g, eps, (uint8_t*)dst + S->tp_rank * shard * S->es, rstd,
                          st));
      return ce_ag(S, dst);
    }
    void* y = (S->t == 1) ? dst : S->ntmp;
    STP_TRY(rmsnorm_fwd(dt, S->sl, h, x, resid, x_out, g, eps, y, rstd, st));
    if (S->t > 1) STP_TRY(all_gather(S, S->ntmp, dst, (size_t)shard));
    return STP_OK;
  };
  auto rs_src = [&](const void** out) {
    if (S->t == 1) {
      *out = S->pf;
      return STP_OK;
    }
    STP_TRY(reduce_scatter(S, S->pf, S->rtmp));
    *out = S->rtmp;
    return STP_OK;
  };
  if (k == 0) {
    // input phase: chunk input shard (PP recv or local handoff) -> ln1 -> AG
    if (dev_of_vs(S, C.vs - 1) == S->pp_rank) {
      // local handoff from the other chunk on this device (V-shape turn)
      for (auto& O : S->chunks)
        if (O.vs == C.vs - 1) {
          Slot* src = find_slot(S, O.c, u.mb);
          if (!src) return fail(STP_ESTATE, "handoff source stash missing");
          STP_CUDA_TRY(cudaMemcpyAsync(sl->x_in, O.vit ? src->x_out : src->L[O.nl - 1].xres, shard * S->es,
                                       cudaMemcpyDeviceToDevice, st));
        }
    }
    const LayerIdx& I = LI(S, C.l0);
    return norm_ag(sl->x_in, nullptr, nullptr, P(S, I.ln1), sl->L[0].rstd1, sl->L[0].xn);
  }
  // heavy unit k (1-based) of the forward lane
  int idx = k - 1;
  if (C.first) {
    if (idx == 0) {  // after F_EMB: RS -> chunk input shard -> ln1 -> AG
      if (S->ce) {
        S->pf_pending = true;
        return ce_rs(S, S->pf, nullptr, sl->x_in, P(S, LI(S, C.l0).ln1), sl->L[0].rstd1, sl->L[0].xn);
      }
      if (S->t == 1) STP_CUDA_TRY(cudaMemcpyAsync(sl->x_in, S->pf, shard * S->es, cudaMemcpyDeviceToDevice, st));
      else STP_TRY(reduce_scatter(S, S->pf, sl->x_in));
      S->pf_pending = true;
      const LayerIdx& I = LI(S, C.l0);
      return norm_ag(sl->x_in, nullptr, nullptr, P(S, I.ln1), sl->L[0].rstd1, sl->L[0].xn);
    }
    idx -= 1;
  }
  if (idx < 2 * C.nl) {
    const int j = idx / 2;
    SlotLayer& L = sl->L[j];
    const LayerIdx& I = LI(S, C.l0 + j);
    if (S->ce) {  // fused RS + residual + RMSNorm, then AG (copy engines)
      S->pf_pending = true;
      if (idx % 2 == 0)
        return ce_rs(S, S->pf, j == 0 ? sl->x_in : sl->L[j - 1].xres, L.x1, P(S, I.ln2), L.rstd2, L.xn2);
      if (j + 1 < C.nl)
        return ce_rs(S, S->pf, L.x1, L.xres, P(S, LI(S, C.l0 + j + 1).ln1), sl->L[j + 1].rstd1, sl->L[j + 1].xn);
      if (C.last) return ce_rs(S, S->pf, L.x1, L.xres, P(S, S->p_final), sl->rstdf, sl->xf);
      return ce_rs(S, S->pf, L.x1, L.xres, nullptr, nullptr, nullptr);
    }
    const void* src = nullptr;
    STP_TRY(rs_src(&src));
    S->pf_pending = true;
    if (idx % 2 == 0) {  // after attention: x1 = RS + x; ln2 -> AG
      const void* xprev = j == 0 ? sl->x_in : sl->L[j - 1].xres;
      return norm_ag(src, xprev, L.x1, P(S, I.ln2), L.rstd2, L.xn2);
    }
    // after MLP: x2 = RS + x1; next layer's ln1 (or final norm) -> AG
    if (j + 1 < C.nl) {
      const LayerIdx& I2 = LI(S, C.l0 + j + 1);
      return norm_ag(src, L.x1, L.xres, P(S, I2.ln1), sl->L[j + 1].rstd1, sl->L[j + 1].xn);
    }
    if (C.last) return norm_ag(src, L.x1, L.xres, P(S, S->p_final), sl->rstdf, sl->xf);
    return add(dt, shard, src, L.x1, L.xres, st);
  }
  // after F_HEAD: all-gather the cross-entropy row statistics
  if (S->t == 1) {
    STP_CUDA_TRY(cudaMemcpyAsync(sl->stats_all, sl->stats, S->s * 3 * 4, cudaMemcpyDeviceToDevice, st));
    return STP_OK;
  }
  STP_NCCL_TRY(ncclAllGather(sl->stats, sl->stats_all, (size_t)(S->s * 3), ncclFloat32, S->tpc, st));
  return STP_OK;
}

stp_status cb_handoff(stp_stage* S, Chunk& C, const stp_unit& u, Slot* sl);
stp_status unit_cb(stp_stage* S, const stp_unit& u) {
  Chunk& C = chunk_of(S, u.chunk);
  Slot* sl = find_slot(S, u.chunk, u.mb);
  if (!sl) return fail(STP_ESTATE, "backward comm without stash");
  if (C.vit) {
    S->open_phase = 0;
    return vit_cb(S, C, u, sl);
  }
  const int dt = S->dtype;
  const int64_t h = S->h, shard = S->sl * S->h;
  cudaStream_t st = S->s_comm;
  const int k = u.layer;
  S->open_phase = 0;
  auto rs_src = [&](const void** out) {
    if (S->t == 1) {
      *out = S->pb;
      return STP_OK;
    }
    if (S->ce) {  // RS (copy engines) + sum into rtmp; the AG below reuses the phase
      STP_TRY(ce_rs(S, S->pb, nullptr, S->rtmp, nullptr, nullptr, nullptr));
      *out = S->rtmp;
      return STP_OK;
    }
    STP_TRY(reduce_scatter(S, S->pb, S->rtmp));
    *out = S->rtmp;
    return STP_OK;
  };
  if (k == 0) {  // incoming gradient shard -> AG for the last layer's MLP B unit
    return ag_dx(S, sl->dx_in, sl->L[C.nl - 1].dy_mlp, (size_t)shard);
  }
  int idx = k - 1;
  if (S->ce) {  // fused RS + RMSNorm-bwd + residual grad (+ AG) per phase: p2p kernel or copy-engine pulls
    S->pb_pending = true;
    if (C.last && idx == 0)
      return fused_bwd(S, sl->L[C.nl - 1].xres, P(S, S->p_final), sl->rstdf, nullptr, sl->dx_in, DG(S, S->p_final),
                     sl->L[C.nl - 1].dy_mlp);
    const int id2 = C.last ? idx - 1 : idx;
    const int j = C.nl - 1 - id2 / 2;
    SlotLayer& L = sl->L[j];
    const LayerIdx& I = LI(S, C.l0 + j);
    if (id2 % 2 == 0) return fused_bwd(S, L.x1, P(S, I.ln2), L.rstd2, sl->dx_in, sl->dx_in, DG(S, I.ln2), L.dy_attn);
    const void* xprev = j == 0 ? sl->x_in : sl->L[j - 1].xres;
    void* dst = j > 0 ? sl->L[j - 1].dy_mlp : (C.first ? sl->dx0 : nullptr);
    STP_TRY(fused_bwd(S, xprev, P(S, I.ln1), L.rstd1, sl->dx_in, sl->dx_in, DG(S, I.ln1), dst));
    if (j > 0 || C.first) return STP_OK;
    return cb_handoff(S, C, u, sl);
  }
  if (C.last) {
    if (idx == 0) {  // after B_HEAD: RS -> final-norm bwd -> residual grad -> AG
      const void* src = nullptr;
      STP_TRY(rs_src(&src));
      S->pb_pending = true;
      STP_TRY(rmsnorm_bwd(dt, S->sl, h, src, sl->L[C.nl - 1].xres, P(S, S->p_final), sl->rstdf, nullptr, sl->dx_in,
                          DG(S, S->p_final), st));
      return ag_dx(S, sl->dx_in, sl->L[C.nl - 1].dy_mlp, (size_t)shard);
    }
    idx -= 1;
  }
  // backward heavy order: MLP(L-1), ATTN(L-1), ..., MLP(0), ATTN(0)
  const int jj = idx / 2;
  const int j = C.nl - 1 - jj;
  SlotLayer& L = sl->L[j];
  const LayerIdx& I = LI(S, C.l0 + j);
  const void* src = nullptr;
  STP_TRY(rs_src(&src));
  S->pb_pending = true;
  if (idx % 2 == 0) {  // after B_MLP: ln2 bwd + residual grad -> AG for B_ATTN
    STP_TRY(rmsnorm_bwd(dt, S->sl, h, src, L.x1, P(S, I.ln2), L.rstd2, sl->dx_in, sl->dx_in, DG(S, I.ln2), st));
    return ag_dx(S, sl->dx_in, L.dy_attn, (size_t)shard);
  }
  // after B_ATTN: ln1 bwd + residual grad
  const void* xprev = j == 0 ? sl->x_in : sl->L[j - 1].xres;
  STP_TRY(rmsnorm_bwd(dt, S->sl, h, src, xprev, P(S, I.ln1), L.rstd1, sl->dx_in, sl->dx_in, DG(S, I.ln1), st));
  if (j > 0) return ag_dx(S, sl->dx_in, sl->L[j - 1].dy_mlp, (size_t)shard);
  if (C.first) return ag_dx(S, sl->dx_in, sl->dx0, (size_t)shard);
  return cb_handoff(S, C, u, sl);
}

// End of a chunk's backward on a non-first chunk: at the V-shape turn hand
// the gradient shard to the other chunk on this device now.
stp_status cb_handoff(stp_stage* S, Chunk& C, const stp_unit& u, Slot* sl) {
  const int64_t shard = S->sl * S->h;
  cudaStream_t st = S->s_comm;
  if (dev_of_vs(S, C.vs - 1) == S->pp_rank) {  // V-shape turn: hand the grad to the other chunk now
    for (auto& O : S->chunks)
      if (O.vs == C.vs - 1) {
        Slot* dst = find_slot(S, O.c, u.mb);
        if (!dst) return fail(STP_ESTATE, "handoff destination stash missing");
        STP_CUDA_TRY(cudaMemcpyAsync(dst->dx_in, sl->dx_in, shard * S->es, cudaMemcpyDeviceToDevice, st));
      }
  }
  return STP_OK;
}

stp_status unit_pp(stp_stage* S, int ui, const stp_unit& u, cudaStream_t st) {
  Chunk& C = chunk_of(S, u.chunk);
  const size_t count = (size_t)(S->sl * S->h);
  const bool fwd = S->unit_fwd[ui] != 0;
  const auto edge = S->unit_edge[ui];
  Slot* sl = nullptr;
  if (u.op == STP_U_PP_RECV) {
    // a forward recv opens the pass's stash slot; a backward recv fills it
    if (fwd) STP_TRY(acquire(S, u.chunk, u.mb, &sl));
    else sl = find_slot(S, u.chunk, u.mb);
    if (!sl) return fail(STP_ESTATE, "recv without stash");
    STP_NCCL_TRY(ncclRecv(fwd ? sl->x_in : sl->dx_in, count, (ncclDataType_t)ncdt(S->dtype), 0, S->c_recv.at(edge),
                          st));
    return STP_OK;
  }
  sl = find_slot(S, u.chunk, u.mb);
  if (!sl) return fail(STP_ESTATE, "send without stash");
  const void* src = fwd ? (C.vit ? sl->x_out : sl->L[C.nl - 1].xres) : sl->dx_in;
  STP_NCCL_TRY(ncclSend(src, count, (ncclDataType_t)ncdt(S->dtype), 1, S->c_send.at(edge), st));
  cudaEvent_t e = pool_event(S);
  STP_CUDA_TRY(cudaEventRecord(e, st));
  sl->free_events.push_back(e);
  return STP_OK;
}

cudaStream_t stream_of(stp_stage* S, int ui, const stp_unit& u) {
  if (u.stream == 0) return S->s_comp;
  if (u.stream == 1) return S->s_comm;
  return u.op == STP_U_PP_SEND ? S->s_send.at(S->unit_edge[ui]) : S->s_recv.at(S->unit_edge[ui]);
}

// PP edge of every PP unit: sends follow their lane's last comm phase (CF =
// forward); a recv is forward iff a CF unit depends on it.
void classify_pp_units(const Schedule& sched, int p, int d, const std::vector<stp_unit>& us,
                       std::vector<std::pair<int, int>>& edge, std::vector<char>& fwd) {
  const int kind = sched.kind;
  edge.assign(us.size(), {-1, -1});
  fwd.assign(us.size(), 0);
  std::vector<char> recv_fwd(us.size(), 0);
  for (size_t i = 0; i < us.size(); ++i)
    if (us[i].op == STP_U_CF && us[i].dep0 >= 0 && us[us[i].dep0].op == STP_U_PP_RECV) recv_fwd[us[i].dep0] = 1;
  for (size_t i = 0; i < us.size(); ++i) {
    const stp_unit& u = us[i];
    const int vs = sched_vstage(kind, p, d, u.chunk);
    if (u.op == STP_U_PP_SEND) {
      const bool f = us[u.dep0].op == STP_U_CF;
      fwd[i] = f;
      edge[i] = {vs, f ? vs + 1 : vs - 1};
    } else if (u.op == STP_U_PP_RECV) {
      const bool f = recv_fwd[i] != 0;
      fwd[i] = f;
      edge[i] = {f ? vs - 1 : vs + 1, vs};
    }
  }
}

bool is_last_w(stp_stage* S, const stp_unit& u) {
  const Chunk& C = S->chunks[u.chunk];
  if (C.first) return u.op == STP_U_W_EMB;
  return u.op == STP_U_W_ATTN && u.layer == C.l0;
}

void reset_step_state(stp_stage* S) {
  S->ev_pool_next = 0;
  S->trace.clear();
  S->pf_pending = S->pb_pending = false;
  S->pfi = S->pbi = 0;
  S->pf = S->pfb[0];
  S->pb = S->pbb[0];
  for (int i = 0; i < 2; ++i) S->pfb_pending[i] = S->pbb_pending[i] = false;
  S->off_reloaded.clear();
  S->off_d2h_bytes = S->off_h2d_bytes = 0;
  for (auto& C : S->chunks) {
    C.mb2slot.clear();
    for (auto& sl : C.slots) {
      sl.busy = false;
      sl.mb = -1;
      sl.free_events.clear();  // the previous step has completed (run_step synchronises)
    }
  }
  for (auto& b : S->off_pool) b.ev_valid = false;
}

// Enqueue one whole step on the stage's streams (everything joins back into
// s_comp at the end), eagerly or inside a CUDA-graph capture of s_comp.
stp_status enqueue_step(stp_stage* S) {
  // start: everything after whatever the caller enqueued before
  STP_CUDA_TRY(cudaEventRecord(S->ev_base, S->s_comp));
  STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comm, S->ev_base, 0));
  for (auto& kv : S->s_send) STP_CUDA_TRY(cudaStreamWaitEvent(kv.second, S->ev_base, 0));
  for (auto& kv : S->s_recv) STP_CUDA_TRY(cudaStreamWaitEvent(kv.second, S->ev_base, 0));
  STP_CUDA_TRY(cudaMemsetAsync(S->loss_acc, 0, sizeof(float), S->s_comp));
  STP_CUDA_TRY(cudaMemsetAsync(S->dgamma, 0, S->dgamma_n * sizeof(float), S->s_comp));
  STP_CUDA_TRY(cudaEventRecord(S->ev_base, S->s_comp));
  STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comm, S->ev_base, 0));
  const int n = (int)S->units.size();
  struct Pending {
    int c, mb;
    cudaEvent_t ev;
  };
  std::vector<Pending> pending;
  for (int i = 0; i < n; ++i) {
    const stp_unit& u = S->units[i];
    cudaStream_t st = stream_of(S, i, u);
    if (u.dep0 >= 0) STP_CUDA_TRY(cudaStreamWaitEvent(st, S->ev_done[u.dep0], 0));
    if (u.dep1 >= 0) STP_CUDA_TRY(cudaStreamWaitEvent(st, S->ev_done[u.dep1], 0));
    if (S->off_n > 0 && u.op == STP_U_CB && u.layer == 0 && u.chunk == 0 && !S->chunks[0].vit) {
      auto key = std::make_pair(u.chunk, u.mb);
      if (!S->off_reloaded[key]) {
        Slot* osl = find_slot(S, u.chunk, u.mb);
        if (!osl) return fail(STP_ESTATE, "reload without stash");
        STP_TRY(off_reload(S, S->chunks[0], osl));
        S->off_reloaded[key] = true;
      }
    }
    if (S->timing) STP_CUDA_TRY(cudaEventRecord(S->ev_t0[i], st));
    stp_status r = STP_OK;
    switch (u.op) {
      case STP_U_CF: r = unit_cf(S, u); break;
      case STP_U_CB: r = unit_cb(S, u); break;
      case STP_U_PP_SEND:
      case STP_U_PP_RECV: r = unit_pp(S, i, u, st); break;
      default: r = unit_compute(S, u); break;
    }
    if (r != STP_OK) {
      if (r == STP_ECUDA || r == STP_ENCCL) S->poisoned = true;
      return r;
    }
    STP_CUDA_TRY(cudaEventRecord(S->ev_done[i], st));
    if (S->off_n > 0 && u.chunk == 0 && (u.op == STP_U_F_MLP || u.op == STP_U_W_MLP)) {
      Chunk& C0 = S->chunks[0];
      const int j = u.layer - C0.l0;
      if (off_layer(S, C0, j)) {
        Slot* osl = find_slot(S, u.chunk, u.mb);
        if (!osl) return fail(STP_ESTATE, "offload without stash");
        if (u.op == STP_U_F_MLP) {
          STP_TRY(off_store(S, osl, j, S->ev_done[i]));
          S->off_reloaded[{u.chunk, u.mb}] = false;
        } else {
          STP_TRY(off_release(S, osl->L[j].blk, st));
          osl->L[j].blk = -1;
          osl->L[j].gu = osl->L[j].hh = nullptr;
        }
      }
    }
    if (S->debug) {  // STP_DEBUG=1: log every unit and run it to completion
      fprintf(stderr, "[stp pp%d tp%d] unit %d/%d a%d s%d op%d l%d c%d mb%d dep%d\n", S->pp_rank, S->tp_rank, i, n,
              u.action, u.stream, u.op, u.layer, u.chunk, u.mb, u.dep0);
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return fail(STP_ECUDA, std::string("debug sync: ") + cudaGetErrorString(e));
    }
    if (S->timing) STP_CUDA_TRY(cudaEventRecord(S->ev_t1[i], st));
    // comm phases consuming the partial buffers release them for the next writer
    if (u.op == STP_U_CF && S->pf_pending) {
      STP_CUDA_TRY(cudaEventRecord(S->ev_pfb[S->pfi], st));
      S->pfb_pending[S->pfi] = true;
      S->pf_pending = false;
    }
    if (u.op == STP_U_CB && S->pb_pending) {
      STP_CUDA_TRY(cudaEventRecord(S->ev_pbb[S->pbi], st));
      S->pbb_pending[S->pbi] = true;
      S->pb_pending = false;
    }
    // a slot is released once its last W unit is enqueued, but only at the
    // end of that action: the action's backward PP send (emitted after the W
    // units of a full backward) still reads the slot and adds its event.
    if (is_last_w(S, u)) pending.push_back({u.chunk, u.mb, S->ev_done[i]});
    if (!pending.empty() && (i + 1 == n || S->units[i + 1].action != u.action)) {
      for (auto& pr : pending) release(S, pr.c, pr.mb, pr.ev);
      pending.clear();
    }
    S->trace.push_back(u);
  }
  // end of step: TP all-reduce of the replicated gamma gradients, add to grads
  STP_CUDA_TRY(cudaEventRecord(S->ev_end, S->s_comp));
  STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comm, S->ev_end, 0));
  if (S->t > 1)
    STP_NCCL_TRY(ncclAllReduce(S->dgamma, S->dgamma, (size_t)S->dgamma_n, ncclFloat32, ncclSum, S->tpc, S->s_comm));
  for (auto& kv : S->dgamma_off) {
    const int pi = kv.first;
    STP_TRY(add(STP_DTYPE_F32, S->params[pi].numel(), S->params[pi].g, S->dgamma + kv.second, S->params[pi].g,
                S->s_comm));
  }
  for (auto& kv : S->s_send) {
    STP_CUDA_TRY(cudaEventRecord(S->ev_end, kv.second));
    STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comm, S->ev_end, 0));
  }
  for (cudaStream_t cs : {S->s_d2h, S->s_h2d}) {
    if (!cs) continue;
    STP_CUDA_TRY(cudaEventRecord(S->ev_end, cs));
    STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comm, S->ev_end, 0));
  }
  for (auto& kv : S->s_recv) {
    STP_CUDA_TRY(cudaEventRecord(S->ev_end, kv.second));
    STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comm, S->ev_end, 0));
  }
  STP_CUDA_TRY(cudaEventRecord(S->ev_end, S->s_comm));
  STP_CUDA_TRY(cudaMemcpyAsync(S->h_loss_pin, S->loss_acc, sizeof(float), cudaMemcpyDeviceToHost, S->s_comm));
  STP_CUDA_TRY(cudaEventRecord(S->ev_join, S->s_comm));
  STP_CUDA_TRY(cudaStreamWaitEvent(S->s_comp, S->ev_join, 0));
  return STP_OK;
}

// One step: eager enqueue, or (STP_GRAPH=1, not in timing / debug mode) the
// step captured once as a CUDA graph over all of the stage's streams and
// replayed while the device inputs (tokens, targets, patches) stay the same.
stp_status run_step(stp_stage* S, float* h_loss, stp_step_stats* stats) {
  if (S->poisoned) return fail(STP_ESTATE, "stage poisoned by an earlier CUDA/NCCL error");
  if (!S->bound) return fail(STP_ESTATE, "stp_bind_params not called");
  STP_CUDA_TRY(cudaSetDevice(S->dev));
  const int64_t launches0 = g_kernel_launches;
  const int n = (int)S->units.size();
  const bool graph = S->use_graph && !S->timing && !S->debug;
  const std::array<const void*, 3> key{S->tokens, S->targets, S->patches};
  // events recorded inside a graph carry no timestamps: a graph step is timed
  // by an event pair around the launch on s_comp (where the graph starts and joins)
  bool timed_launch = false;
  S->ev_last = S->ev_end;
  if (graph && S->graph_exec && S->graph_key == key) {
    STP_CUDA_TRY(cudaEventRecord(S->ev_gstart, S->s_comp));
    STP_CUDA_TRY(cudaGraphLaunch(S->graph_exec, S->s_comp));
    STP_CUDA_TRY(cudaEventRecord(S->ev_gend, S->s_comp));
    timed_launch = true;
    S->ev_last = S->ev_gend;
    g_kernel_launches += S->graph_launches;
  } else if (graph && S->steps_done > 0) {  // first step eager: lazily created tables / counters exist
    if (S->graph_exec) {
      cudaGraphExecDestroy(S->graph_exec);
      S->graph_exec = nullptr;
    }
    reset_step_state(S);
    STP_CUDA_TRY(cudaStreamBeginCapture(S->s_comp, cudaStreamCaptureModeRelaxed));
    const stp_status r = enqueue_step(S);
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(S->s_comp, &g);
    if (r != STP_OK || ec != cudaSuccess || !g) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      return r != STP_OK ? r : fail(STP_ECUDA, std::string("step capture: ") + cudaGetErrorString(ec));
    }
    const cudaError_t ei = cudaGraphInstantiate(&S->graph_exec, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) return fail(STP_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
    S->graph_key = key;
    S->graph_launches = g_kernel_launches - launches0;
    STP_CUDA_TRY(cudaEventRecord(S->ev_gstart, S->s_comp));
    STP_CUDA_TRY(cudaGraphLaunch(S->graph_exec, S->s_comp));
    STP_CUDA_TRY(cudaEventRecord(S->ev_gend, S->s_comp));
    timed_launch = true;
    S->ev_last = S->ev_gend;
  } else {
    reset_step_state(S);
    STP_TRY(enqueue_step(S));
  }
  ++S->steps_done;
  cudaError_t e = cudaStreamSynchronize(S->s_comp);
  if (e != cudaSuccess) {
    S->poisoned = true;
    return fail(STP_ECUDA, std::string("step failed: ") + cudaGetErrorString(e));
  }
  STP_CUDA_TRY(cudaDeviceSynchronize());
  const bool holds_loss = S->chunks.back().last || S->chunks.front().last;
  if (h_loss) *h_loss = holds_loss ? *S->h_loss_pin : 0.f;
  S->launches_step = g_kernel_launches - launches0;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    float ms = 0.f;
    if (timed_launch) STP_CUDA_TRY(cudaEventElapsedTime(&ms, S->ev_gstart, S->ev_gend));
    else STP_CUDA_TRY(cudaEventElapsedTime(&ms, S->ev_base, S->ev_end));
    stats->step_ms = ms;
    stats->n_units = n;
    stats->n_kernels = (int32_t)S->launches_step;
    stats->peak_act_bytes = S->peak_bytes;
    if (S->timing) {
      S->t_start.assign(n, 0.f);
      S->t_end.assign(n, 0.f);
      for (int i = 0; i < n; ++i) {
        STP_CUDA_TRY(cudaEventElapsedTime(&S->t_start[i], S->ev_base, S->ev_t0[i]));
        STP_CUDA_TRY(cudaEventElapsedTime(&S->t_end[i], S->ev_base, S->ev_t1[i]));
      }
      // compute-stream idle gaps: waiting on a TP comm phase (exposed TP) or
      // on PP data / an empty pipeline (PP bubble)
      double busy = 0, exposed = 0, bubble = 0;
      float prev_end = 0.f;
      bool first = true;
      for (int i = 0; i < n; ++i) {
        const stp_unit& u = S->units[i];
        if (u.stream != 0) continue;
        busy += S->t_end[i] - S->t_start[i];
        const float gap = first ? S->t_start[i] : S->t_start[i] - prev_end;
        if (gap > 0) {
          bool tp = false;
          if (u.dep0 >= 0 && S->units[u.dep0].stream == 1) {
            const stp_unit& c = S->units[u.dep0];
            const bool waits_pp = c.dep0 >= 0 && S->units[c.dep0].stream == 2 && S->t_end[c.dep0] > prev_end;
            tp = !waits_pp && S->t_end[u.dep0] > prev_end;
          }
          if (tp) exposed += gap;
          else bubble += gap;
        }
        prev_end = std::max(prev_end, S->t_end[i]);
        first = false;
      }
      bubble += std::max(0.0, (double)ms - (double)prev_end);
      stats->compute_busy_ms = busy;
      stats->exposed_tp_ms = exposed;
      stats->pp_bubble_ms = bubble;
    }
  }
  return STP_OK;
}

// ---------------------------------------------------------------- init
stp_status build_params(stp_stage* S) {
  S->params.clear();
  auto add_p = [&](const std::string& name, int64_t d0, int64_t d1) {
    Param p;
    p.name = name;
    p.d0 = d0;
    p.d1 = d1;
    S->params.push_back(p);
    return (int)S->params.size() - 1;
  };
  for (auto& C : S->chunks) {
    if (C.vit) {  // oracle/vit.py names; column-parallel qkv / w1 / merger w1, row-parallel wo / w2 / merger w2
      S->p_patch = add_p("vit.patch", S->hv, S->vpd);
      for (int l = C.l0; l < C.l0 + C.nl; ++l) {
        const std::string pre = "vit." + std::to_string(l) + ".";
        VitIdx I;
        I.ln1_g = add_p(pre + "ln1_g", S->hv, 1);
        I.ln1_b = add_p(pre + "ln1_b", S->hv, 1);
        I.wqkv = add_p(pre + "wqkv", S->vqkv_w, S->hv);
        I.bqkv = add_p(pre + "bqkv", S->vqkv_w, 1);
        I.wo = add_p(pre + "wo", S->hv, S->vo_w);
        I.bo = add_p(pre + "bo", S->hv, 1);
        I.ln2_g = add_p(pre + "ln2_g", S->hv, 1);
        I.ln2_b = add_p(pre + "ln2_b", S->hv, 1);
        I.w1 = add_p(pre + "w1", S->vml, S->hv);
        I.b1 = add_p(pre + "b1", S->vml, 1);
        I.w2 = add_p(pre + "w2", S->hv, S->vml);
        I.b2 = add_p(pre + "b2", S->hv, 1);
        S->vidx[l] = I;
      }
      S->p_mln_g = add_p("merger.ln_g", S->hv, 1);
      S->p_mln_b = add_p("merger.ln_b", S->hv, 1);
      S->p_mw1 = add_p("merger.w1", S->m4l, S->m4);
      S->p_mb1 = add_p("merger.b1", S->m4l, 1);
      S->p_mw2 = add_p("merger.w2", S->h, S->m4l);
      S->p_mb2 = add_p("merger.b2", S->h, 1);
      continue;
    }
    for (int l = C.l0; l < C.l0 + C.nl; ++l) {
      // LM layers are numbered from 0 in parameter names (the ViT layers of an
      // MLLM's vs 0 take global unit-layer indices 0..nvit-1)
      const std::string pre = "layers." + std::to_string(l - S->nvit) + ".";
      LayerIdx I;
      I.ln1 = add_p(pre + "ln1", S->h, 1);
      I.wqkv = add_p(pre + "wqkv", S->qkv_w, S->h);
      if (S->mc.qkv_bias) I.bqkv = add_p(pre + "bqkv", S->qkv_w, 1);
      I.wo = add_p(pre + "wo", S->h, S->o_w);
      I.ln2 = add_p(pre + "ln2", S->h, 1);
      I.wgu = add_p(pre + "wgu", 2 * S->fi, S->h);
      I.wd = add_p(pre + "wd", S->h, S->fi);
      S->lidx[l] = I;
    }
  }
  for (auto& C : S->chunks)
    if (C.first) S->p_embed = add_p("embed", S->Vl, S->h);
  for (auto& C : S->chunks)
    if (C.last) {
      S->p_final = add_p("final_ln", S->h, 1);
      S->p_lm = add_p("lm_head", S->Vl, S->h);
    }
  // internal accumulators of the replicated parameters whose gradient is a
  // sum over the sequence-parallel shards (TP all-reduced at the end of the
  // step): norm gains (and ViT LayerNorm biases) and the patch embedding
  S->dgamma_off.clear();
  int64_t off = 0;
  auto ends = [](const std::string& nm, const char* suf) {
    const size_t n = strlen(suf);
    return nm.size() >= n && nm.compare(nm.size() - n, n, suf) == 0;
  };
  for (size_t i = 0; i < S->params.size(); ++i) {
    const std::string& nm = S->params[i].name;
    const bool gamma = nm == "final_ln" || ends(nm, ".ln1") || ends(nm, ".ln2") || ends(nm, ".ln1_g") ||
                       ends(nm, ".ln1_b") || ends(nm, ".ln2_g") || ends(nm, ".ln2_b") || nm == "merger.ln_g" ||
                       nm == "merger.ln_b" || nm == "vit.patch";
    if (gamma) {
      S->dgamma_off[(int)i] = off;
      off += S->params[i].numel();
    }
  }
  S->dgamma_n = off;
  return STP_OK;
}

stp_status init_nccl(stp_stage* S, const void* uid) {
  const int world = S->t * S->p;
  if (world == 1) return STP_OK;
  if (!uid) return fail(STP_EINVAL, "world_nccl_id required when tp*pp > 1");
  {
    const char* c = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    if (!c || atoi(c) < 16)
      return fail(STP_EUNSUPPORTED,
                  "set CUDA_DEVICE_MAX_CONNECTIONS>=16 (32 recommended) before CUDA initialises: with the default 8 "
                  "hardware queues a spinning NCCL recv can serialise the matching send (deadlock)");
  }
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  setenv("NCCL_RUNTIME_CONNECT", "0", 0);  // connect at init (see warmup_comms)
  const int rank = S->pp_rank * S->t + S->tp_rank;
  STP_NCCL_TRY(ncclCommInitRank(&S->world, world, id, rank));
  S->owned.push_back(S->world);
  // TP group: same PP rank.  The TP collectives run concurrently with the
  // other microbatch's GEMMs (the braid), so their SM footprint is capped
  // (STP_NCCL_TP_CTAS, default 16): NCCL's default 32-channel kernels take SMs
  // from the overlapped GEMM (App. F contention).
  ncclConfig_t tcfg = NCCL_CONFIG_INITIALIZER;
  {
    const char* e = getenv("STP_NCCL_TP_CTAS");
    const int ctas = e ? atoi(e) : 16;
    if (ctas > 0) {
      tcfg.maxCTAs = ctas;
      tcfg.minCTAs = std::min(ctas, 2);
    }
  }
  STP_NCCL_TRY(ncclCommSplit(S->world, S->pp_rank, S->tp_rank, &S->tpc, &tcfg));
  if (S->tpc) S->owned.push_back(S->tpc);
  // PP channels: one 2-rank communicator per (virtual-stage edge, tp rank),
  // sender = rank 0.  Every rank enumerates every device's edges (the
  // schedule is deterministic), then splits them in rounds in which each
  // device appears in at most one edge.
  struct Edge {
    int src_vs, dst_vs, src_dev, dst_dev;
  };
  std::vector<Edge> edges;
  for (int d = 0; d < S->p; ++d) {
    std::vector<stp_unit> us;
    STP_TRY(schedule_expand(S->sched, d, S->lay, us, S->mllm));
    std::vector<std::pair<int, int>> ue;
    std::vector<char> uf;
    classify_pp_units(S->sched, S->p, d, us, ue, uf);
    for (size_t i = 0; i < us.size(); ++i)
      if (us[i].op == STP_U_PP_SEND) {
        Edge e{ue[i].first, ue[i].second, d, us[i].layer};
        bool seen = false;
        for (auto& x : edges) seen |= (x.src_vs == e.src_vs && x.dst_vs == e.dst_vs);
        if (!seen) edges.push_back(e);
      }
  }
  std::sort(edges.begin(), edges.end(), [](const Edge& a, const Edge& b) {
    return a.src_vs != b.src_vs ? a.src_vs < b.src_vs : a.dst_vs < b.dst_vs;
  });
  std::vector<std::vector<Edge>> rounds;
  for (auto& e : edges) {
    bool placed = false;
    for (auto& rd : rounds) {
      bool clash = false;
      for (auto& q : rd)
        clash |= q.src_dev == e.src_dev || q.src_dev == e.dst_dev || q.dst_dev == e.src_dev || q.dst_dev == e.dst_dev;
      if (!clash) {
        rd.push_back(e);
        placed = true;
        break;
      }
    }
    if (!placed) rounds.push_back({e});
  }
  const int me = S->pp_rank;
  for (auto& rd : rounds) {
    int color = NCCL_SPLIT_NOCOLOR, key = 0;
    const Edge* mine = nullptr;
    for (size_t i = 0; i < rd.size(); ++i)
      if (rd[i].src_dev == me || rd[i].dst_dev == me) {
        color = (int)i * S->t + S->tp_rank;
        key = rd[i].src_dev == me ? 0 : 1;
        mine = &rd[i];
      }
    ncclComm_t c = nullptr;
    ncclConfig_t pcfg = NCCL_CONFIG_INITIALIZER;
    {
      const char* e = getenv("STP_NCCL_PP_CTAS");
      const int ctas = e ? atoi(e) : 4;
      if (ctas > 0) {
        pcfg.maxCTAs = ctas;
        pcfg.minCTAs = 1;
      }
    }
    STP_NCCL_TRY(ncclCommSplit(S->world, color, key, &c, &pcfg));
    if (c && mine) {
      S->owned.push_back(c);
      const std::pair<int, int> k(mine->src_vs, mine->dst_vs);
      if (mine->src_dev == me) S->c_send[k] = c;
      else S->c_recv[k] = c;
    }
  }
  S->edges_sorted.clear();
  for (auto& e : edges) S->edges_sorted.push_back({e.src_vs, e.dst_vs});
  return STP_OK;
}

// NCCL sets up connections lazily, and the setup handshake blocks the host.
// Two ranks that first touch different communicators in different orders can
// therefore deadlock inside the handshake.  Touch every communicator once at
// init, in one global order: TP groups first (every rank is in exactly one),
// then every PP edge in sorted order (the globally smallest unfinished edge
// always has both endpoints waiting on it, so the sequence cannot deadlock).
// The TP collectives use the step's real message sizes so the algorithms the
// step will pick are the ones connected here.
stp_status warmup_comms(stp_stage* S) {
  const ncclDataType_t dt = (ncclDataType_t)ncdt(S->dtype);
  const size_t shard = (size_t)(S->sl * S->h);
  if (S->t > 1) {
    STP_NCCL_TRY(ncclReduceScatter(S->pf, S->rtmp, shard, dt, ncclSum, S->tpc, S->s_comm));
    STP_NCCL_TRY(ncclAllGather(S->ntmp, S->pf, shard, dt, S->tpc, S->s_comm));
    STP_NCCL_TRY(ncclAllGather(S->pf, S->pb, (size_t)(S->s * 3), ncclFloat32, S->tpc, S->s_comm));
    STP_NCCL_TRY(ncclAllReduce(S->dgamma, S->dgamma, (size_t)std::max<int64_t>(1, S->dgamma_n), ncclFloat32, ncclSum,
                               S->tpc, S->s_comm));
    if (S->mllm) {
      const size_t vsh = (size_t)(S->svl * S->hv);
      STP_NCCL_TRY(ncclReduceScatter(S->pf, S->vrtmp, vsh, dt, ncclSum, S->tpc, S->s_comm));
      STP_NCCL_TRY(ncclAllGather(S->vntmp, S->pf, vsh, dt, S->tpc, S->s_comm));
    }
    STP_CUDA_TRY(cudaStreamSynchronize(S->s_comm));
  }
  for (auto& e : S->edges_sorted) {
    auto is = S->c_send.find(e);
    if (is != S->c_send.end()) {
      cudaStream_t st = S->s_send.at(e);
      STP_NCCL_TRY(ncclSend(S->pf, shard, dt, 1, is->second, st));
      STP_CUDA_TRY(cudaStreamSynchronize(st));
    }
    auto ir = S->c_recv.find(e);
    if (ir != S->c_recv.end()) {
      cudaStream_t st = S->s_recv.at(e);
      STP_NCCL_TRY(ncclRecv(S->pb, shard, dt, 0, ir->second, st));
      STP_CUDA_TRY(cudaStreamSynchronize(st));
    }
  }
  return STP_OK;
}

}  // namespace
}  // namespace stp

// ------------------------------------------------------------------ C ABI
using namespace stp;

extern "C" {

int32_t stp_nccl_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

stp_status stp_nccl_get_id(void* buf) {
  if (!buf) return fail(STP_EINVAL, "buf is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(STP_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  memcpy(buf, &id, sizeof(id));
  return STP_OK;
}

static stp_status init_stage_impl(const stp_model_cfg* mc, const stp_vit_cfg* vc, const stp_parallel_cfg* pc,
                                  const void* world_nccl_id, int32_t cuda_device, stp_stage** out) {
  if (!mc || !pc || !out) return fail(STP_EINVAL, "NULL argument");
  *out = nullptr;
  const int t = pc->tp, p = pc->pp;
  STP_CHECK_ARG(t >= 1 && p >= 1, "tp, pp >= 1");
  STP_CHECK_ARG(pc->tp_rank >= 0 && pc->tp_rank < t && pc->pp_rank >= 0 && pc->pp_rank < p, "ranks");
  STP_CHECK_ARG(pc->n_micro >= 1, "n_micro >= 1");
  STP_CHECK_ARG(mc->dtype == STP_DTYPE_F32 || mc->dtype == STP_DTYPE_BF16, "dtype");
  STP_CHECK_ARG(mc->n_q_heads % t == 0 && mc->n_kv_heads % t == 0, "heads % tp == 0");
  STP_CHECK_ARG(mc->n_q_heads % mc->n_kv_heads == 0, "n_q_heads % n_kv_heads == 0");
  STP_CHECK_ARG(mc->ffn % t == 0 && mc->vocab % t == 0 && mc->seq % t == 0, "ffn, vocab, seq % tp == 0");
  STP_CHECK_ARG(mc->hidden % 8 == 0 && (mc->ffn / t) % 8 == 0, "hidden and ffn/tp multiples of 8");
  std::unique_ptr<stp_stage> S(new stp_stage);
  S->mc = *mc;
  S->t = t;
  S->p = p;
  S->vpp = pc->vpp;
  S->m = pc->n_micro;
  S->tp_rank = pc->tp_rank;
  S->pp_rank = pc->pp_rank;
  S->kind = pc->sched_kind;
  S->dtype = mc->dtype;
  S->es = dtype_size(mc->dtype);
  S->dev = cuda_device;
  S->s = mc->seq;
  S->sl = mc->seq / t;
  S->h = mc->hidden;
  S->d = mc->head_dim;
  S->qh = mc->n_q_heads / t;
  S->kh = mc->n_kv_heads / t;
  S->qkv_w = (S->qh + 2 * S->kh) * S->d;
  S->o_w = S->qh * S->d;
  S->fi = mc->ffn / t;
  S->Vl = mc->vocab / t;
  STP_CHECK_ARG(S->qkv_w % 8 == 0 && S->o_w % 8 == 0 && S->Vl % 8 == 0, "per-rank widths multiples of 8");
  if (vc) {
    S->mllm = true;
    S->vc = *vc;
    STP_CHECK_ARG(vc->n_layers >= 1 && vc->hidden % 8 == 0 && vc->patch_dim % 8 == 0, "ViT dims");
    STP_CHECK_ARG(vc->grid_h % 2 == 0 && vc->grid_w % 2 == 0, "ViT grid even (2x2 merge)");
    STP_CHECK_ARG(vc->n_heads % t == 0 && vc->mlp % t == 0 && (4 * vc->hidden) % t == 0, "ViT heads, mlp, 4h % tp");
    STP_CHECK_ARG(vc->n_heads * vc->head_dim == vc->hidden, "ViT n_heads * head_dim == hidden");
    STP_CHECK_ARG((vc->mlp / t) % 8 == 0 && (4 * vc->hidden / t) % 8 == 0, "ViT per-rank widths multiples of 8");
    S->nvit = vc->n_layers;
    S->sv = (int64_t)vc->grid_h * vc->grid_w;
    STP_CHECK_ARG(S->sv % (4 * t) == 0, "grid_h * grid_w % (4 tp) == 0");
    S->svl = S->sv / t;
    S->hv = vc->hidden;
    S->vnh = vc->n_heads / t;
    S->vd = vc->head_dim;
    S->vqkv_w = 3 * S->vnh * S->vd;
    S->vo_w = S->vnh * S->vd;
    S->vml = vc->mlp / t;
    S->vpd = vc->patch_dim;
    S->n_img = S->sv / 4;
    S->m4 = 4 * S->hv;
    S->m4l = S->m4 / t;
    STP_CHECK_ARG(S->n_img < S->s, "image tokens fewer than the LM sequence");
    STP_CHECK_ARG(mc->dtype == STP_DTYPE_F32 || S->vd == 80 || S->vd == 128, "bf16 ViT head_dim 80 or 128");
  }
  STP_TRY(schedule_build(p, pc->vpp, t, pc->n_micro, pc->sched_kind, S->sched));
  const int V = sched_n_vstages(S->kind, p);
  S->lay.resize(V);
  if (S->mllm) {
    STP_CHECK_ARG(V >= 2, "MLLM needs >= 2 virtual stages (ViT + LM)");
    S->lay[0] = (int)S->nvit;
    int sum = 0;
    if (pc->layers_per_vstage) {
      STP_CHECK_ARG(pc->layers_per_vstage[0] == S->nvit, "layers_per_vstage[0] must equal the ViT layer count");
      for (int i = 1; i < V; ++i) S->lay[i] = pc->layers_per_vstage[i];
    } else {
      STP_TRY(layer_split(mc->n_layers, V - 1, S->lay.data() + 1));
    }
    for (int i = 1; i < V; ++i) {
      STP_CHECK_ARG(S->lay[i] >= 1, "every LM virtual stage needs >= 1 layer");
      sum += S->lay[i];
    }
    if (sum != mc->n_layers) return fail(STP_EINVAL, "IndivisibleLayers: LM layers_per_vstage does not sum to n_layers");
  } else if (pc->layers_per_vstage) {
    int sum = 0;
    for (int i = 0; i < V; ++i) {
      S->lay[i] = pc->layers_per_vstage[i];
      STP_CHECK_ARG(S->lay[i] >= 1, "every virtual stage needs >= 1 layer");
      sum += S->lay[i];
    }
    if (sum != mc->n_layers) return fail(STP_EINVAL, "IndivisibleLayers: layers_per_vstage does not sum to n_layers");
  } else {
    STP_TRY(layer_split(mc->n_layers, V, S->lay.data()));
  }
  STP_TRY(schedule_expand(S->sched, S->pp_rank, S->lay, S->units, S->mllm));
  classify_pp_units(S->sched, p, S->pp_rank, S->units, S->unit_edge, S->unit_fwd);
  STP_CUDA_TRY(cudaSetDevice(cuda_device));
  // chunks held by this rank
  const int nchunks = sched_n_chunks(S->kind);
  for (int c = 0; c < nchunks; ++c) {
    Chunk C;
    C.c = c;
    C.vs = sched_vstage(S->kind, p, S->pp_rank, c);
    C.l0 = 0;
    for (int i = 0; i < C.vs; ++i) C.l0 += S->lay[i];
    C.nl = S->lay[C.vs];
    C.first = C.vs == 0;
    C.last = C.vs == V - 1;
    C.vit = S->mllm && C.vs == 0;
    S->chunks.push_back(C);
  }
  STP_TRY(build_params(S.get()));
  if (const char* e = getenv("STP_OFFLOAD_ALPHA")) {
    S->off_alpha = (float)atof(e);
    STP_CHECK_ARG(S->off_alpha >= 0.f && S->off_alpha <= 1.f, "STP_OFFLOAD_ALPHA in [0, 1]");
    if (!S->chunks[0].vit && S->chunks.size() == 2) S->off_n = (int)std::lround(S->off_alpha * S->chunks[0].nl);
  }
  // stash slots per chunk: program-order peak of live chunk-microbatches
  std::vector<int> cur(nchunks, 0), best(nchunks, 0);
  for (const auto& a : S->sched.ranks[S->pp_rank]) {
    const bool f = a.kind == STP_A_F || a.kind == STP_A_FB || a.kind == STP_A_FBS || a.kind == STP_A_FW;
    if (f) best[a.chunk] = std::max(best[a.chunk], ++cur[a.chunk]);
    if (a.kind == STP_A_BFULL || a.kind == STP_A_FB) --cur[a.chunk];
    if (a.kind == STP_A_W || a.kind == STP_A_FW) --cur[a.w_chunk];
  }
  S->peak_bytes = 0;
  for (auto& C : S->chunks) {
    Slot probe;
    Carver dry{nullptr, 0, true};
    carve_slot(S.get(), C, probe, dry);
    C.slot_bytes = dry.off + 256;
    C.slots.resize(best[C.c]);
    for (auto& sl : C.slots) {
      STP_TRY(dalloc(S.get(), &sl.mem, C.slot_bytes));
      Carver cv{(uint8_t*)sl.mem, 0, false};
      carve_slot(S.get(), C, sl, cv);
    }
    S->peak_bytes += (int64_t)C.slot_bytes * best[C.c];
  }
  if (S->off_n > 0) {
    // pool size: dry run of the unit list (acquire at F_MLP, release at the
    // D2H issue; n_off acquires at the reload, one release per W_MLP) + 2
    // blocks of slack so a forward does not wait for the previous D2H
    S->off_bytes = (size_t)(S->s * 3 * S->fi) * S->es;
    const Chunk& C0 = S->chunks[0];
    int cur = 0, peak = 0;
    std::map<int, bool> reloaded;
    for (const auto& u : S->units) {
      if (u.chunk != 0) continue;
      const int j = u.layer - C0.l0;
      if (u.op == STP_U_F_MLP && off_layer(S.get(), C0, j)) {
        peak = std::max(peak, ++cur);
        --cur;
        reloaded[u.mb] = false;
      } else if (u.op == STP_U_CB && u.layer == 0 && !reloaded[u.mb]) {
        cur += std::min(S->off_n, C0.nl);
        peak = std::max(peak, cur);
        reloaded[u.mb] = true;
      } else if (u.op == STP_U_W_MLP && off_layer(S.get(), C0, j)) {
        --cur;
      }
    }
    S->off_pool.resize(peak + 2);
    for (auto& b : S->off_pool) {
      STP_TRY(dalloc(S.get(), &b.dev, S->off_bytes));
      STP_CUDA_TRY(cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
    }
    S->peak_bytes += (int64_t)S->off_bytes * (int64_t)S->off_pool.size();
    for (auto& sl : S->chunks[0].slots)
      for (int j = 0; j < std::min(S->off_n, C0.nl); ++j) {
        void* hp = nullptr;
        STP_CUDA_TRY(cudaHostAlloc(&hp, S->off_bytes, cudaHostAllocDefault));
        S->host_allocs.push_back(hp);
        sl.L[j].host = hp;
        STP_CUDA_TRY(cudaEventCreateWithFlags(&sl.L[j].ev_d2h, cudaEventDisableTiming));
        STP_CUDA_TRY(cudaEventCreateWithFlags(&sl.L[j].ev_h2d, cudaEventDisableTiming));
      }
  }
  const size_t es = S->es;
  {
    // TP transport: p2p (default; fused NVLink kernels), ce (copy engines),
    // nccl (NCCL reduce-scatter / all-gather: the baseline)
    const char* e = getenv("STP_TP_TRANSPORT");
    // Default per schedule (round-2 contention sweep): braided
    // schedules overlap every comm phase with the other microbatch's GEMMs, so
    // they take the copy-engine transport (no SM-resident transfer kernel next
    // to the GEMMs); schedules whose forward comm is exposed take the fused p2p
    // kernel (the shortest phase).
    // (Ours^ braids only part of its units -- lone B / F expose their phases --
    // and measured faster on p2p: 69.3k vs 63.0k tokens/s at TP4)
    const bool braided = S->kind == STP_SCHED_STP || S->kind == STP_SCHED_STP_NOSEP;
    const std::string tr = e ? e : (S->mllm ? "nccl" : braided ? "ce" : "p2p");
    if (tr != "p2p" && tr != "ce" && tr != "nccl") return fail(STP_EINVAL, "STP_TP_TRANSPORT must be p2p, ce or nccl");
    S->ce = S->t > 1 && (tr == "ce" || tr == "p2p");
    S->p2p = S->ce && tr == "p2p";
    if (S->mllm && S->ce)
      return fail(STP_EUNSUPPORTED, "MLLM stages with tp > 1 need STP_TP_TRANSPORT=nccl (ViT phases use NCCL RS/AG)");
    const char* pu = getenv("STP_P2P_PUSH");
    S->p2p_push = S->p2p && S->dtype == STP_DTYPE_BF16 && S->t <= 8 && pu && atoi(pu) > 0;
    const char* w = getenv("STP_CE_WAIT");
    S->ce_spin = w && std::string(w) == "spin";
  }
  const int64_t part_elems = std::max(S->s * S->h, S->sv * S->hv);  // LM [S, h] and ViT [sv, hv] partials
  STP_TRY(dalloc(S.get(), &S->pfb[0], part_elems * es));
  STP_TRY(dalloc(S.get(), &S->pbb[0], part_elems * es));
  if (S->ce) {
    STP_TRY(dalloc(S.get(), &S->pfb[1], S->s * S->h * es));
    STP_TRY(dalloc(S.get(), &S->pbb[1], S->s * S->h * es));
    STP_TRY(dalloc(S.get(), &S->stage_buf, S->s * S->h * es));
    void* f = nullptr;
    STP_TRY(dalloc(S.get(), &f, 4096));
    S->flags = (uint32_t*)f;
    STP_CUDA_TRY(cudaMemset(S->flags, 0, 4096));
  } else {
    S->pfb[1] = S->pfb[0];
    S->pbb[1] = S->pbb[0];
  }
  S->pf = S->pfb[0];
  S->pb = S->pbb[0];
  STP_TRY(dalloc(S.get(), &S->rtmp, S->sl * S->h * es));
  STP_TRY(dalloc(S.get(), &S->ntmp, S->sl * S->h * es));
  STP_TRY(dalloc(S.get(), &S->dtmp_h, S->s * S->fi * es));
  STP_TRY(dalloc(S.get(), &S->dtmp_o, S->s * S->o_w * es));
  STP_TRY(dalloc(S.get(), &S->attn_ws, attn_bwd_ws_bytes(S->s, (int)S->qh, (int)S->kh, (int)S->d)));
  STP_TRY(dalloc(S.get(), &S->ce_ws, lm_head_ce_ws_bytes(S->s, S->Vl)));
  if (S->mllm) {
    STP_TRY(dalloc(S.get(), &S->vrtmp, S->svl * S->hv * es));
    STP_TRY(dalloc(S.get(), &S->vntmp, S->svl * S->hv * es));
    STP_TRY(dalloc(S.get(), &S->vdtmp_h, S->sv * S->vml * es));
    STP_TRY(dalloc(S.get(), &S->vdtmp_o, S->sv * S->vo_w * es));
    STP_TRY(dalloc(S.get(), &S->vdtmp_m, S->n_img * S->m4l * es));
    STP_TRY(dalloc(S.get(), &S->vattn_ws, attn_bwd_ws_bytes(S->sv, (int)S->vnh, (int)S->vnh, (int)S->vd)));
  }
  void* tmp = nullptr;
  STP_TRY(dalloc(S.get(), &tmp, std::max<int64_t>(1, S->dgamma_n) * sizeof(float)));
  S->dgamma = (float*)tmp;
  STP_TRY(dalloc(S.get(), &tmp, 256));
  S->loss_acc = (float*)tmp;
  STP_TRY(dalloc(S.get(), &tmp, (size_t)S->m * S->s * 4));
  S->tok_buf = (int32_t*)tmp;
  STP_TRY(dalloc(S.get(), &tmp, (size_t)S->m * S->s * 4));
  S->tgt_buf = (int32_t*)tmp;
  // streams
  int lo = 0, hi = 0;
  STP_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  STP_CUDA_TRY(cudaStreamCreateWithFlags(&S->s_comp, cudaStreamNonBlocking));
  STP_CUDA_TRY(cudaStreamCreateWithPriority(&S->s_comm, cudaStreamNonBlocking, hi));
  if (S->off_n > 0) {
    STP_CUDA_TRY(cudaStreamCreateWithFlags(&S->s_d2h, cudaStreamNonBlocking));
    STP_CUDA_TRY(cudaStreamCreateWithFlags(&S->s_h2d, cudaStreamNonBlocking));
  }
  // events
  const int n = (int)S->units.size();
  S->ev_done.resize(n);
  S->ev_t0.resize(n);
  S->ev_t1.resize(n);
  for (int i = 0; i < n; ++i) {
    STP_CUDA_TRY(cudaEventCreateWithFlags(&S->ev_done[i], cudaEventDisableTiming));
    STP_CUDA_TRY(cudaEventCreate(&S->ev_t0[i]));
    STP_CUDA_TRY(cudaEventCreate(&S->ev_t1[i]));
  }
  STP_CUDA_TRY(cudaEventCreate(&S->ev_base));
  STP_CUDA_TRY(cudaEventCreateWithFlags(&S->ev_caller, cudaEventDisableTiming));
  STP_CUDA_TRY(cudaEventCreate(&S->ev_end));
  STP_CUDA_TRY(cudaEventCreateWithFlags(&S->ev_join, cudaEventDisableTiming));
  STP_CUDA_TRY(cudaEventCreate(&S->ev_gstart));
  STP_CUDA_TRY(cudaEventCreate(&S->ev_gend));
  STP_CUDA_TRY(cudaHostAlloc((void**)&S->h_loss_pin, sizeof(float), cudaHostAllocDefault));
  *S->h_loss_pin = 0.f;
  // Graph replay needs replay-invariant synchronisation: the p2p / ce
  // transports' flag handshakes compare against phase numbers that grow every
  // step, so graphs are used with TP = 1 or the NCCL transport only.
  if (const char* e = getenv("STP_GRAPH")) S->use_graph = atoi(e) > 0 && !S->ce;
  for (int i = 0; i < 2; ++i) {
    STP_CUDA_TRY(cudaEventCreateWithFlags(&S->ev_pfb[i], cudaEventDisableTiming));
    STP_CUDA_TRY(cudaEventCreateWithFlags(&S->ev_pbb[i], cudaEventDisableTiming));
  }
  if (const char* e = getenv("STP_GEMM_MAX_CTAS")) S->gemm_max_ctas = atoi(e);
  S->debug = getenv("STP_DEBUG") != nullptr;
  STP_TRY(init_nccl(S.get(), world_nccl_id));
  for (auto& kv : S->c_send) {
    cudaStream_t st;
    STP_CUDA_TRY(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
    S->s_send[kv.first] = st;
  }
  for (auto& kv : S->c_recv) {
    cudaStream_t st;
    STP_CUDA_TRY(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
    S->s_recv[kv.first] = st;
  }
  // Optional NCCL user-buffer registration of every TP-collective buffer
  // (STP_NCCL_REGISTER=1): lets NVLink collectives read/write user buffers
  // directly instead of staging through NCCL's own buffers.
  if (S->tpc && S->t > 1 && getenv("STP_NCCL_REGISTER") && atoi(getenv("STP_NCCL_REGISTER")) > 0) {
    for (auto& C : S->chunks)
      for (auto& sl : C.slots) {
        void* h = nullptr;
        STP_NCCL_TRY(ncclCommRegister(S->tpc, sl.mem, C.slot_bytes, &h));
        S->nccl_regs.push_back({S->tpc, h});
      }
    for (void* b : {S->pf, S->pb, S->rtmp, S->ntmp}) {
      void* h = nullptr;
      const size_t bytes = (b == S->pf || b == S->pb) ? (size_t)(S->s * S->h * S->es) : (size_t)(S->sl * S->h * S->es);
      STP_NCCL_TRY(ncclCommRegister(S->tpc, b, bytes, &h));
      S->nccl_regs.push_back({S->tpc, h});
    }
  }
  STP_TRY(warmup_comms(S.get()));
  if (S->ce) STP_TRY(ce_init(S.get()));
  // every PP edge used by the unit list must have its communicator
  for (size_t i = 0; i < S->units.size(); ++i) {
    const stp_unit& u = S->units[i];
    if (u.op == STP_U_PP_SEND && !S->c_send.count(S->unit_edge[i])) return fail(STP_ENCCL, "missing PP send channel");
    if (u.op == STP_U_PP_RECV && !S->c_recv.count(S->unit_edge[i])) return fail(STP_ENCCL, "missing PP recv channel");
  }
  *out = S.release();
  return STP_OK;
}

stp_status stp_init_stage(const stp_model_cfg* mc, const stp_parallel_cfg* pc, const void* world_nccl_id,
                          int32_t cuda_device, stp_stage** out) {
  return init_stage_impl(mc, nullptr, pc, world_nccl_id, cuda_device, out);
}

stp_status stp_init_stage_mllm(const stp_model_cfg* mc, const stp_vit_cfg* vc, const stp_parallel_cfg* pc,
                               const void* world_nccl_id, int32_t cuda_device, stp_stage** out) {
  if (!vc) return fail(STP_EINVAL, "NULL vit cfg");
  return init_stage_impl(mc, vc, pc, world_nccl_id, cuda_device, out);
}

stp_status stp_stage_bind_images(stp_stage* st, const void* d_patches) {
  if (!st) return fail(STP_EINVAL, "NULL stage");
  if (!st->mllm) return fail(STP_ESTATE, "not an MLLM stage");
  if (!d_patches || (reinterpret_cast<uintptr_t>(d_patches) & 15)) return fail(STP_EINVAL, "patches: 16-byte aligned");
  st->patches = d_patches;
  return STP_OK;
}

stp_status stp_stage_param_count(const stp_stage* st, int32_t* n_out) {
  if (!st || !n_out) return fail(STP_EINVAL, "NULL argument");
  *n_out = (int32_t)st->params.size();
  return STP_OK;
}

stp_status stp_stage_param_info(const stp_stage* st, int32_t i, const char** name, int64_t* numel, int64_t* dim0,
                                int64_t* dim1) {
  if (!st) return fail(STP_EINVAL, "NULL stage");
  if (i < 0 || i >= (int32_t)st->params.size()) return fail(STP_EINVAL, "param index out of range");
  const Param& p = st->params[i];
  if (name) *name = p.name.c_str();
  if (numel) *numel = p.numel();
  if (dim0) *dim0 = p.d0;
  if (dim1) *dim1 = p.d1;
  return STP_OK;
}

stp_status stp_bind_params(stp_stage* st, int32_t n, void* const* param_ptrs, void* const* grad_ptrs) {
  if (!st || !param_ptrs || !grad_ptrs) return fail(STP_EINVAL, "NULL argument");
  if (n != (int32_t)st->params.size()) return fail(STP_EINVAL, "param count mismatch");
  for (int i = 0; i < n; ++i) {
    if (!param_ptrs[i] || !grad_ptrs[i]) return fail(STP_EINVAL, "NULL param/grad pointer");
    if ((reinterpret_cast<uintptr_t>(param_ptrs[i]) & 15) || (reinterpret_cast<uintptr_t>(grad_ptrs[i]) & 15))
      return fail(STP_EINVAL, "param/grad pointers must be 16-byte aligned");
    st->params[i].p = param_ptrs[i];
    st->params[i].g = (float*)grad_ptrs[i];
  }
  st->bound = true;
  return STP_OK;
}

stp_status stp_stage_set_timing(stp_stage* st, int32_t mode) {
  if (!st) return fail(STP_EINVAL, "NULL stage");
  st->timing = mode ? 1 : 0;
  return STP_OK;
}

// The step's first enqueue waits for everything the caller put on `stream`
// before the call (parameter updates, zero_grads, token writes); the caller's
// later work on `stream` is ordered after the step's last event.
static stp_status order_after_caller(stp_stage* st, void* stream) {
  STP_CUDA_TRY(cudaSetDevice(st->dev));
  STP_CUDA_TRY(cudaEventRecord(st->ev_caller, (cudaStream_t)stream));
  STP_CUDA_TRY(cudaStreamWaitEvent(st->s_comp, st->ev_caller, 0));
  return STP_OK;
}

stp_status stp_train_step(stp_stage* st, const int32_t* d_tokens, const int32_t* d_targets, float* h_loss,
                          stp_step_stats* stats, void* stream) {
  if (!st) return fail(STP_EINVAL, "NULL stage");
  if (st->poisoned) return fail(STP_ESTATE, "stage poisoned by an earlier CUDA/NCCL error");
  STP_TRY(order_after_caller(st, stream));
  bool need_tok = false, need_tgt = false;
  for (auto& C : st->chunks) {
    need_tok |= C.first;
    need_tgt |= C.last;
  }
  if (need_tok && !d_tokens) return fail(STP_EINVAL, "tokens required on the rank holding virtual stage 0");
  if (need_tgt && !d_targets) return fail(STP_EINVAL, "targets required on the rank holding the last virtual stage");
  st->tokens = d_tokens;
  st->targets = d_targets;
  STP_TRY(run_step(st, h_loss, stats));
  STP_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, st->ev_last ? st->ev_last : st->ev_end, 0));
  return STP_OK;
}

stp_status stp_train_step_host(stp_stage* st, const int32_t* h_tokens, const int32_t* h_targets, float* h_loss,
                               stp_step_stats* stats, void* stream) {
  if (!st) return fail(STP_EINVAL, "NULL stage");
  if (st->poisoned) return fail(STP_ESTATE, "stage poisoned by an earlier CUDA/NCCL error");
  STP_TRY(order_after_caller(st, stream));
  const size_t bytes = (size_t)st->m * st->s * 4;
  const int32_t* dt = nullptr;
  const int32_t* dg = nullptr;
  if (h_tokens) {
    STP_CUDA_TRY(cudaMemcpyAsync(st->tok_buf, h_tokens, bytes, cudaMemcpyHostToDevice, st->s_comp));
    dt = st->tok_buf;
  }
  if (h_targets) {
    STP_CUDA_TRY(cudaMemcpyAsync(st->tgt_buf, h_targets, bytes, cudaMemcpyHostToDevice, st->s_comp));
    dg = st->tgt_buf;
  }
  return stp_train_step(st, dt, dg, h_loss, stats, stream);
}

stp_status stp_stage_trace(const stp_stage* st, stp_unit* buf, int32_t cap, int32_t* n_out) {
  if (!st || !n_out) return fail(STP_EINVAL, "NULL argument");
  *n_out = (int32_t)st->trace.size();
  if (cap < (int32_t)st->trace.size()) return fail(STP_ECAPACITY, "buffer too small");
  std::copy(st->trace.begin(), st->trace.end(), buf);
  return STP_OK;
}

stp_status stp_stage_unit_times(const stp_stage* st, float* start_ms, float* end_ms, int32_t cap, int32_t* n_out) {
  if (!st || !n_out) return fail(STP_EINVAL, "NULL argument");
  *n_out = (int32_t)st->t_start.size();
  if (cap < (int32_t)st->t_start.size()) return fail(STP_ECAPACITY, "buffer too small");
  std::copy(st->t_start.begin(), st->t_start.end(), start_ms);
  std::copy(st->t_end.begin(), st->t_end.end(), end_ms);
  return STP_OK;
}

void stp_destroy_stage(stp_stage* st) {
  if (!st) return;
  cudaSetDevice(st->dev);
  cudaDeviceSynchronize();
  for (auto& r : st->nccl_regs) ncclCommDeregister(r.first, r.second);
  if (!st->sym_peer.empty()) {
    // close this rank's mappings of the peers' memory, then wait until every
    // peer has closed its mappings of ours before freeing it
    for (auto& v : st->sym_peer)
      for (uint8_t* p : v)
        if (p) cudaIpcCloseMemHandle(p);
    if (st->tpc && st->flags) {
      ncclAllReduce(st->flags, st->flags, 1, ncclUint32, ncclMax, st->tpc, st->s_comm);
      cudaStreamSynchronize(st->s_comm);
    }
  }
  for (auto s : st->s_pull) cudaStreamDestroy(s);
  for (auto c : st->owned)
    if (c) ncclCommDestroy(c);
  for (auto e : st->ev_done) cudaEventDestroy(e);
  for (auto e : st->ev_t0) cudaEventDestroy(e);
  for (auto e : st->ev_t1) cudaEventDestroy(e);
  for (auto e : st->ev_pool) cudaEventDestroy(e);
  if (st->ev_base) cudaEventDestroy(st->ev_base);
  if (st->ev_caller) cudaEventDestroy(st->ev_caller);
  if (st->ev_end) cudaEventDestroy(st->ev_end);
  if (st->ev_join) cudaEventDestroy(st->ev_join);
  if (st->ev_gstart) cudaEventDestroy(st->ev_gstart);
  if (st->ev_gend) cudaEventDestroy(st->ev_gend);
  if (st->graph_exec) cudaGraphExecDestroy(st->graph_exec);
  if (st->h_loss_pin) cudaFreeHost(st->h_loss_pin);
  for (int i = 0; i < 2; ++i) {
    if (st->ev_pfb[i]) cudaEventDestroy(st->ev_pfb[i]);
    if (st->ev_pbb[i]) cudaEventDestroy(st->ev_pbb[i]);
  }
  for (auto& b : st->off_pool)
    if (b.ev) cudaEventDestroy(b.ev);
  for (auto& C : st->chunks)
    for (auto& sl : C.slots)
      for (auto& L : sl.L) {
        if (L.ev_d2h) cudaEventDestroy(L.ev_d2h);
        if (L.ev_h2d) cudaEventDestroy(L.ev_h2d);
      }
  for (void* hp : st->host_allocs) cudaFreeHost(hp);
  if (st->s_d2h) cudaStreamDestroy(st->s_d2h);
  if (st->s_h2d) cudaStreamDestroy(st->s_h2d);
  for (auto& kv : st->s_send) cudaStreamDestroy(kv.second);
  for (auto& kv : st->s_recv) cudaStreamDestroy(kv.second);
  if (st->s_comp) cudaStreamDestroy(st->s_comp);
  if (st->s_comm) cudaStreamDestroy(st->s_comm);
  for (void* p : st->allocs) cudaFree(p);
  delete st;
}

}  // extern "C"
