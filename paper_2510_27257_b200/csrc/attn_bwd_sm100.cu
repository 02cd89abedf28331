// Causal GQA attention backward on the 5th-generation tensor cores (sm_100a),
// head_dim 128, bf16 operands / fp32 accumulation: ONE fused kernel computing
// dQ, dK and dV (FlashAttention-2's backward, the paper's attention kernel,
// PAPER.md §5 setup P:L169; math: SURVEY §8c.1 "Attention" —
//   P = exp(S - lse), dV = P^T dO, dP = dO V^T, dS = P (dP - D),
//   dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d), D = rowsum(dO O)).
//
// One CTA per (128-row key tile kt, query head h); grouped by kv head, heavy key
// tiles first within a group (kt = 0 sees every query tile).  Loop over the 64-row query
// tiles i >= 2 kt (causal), five GEMMs per (key tile, query tile):
//   S^T  = K Q_i^T              (TMEM, M = 128 keys, N = 64 queries)
//   dP^T = V dO_i^T             (TMEM)
//   dV  += P^T dO_i             (A = P^T from TMEM, bf16, written over S^T)
//   dK  += dS^T Q_i             (A = dS^T from TMEM, beside P^T)
//   dQ_i^T = K^T dS_i^T         (M = d, N = 64; A = K^T and B = dS^T from smem,
//                                both MN-major; D written over dP^T)
// dQ_i^T is drained from TMEM by the warp group that converted tile i, staged
// in shared memory as fp32 [64 queries][128 d] (in the tile's dS^T buffer,
// free once dQ_i has read it, plus a 16 KB buffer) and added into a head-major
// fp32 [nq + 2 nkv][s][128] accumulator by two bulk (TMA engine) reductions of
// contiguous rows (d = 80: per-element red.global.add); dK / dV are accumulated over the query
// loop in TMEM and added into the same accumulator once per CTA (the GQA sum
// over a kv head's query heads happens there: no per-head partials and no
// reduce pass).  attn_bwd_finalize converts the accumulator to bf16 (x 1/sqrt(d)
// for dQ, dK).  Work per (key, query) tile: 5 GEMMs, against 7 in the earlier
// two-kernel design (S and dP recomputed in a separate dQ kernel).
//
// Warp roles (384 threads): warp 0 TMA producer (K, V once; Q_i, dO_i and
// the per-row -lse*log2(e) / D vectors through a 3-stage ring), warp 1 MMA
// issuer (one lane), warp 2 TMEM allocator (512 columns), warps 4-7 / 8-11
// two ping-pong softmax groups (group g converts the query tiles with
// i % 2 == g; one key row per thread, 64 query columns).  TMEM: dV [0,128),
// dK [128,256), buffer b (= g) at 256 + 128 b: S^T [0,64) -> P^T [0,32) +
// dS^T [32,64); dP^T [64,128) -> dQ^T.  The MMA order per tile,
//   S(i+1), dV(i), dP(i+1), dQ(i), dK(i)   (dQ first: drained while dK runs),
// lets the tensor pipe compute tile i+1's S^T while group (i % 2) converts
// tile i; tcgen05.mma executes in issue order, so S(i+2) cannot overwrite
// P^T / dS^T(i) before dV(i) / dK(i) have read them, and dP(i+2) waits for
// the group to have drained dQ^T(i) (dq_free).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "attn_sm100_common.h"
#include "common.h"
#include "prof.h"

namespace stp {

stp_status tensor_map_heads(CUtensorMap* out, const void* ptr, int dh, int heads, int64_t rows, int64_t ld,
                            int box_rows);
stp_status set_max_smem_once(const void* func, int bytes, unsigned long long* mask);

namespace {

using namespace sm100;
using namespace attn;

constexpr int QT = 64;                    // query rows per tile
constexpr int QT_BYTES = QT * D * 2;      // 16 KB
constexpr int QATOM = QT * 64 * 2;        // 8 KB
constexpr int ST = 3;                     // Q_i / dO_i / (nl2, D) ring stages
constexpr int DS_BYTES = T * QT * 2;      // dS^T tile [128 keys][64 queries] bf16, 16 KB
constexpr int STG_BYTES = 32 * D * 4;     // dQ staging: query rows [32, 64) of a tile, fp32 [32][128]
constexpr int FB_SMEM = 1024 + 2 * TILE_BYTES + 2 * ST * QT_BYTES + 2 * DS_BYTES + 2 * STG_BYTES + 2 * ST * QT * 4 + 256;
static_assert(FB_SMEM <= 232448, "shared memory");

struct FusedArgs {
  int s, nq, nkv, sp;  // sp: padded row stride (multiple of QT) of nl2 / Dp
  int dh;              // head dim 128 (LM) or 80 (ViT, zero-padded to 128 by TMA)
  int causal;          // 1: causal (LM), 0: bidirectional (ViT)
  const float* nl2;    // [nq, sp]: -lse * log2(e); -inf beyond s (masks the ragged tail)
  const float* Dp;     // [nq, sp]: rowsum(dO * O); 0 beyond s
  float* acc;          // fp32 [nq + 2 nkv][s][128] (head-major): dq heads | dk | dv kv heads, zeroed
  float scale_log2;    // log2(e) / sqrt(d)
  int nt;              // key tiles
  int kv_major;        // 1: CTAs ordered by kv head, then key tile (heavy first), then query head
  int dq_bulk;         // 1: dQ tiles staged in smem and added by bulk (TMA) reductions; 0: red.add per element
};

__global__ void __launch_bounds__(384, 1)
    attn_bwd_fused_sm100(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q64,
                         const __grid_constant__ CUtensorMap tm_do64, const FusedArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by a pointer offset (not an integer round trip), so every
  // pointer derived from it keeps the shared state space: LDS / STS, not generic LD / ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE_BYTES;
  uint8_t* sQ = smem + 2 * TILE_BYTES;  // [ST]
  uint8_t* sdO = sQ + ST * QT_BYTES;    // [ST]
  uint8_t* sdS = sdO + ST * QT_BYTES;   // [2]
  float* s_stg = reinterpret_cast<float*>(sdS + 2 * DS_BYTES);  // [2][32][128] fp32
  float* s_nl = s_stg + 2 * 32 * D;                              // [ST][QT]
  float* s_D = s_nl + ST * QT;                                 // [ST][QT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_D + ST * QT);
  uint64_t* kv_full = bar;
  uint64_t* qdo_full = bar + 1;         // [ST]
  uint64_t* qdo_empty = qdo_full + ST;  // [ST]
  uint64_t* s_full = qdo_empty + ST;    // [2]
  uint64_t* dp_full = s_full + 2;       // [2]
  uint64_t* p_full = dp_full + 2;       // [2]  128 arrivals
  uint64_t* ds_full = p_full + 2;       // [2]  128 arrivals
  uint64_t* dq_full = ds_full + 2;      // [2]
  uint64_t* dq_free = dq_full + 2;      // [2]  128 arrivals
  uint64_t* done = dq_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = a.nq / a.nkv;
  int h, kt;
  if (a.kv_major) {
    // One GQA group (a kv head and its grp query heads) at a time: the CTAs in
    // flight then red.add into ~grp + 2 heads' rows of the accumulator (28 MB at
    // TP1, s 6144), which stay in L2; ordered by key tile within the group.
    const int b = blockIdx.x, per_g = grp * a.nt;
    kt = (b % per_g) / grp;
    h = (b / per_g) * grp + b % grp;
  } else {
    h = blockIdx.x % a.nq;
    kt = blockIdx.x / a.nq;
  }
  const int g = h / grp;
  const int nq64 = (a.s + QT - 1) / QT;
  const int q0 = a.causal ? 2 * kt : 0;  // first query tile that sees key tile kt
  const int n_q = nq64 - q0;
  const int kh = a.nq + g, vh = a.nq + a.nkv + g;  // head indices in the [q | k | v] row

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < ST; ++i) {
      mbar_init(qdo_full + i, 1);
      mbar_init(qdo_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(dp_full + i, 1);
      mbar_init(p_full + i, 128);
      mbar_init(ds_full + i, 128);
      mbar_init(dq_full + i, 1);
      mbar_init(dq_free + i, 128);
    }
    mbar_init(done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_q64);
    tma_prefetch_desc(&tm_do64);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tdV = tmem, tdK = tmem + 128, tB = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE_BYTES);
      tma_load_3d(sK, &tm_kv, kv_full, 0, kh, kt * T);
      tma_load_3d(sK + ATOM, &tm_kv, kv_full, 64, kh, kt * T);
      tma_load_3d(sV, &tm_kv, kv_full, 0, vh, kt * T);
      tma_load_3d(sV + ATOM, &tm_kv, kv_full, 64, vh, kt * T);
      for (int it = 0; it < n_q; ++it) {
        const int st = it % ST, qi = q0 + it;
        mbar_wait_wd(qdo_empty + st, ((it / ST) & 1) ^ 1, 301, a.s, h, kt);
        mbar_arrive_expect_tx(qdo_full + st, 2 * QT_BYTES + 2 * QT * 4);
        uint8_t* q = sQ + st * QT_BYTES;
        uint8_t* o = sdO + st * QT_BYTES;
        tma_load_3d(q, &tm_q64, qdo_full + st, 0, h, qi * QT);
        tma_load_3d(q + QATOM, &tm_q64, qdo_full + st, 64, h, qi * QT);
        tma_load_3d(o, &tm_do64, qdo_full + st, 0, h, qi * QT);
        tma_load_3d(o + QATOM, &tm_do64, qdo_full + st, 64, h, qi * QT);
        bulk_load(s_nl + st * QT, a.nl2 + (int64_t)h * a.sp + qi * QT, QT * 4, qdo_full + st);
        bulk_load(s_D + st * QT, a.Dp + (int64_t)h * a.sp + qi * QT, QT * 4, qdo_full + st);
      }
    }
  } else if (warp == 1) {
    // all 32 lanes run the issue loop (uniform descriptor arithmetic); one
    // elected lane issues each tcgen05 op.  SW128 descriptors of a tile base
    // plus a byte offset: desc(addr + off) = desc(addr) + off / 16.
    constexpr uint32_t idS = make_idesc_bf16(T, QT, false, false);  // S^T, dP^T: M = 128 keys, N = 64 queries
    const uint32_t idMN = make_idesc_bf16(T, a.dh, false, true);    // dV, dK: N = dh, B (dO_i, Q_i) MN-major
    const int nk = a.dh / 16;                                        // S^T / dP^T K-steps over d
    constexpr uint32_t idQ = make_idesc_bf16(T, QT, true, true);    // dQ^T: M = d (A = K^T), N = 64 (B = dS^T)
    const uint64_t dK_kmaj = make_sw128_desc(smem_u32(sK), 16, 1024);      // K as the K-major A of S^T
    const uint64_t dV_kmaj = make_sw128_desc(smem_u32(sV), 16, 1024);      // V as the K-major A of dP^T
    const uint64_t dK_mn = make_sw128_desc(smem_u32(sK), ATOM, 1024);      // K^T as the MN-major A of dQ^T
    const uint64_t dQ0_kmaj = make_sw128_desc(smem_u32(sQ), 16, 1024);     // Q_i (stage 0) K-major B of S^T
    const uint64_t ddO0_kmaj = make_sw128_desc(smem_u32(sdO), 16, 1024);   // dO_i K-major B of dP^T
    const uint64_t dQ0_mn = make_sw128_desc(smem_u32(sQ), QATOM, 1024);    // Q_i MN-major B of dK
    const uint64_t ddO0_mn = make_sw128_desc(smem_u32(sdO), QATOM, 1024);  // dO_i MN-major B of dV
    const uint64_t ddS0_mn = make_sw128_desc(smem_u32(sdS), QATOM, 1024);  // dS^T MN-major B of dQ^T
    mbar_wait_wd(kv_full, 0, 302, a.s, h, kt);
    auto issue_s = [&](int it) {
      const int st = it % ST, b = it & 1;
      mbar_wait_wd(qdo_full + st, (it / ST) & 1, 303, a.s, h, kt);
      tc_fence_after();
      const uint64_t qd = dQ0_kmaj + (uint64_t)((st * QT_BYTES) >> 4);
      const uint32_t tS = tB + 128 * b;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        if (kk >= nk) break;
        const uint32_t ka = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4, qa = ((kk >> 2) * QATOM + (kk & 3) * 32) >> 4;
        mma_f16_ss_el(tS, dK_kmaj + ka, qd + qa, idS, kk > 0 ? 1u : 0u);
      }
      mma_commit_el(s_full + b);
    };
    auto issue_dp = [&](int it) {
      const int st = it % ST, b = it & 1;
      if (it >= 2) mbar_wait_wd(dq_free + b, ((it >> 1) - 1) & 1, 304, a.s, h, kt);  // dQ^T(it-2) drained
      tc_fence_after();
      const uint64_t od = ddO0_kmaj + (uint64_t)((st * QT_BYTES) >> 4);
      const uint32_t tP = tB + 128 * b + 64;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        if (kk >= nk) break;
        const uint32_t ka = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4, qa = ((kk >> 2) * QATOM + (kk & 3) * 32) >> 4;
        mma_f16_ss_el(tP, dV_kmaj + ka, od + qa, idS, kk > 0 ? 1u : 0u);
      }
      mma_commit_el(dp_full + b);
    };
    issue_s(0);
    issue_dp(0);
    for (int it = 0; it < n_q; ++it) {
      const int st = it % ST, b = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      const uint64_t qmn = dQ0_mn + (uint64_t)((st * QT_BYTES) >> 4), omn = ddO0_mn + (uint64_t)((st * QT_BYTES) >> 4);
      const uint32_t tS = tB + 128 * b, tP = tS + 64;
      if (it + 1 < n_q) issue_s(it + 1);
      mbar_wait_wd(p_full + b, ph, 305, a.s, h, kt);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < QT / 16; ++kk)  // dV += P^T dO_i
        mma_f16_ts_el(tdV, tS + kk * 8, omn + (uint64_t)(kk * 128), idMN, (it > 0 || kk > 0) ? 1u : 0u);
      if (it + 1 < n_q) issue_dp(it + 1);
      mbar_wait_wd(ds_full + b, ph, 306, a.s, h, kt);
      tc_fence_after();
      // dQ first: the group drains it while the tensor pipe runs dK
      const uint64_t dsd = ddS0_mn + (uint64_t)((b * DS_BYTES) >> 4);
#pragma unroll
      for (int kk = 0; kk < T / 16; ++kk)  // dQ_i^T = K^T dS_i^T (K = 128 keys)
        mma_f16_ss_el(tP, dK_mn + (uint64_t)(kk * 128), dsd + (uint64_t)(kk * 128), idQ, kk > 0 ? 1u : 0u);
      mma_commit_el(dq_full + b);
#pragma unroll
      for (int kk = 0; kk < QT / 16; ++kk)  // dK += dS^T Q_i
        mma_f16_ts_el(tdK, tS + 32 + kk * 8, qmn + (uint64_t)(kk * 128), idMN, (it > 0 || kk > 0) ? 1u : 0u);
      mma_commit_el(qdo_empty + st);
    }
    mma_commit_el(done);
  } else if (warp >= 4) {
    const int gi = (warp - 4) >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;  // key row (S^T / dP^T lane); d index of dQ^T
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int krow = kt * T + r;
    const bool vrow = krow < a.s;
    const uint32_t tS = tB + 128 * gi, tP = tS + 64;  // group gi always uses buffer gi (tiles it % 2 == gi)
    uint8_t* dsrow = sdS + gi * DS_BYTES + (r >> 3) * 1024 + (r & 7) * 128;
    const uint64_t sc2 = pk2f(a.scale_log2, a.scale_log2);
    const bool leader = quad == 0 && lane == 0;
    float* stg0 = reinterpret_cast<float*>(sdS + gi * DS_BYTES);  // dQ rows [0, 32): dS^T(i) is consumed once dQ(i) is
    float* stg1 = s_stg + gi * 32 * D;                            // dQ rows [32, 64)
    for (int it = gi; it < n_q; it += 2) {
      const int st = it % ST;
      const uint32_t ph = (it >> 1) & 1;
      const int qbase = (q0 + it) * QT;
      mbar_wait_wd(qdo_full + st, (it / ST) & 1, 307, a.s, h, kt);  // nl2 / D of the tile staged
      mbar_wait_wd(s_full + gi, ph, 308, a.s, h, kt);
      tc_fence_after();
      float p[64];
      {
        uint32_t sv[64];
        tmem_ld_32x32b_x32(tS + lane_off, sv);
        tmem_ld_32x32b_x32(tS + 32 + lane_off, sv + 32);
        tmem_wait_ld();
        const float* nl = s_nl + st * QT;
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(nl + i);
          float t0, t1, t2, t3;
          up2f(ffma2(pk2f(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), sc2, pk2f(l4.x, l4.y)), t0, t1);
          up2f(ffma2(pk2f(__uint_as_float(sv[i + 2]), __uint_as_float(sv[i + 3])), sc2, pk2f(l4.z, l4.w)), t2, t3);
          p[i] = ex2(t0);
          p[i + 1] = ex2(t1);
          p[i + 2] = ex2(t2);
          p[i + 3] = ex2(t3);
        }
      }
      if ((a.causal && it < 2) || !vrow) {  // tiles overlapping the key tile: causal mask (query < key); rows beyond s
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (!vrow || (a.causal && qbase + i < krow)) p[i] = 0.f;
      }
      {
        uint32_t pp[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pp[i] = pack2(p[2 * i], p[2 * i + 1]);
        tmem_st_32x32b_x16(tS + lane_off, pp);  // P^T over S^T columns [0, 32) (this thread read all 64)
        tmem_st_32x32b_x16(tS + 16 + lane_off, pp + 16);
        tmem_wait_st();
      }
      tc_fence_before();
      mbar_arrive(p_full + gi);
      mbar_wait_wd(dp_full + gi, ph, 309, a.s, h, kt);
      tc_fence_after();
      if (a.dq_bulk && it >= 2) {  // the previous tile's bulk reductions have read sdS / the staging buffer
        if (leader) bulk_wait_read_all();
        named_bar_sync(1 + gi, 128);
      }
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t dv[32];
        tmem_ld_32x32b_x32(tP + ch * 32 + lane_off, dv);
        tmem_wait_ld();
        const float* Dq = s_D + st * QT + ch * 32;
        uint32_t pd[16];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 d4 = *reinterpret_cast<const float4*>(Dq + i);
          float d0, d1, d2, d3;
          up2f(fmul2(pk2f(p[ch * 32 + i], p[ch * 32 + i + 1]),
                     fsub2(pk2f(__uint_as_float(dv[i]), __uint_as_float(dv[i + 1])), pk2f(d4.x, d4.y))),
               d0, d1);
          up2f(fmul2(pk2f(p[ch * 32 + i + 2], p[ch * 32 + i + 3]),
                     fsub2(pk2f(__uint_as_float(dv[i + 2]), __uint_as_float(dv[i + 3])), pk2f(d4.z, d4.w))),
               d2, d3);
          pd[i >> 1] = pack2(d0, d1);
          pd[(i >> 1) + 1] = pack2(d2, d3);
        }
        tmem_st_32x32b_x16(tS + 32 + ch * 16 + lane_off, pd);  // dS^T over S^T columns [32, 64)
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // dS^T row r (64 queries = one 128-byte SW128 row, MN-major B of dQ^T)
          const int c = ch * 4 + j;
          *reinterpret_cast<uint4*>(dsrow + ((c ^ (r & 7)) << 4)) =
              make_uint4(pd[4 * j], pd[4 * j + 1], pd[4 * j + 2], pd[4 * j + 3]);
        }
      }
      tmem_wait_st();
      fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
      tc_fence_before();
      mbar_arrive(ds_full + gi);
      // drain dQ_i^T (TMEM lane = d, column = query) into the fp32 accumulator
      mbar_wait_wd(dq_full + gi, ph, 310, a.s, h, kt);
      tc_fence_after();
      uint32_t qv[64];
      tmem_ld_32x32b_x32(tP + lane_off, qv);
      tmem_ld_32x32b_x32(tP + 32 + lane_off, qv + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(dq_free + gi);
      // head-major accumulator: row stride 128 floats, so the 64 query rows of
      // this thread's column d are compile-time offsets of one pointer
      if (a.dq_bulk) {
        // stage the tile as fp32 [64 q][128 d] (rows of dQ^T's lane d = this
        // thread's column; d >= dh hold zeros) and add it with two bulk reductions
        // into the contiguous accumulator rows
#pragma unroll
        for (int j = 0; j < 32; ++j) stg0[j * D + r] = __uint_as_float(qv[j]);
#pragma unroll
        for (int j = 0; j < 32; ++j) stg1[j * D + r] = __uint_as_float(qv[32 + j]);
        fence_proxy_async();
        named_bar_sync(1 + gi, 128);
        if (leader) {
          const int nv = min(QT, a.s - qbase);
          float* dst0 = a.acc + ((int64_t)h * a.s + qbase) * D;
          bulk_reduce_add_f32(dst0, stg0, (uint32_t)min(nv, 32) * D * 4);
          if (nv > 32) bulk_reduce_add_f32(dst0 + 32 * D, stg1, (uint32_t)(nv - 32) * D * 4);
          bulk_commit();
        }
        continue;
      }
      float* dst = a.acc + ((int64_t)h * a.s + qbase) * D + r;
      if (r >= a.dh) {
        // zero-padded d rows of dQ^T: nothing to add
      } else if (qbase + QT <= a.s) {
#pragma unroll
        for (int j = 0; j < QT; ++j) red_add_f32(dst + j * D, __uint_as_float(qv[j]));
      } else {
        const int nv = a.s - qbase;
#pragma unroll
        for (int j = 0; j < QT; ++j)
          if (j < nv) red_add_f32(dst + j * D, __uint_as_float(qv[j]));
      }
    }
    if (a.dq_bulk && leader) bulk_wait_all();
    // dK / dV of the key tile: group gi adds d columns [64 gi, 64 gi + 64)
    mbar_wait_wd(done, 0, 311, a.s, h, kt);
    tc_fence_after();
    float* kr = a.acc + ((int64_t)(a.nq + g) * a.s + (vrow ? krow : 0)) * D + gi * 64;
    float* vr = kr + (int64_t)a.nkv * a.s * D;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      if (gi * 64 + c * 32 >= a.dh) break;  // d columns beyond dh
      uint32_t v[32], k[32];
      tmem_ld_32x32b_x32(tdV + gi * 64 + c * 32 + lane_off, v);
      tmem_ld_32x32b_x32(tdK + gi * 64 + c * 32 + lane_off, k);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          if (gi * 64 + c * 32 + i >= a.dh) break;
          red_add_v4_f32(vr + c * 32 + i, __uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                         __uint_as_float(v[i + 3]));
          red_add_v4_f32(kr + c * 32 + i, __uint_as_float(k[i]), __uint_as_float(k[i + 1]), __uint_as_float(k[i + 2]),
                         __uint_as_float(k[i + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// nl2[h][q] = -lse[h][q] * log2(e), Dp[h][q] = sum_d dO[q][h, d] O[q][h, d] for q < s;
// -inf / 0 for s <= q < sp (the padded tail masks itself in the fused kernel).
// One warp per (row, head); 4 columns per lane.
__global__ void attn_bwd_prep(int s, int sp, int nq, int dh, const bf16* __restrict__ o, const bf16* __restrict__ dout,
                              int64_t ldo, const float* __restrict__ lse, float* __restrict__ nl2,
                              float* __restrict__ Dp) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)sp * nq) return;
  const int q = (int)(w / nq), h = (int)(w % nq);
  if (q >= s) {
    if (lane == 0) {
      nl2[(int64_t)h * sp + q] = -INFINITY;
      Dp[(int64_t)h * sp + q] = 0.f;
    }
    return;
  }
  const int64_t off = (int64_t)q * ldo + (int64_t)h * dh + lane * 4;
  uint2 ov = make_uint2(0u, 0u), dv = make_uint2(0u, 0u);
  if (lane * 4 < dh) {  // dh % 4 == 0
    ov = *reinterpret_cast<const uint2*>(o + off);
    dv = *reinterpret_cast<const uint2*>(dout + off);
  }
  const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
  const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float2 of = __bfloat1622float2(o2[i]), df = __bfloat1622float2(d2[i]);
    acc = fmaf(of.x, df.x, acc);
    acc = fmaf(of.y, df.y, acc);
  }
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, k);
  if (lane == 0) {
    nl2[(int64_t)h * sp + q] = -lse[(int64_t)h * s + q] * LOG2E;
    Dp[(int64_t)h * sp + q] = acc;
  }
}

// dqkv (bf16, [s, ldd], columns dq | dk | dv) = acc (head-major [C][s][128])
// x (1/sqrt(d) for the dq and dk heads, 1 for dv).  One float4 per thread;
// a warp reads one 512-byte head row.
__global__ void attn_bwd_finalize(int s, int C, int qk_heads, int dh, const float* __restrict__ acc, bf16* dst,
                                  int64_t ldd, float scale) {
  const int nd4 = dh / 4;
  const int64_t total = (int64_t)s * C * nd4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int d4 = (int)(i % nd4) * 4;
    const int64_t rc = i / nd4;
    const int c = (int)(rc % C);
    const int64_t row = rc / C;
    const float4 v = *reinterpret_cast<const float4*>(acc + ((int64_t)c * s + row) * D + d4);
    const float sc = c < qk_heads ? scale : 1.f;
    *reinterpret_cast<uint2*>(dst + row * ldd + (int64_t)c * dh + d4) =
        make_uint2(pack2(v.x * sc, v.y * sc), pack2(v.z * sc, v.w * sc));
  }
}

}  // namespace

// Workspace of the fused path: nl2 [nq, sp], Dp [nq, sp], acc [nq + 2 nkv][s][128] (fp32).
int64_t attn_bwd_fused_ws_bytes(int64_t s, int nq, int nkv) {
  const int64_t sp = (s + QT - 1) / QT * QT;
  return 2 * (int64_t)nq * sp * 4 + 256 + s * (int64_t)(nq + 2 * nkv) * D * 4;
}

// d = 128 or 80 bf16, fused [q | k | v] layout of qkv and dqkv (row strides ld,
// ldd); o and dout share row stride ldo; causal (LM) or bidirectional (ViT).
stp_status attn_bwd_fused_launch(int s, int nq, int nkv, int dh, int causal, const void* qkv, int64_t ld,
                                 const void* o, const void* dout, int64_t ldo, const float* lse, void* dqkv,
                                 int64_t ldd, void* ws, cudaStream_t st) {
  static unsigned long long attr_mask = 0;
  STP_TRY(set_max_smem_once((const void*)attn_bwd_fused_sm100, FB_SMEM, &attr_mask));
  const int sp = (s + QT - 1) / QT * QT;
  float* nl2 = reinterpret_cast<float*>(ws);
  float* Dp = nl2 + (int64_t)nq * sp;
  float* acc = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(Dp + (int64_t)nq * sp) + 255) & ~uintptr_t(255));
  const int C = nq + 2 * nkv;
  STP_CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)s * C * D * 4, st));
  {
    const int64_t warps = (int64_t)sp * nq;
    attn_bwd_prep<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(s, sp, nq, dh, (const bf16*)o, (const bf16*)dout, ldo, lse,
                                                               nl2, Dp);
    count_launch();
    STP_LAUNCH_CHECK();
  }
  CUtensorMap tkv, tq64, td64;
  STP_TRY(tensor_map_heads(&tkv, qkv, dh, nq + 2 * nkv, s, ld, T));
  STP_TRY(tensor_map_heads(&tq64, qkv, dh, nq + 2 * nkv, s, ld, QT));
  STP_TRY(tensor_map_heads(&td64, dout, dh, nq, s, ldo, QT));
  FusedArgs a;
  a.s = s;
  a.nq = nq;
  a.nkv = nkv;
  a.sp = sp;
  a.nl2 = nl2;
  a.Dp = Dp;
  a.acc = acc;
  a.dh = dh;
  a.causal = causal;
  a.scale_log2 = LOG2E / sqrtf((float)dh);
  const int nt = (s + T - 1) / T;
  a.nt = nt;
  static const int kv_major = [] {
    const char* e = getenv("STP_ATTN_BWD_ORDER");  // "0": key tile major over all heads (round-2 order)
    return e && e[0] == '0' ? 0 : 1;
  }();
  a.kv_major = kv_major;
  static const int dq_bulk = [] {
    const char* e = getenv("STP_ATTN_DQ_BULK");  // "0": per-element red.add drain of dQ
    return e && e[0] == '0' ? 0 : 1;
  }();
  // d = 80 (ViT): the staged tile would carry 48 zero columns per row through
  // the bulk reductions (kbench 393 -> 363 TFLOP/s); per-element red.add there
  a.dq_bulk = dq_bulk && dh == D;
  attn_bwd_fused_sm100<<<(unsigned)(nq * nt), 384, FB_SMEM, st>>>(tkv, tq64, td64, a);
  count_launch();
  STP_LAUNCH_CHECK();
  {
    const int64_t total = (int64_t)s * C * (dh / 4);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 16 * num_sms());
    attn_bwd_finalize<<<grid, 256, 0, st>>>(s, C, nq + nkv, dh, acc, (bf16*)dqkv, ldd, 1.f / sqrtf((float)dh));
    count_launch();
    STP_LAUNCH_CHECK();
  }
  return STP_OK;
}

}  // namespace stp
