// Causal GQA attention forward on the 5th-generation tensor cores (sm_100a):
// tcgen05.mma with TMEM accumulators, operands staged by TMA (128-byte
// swizzle).  head_dim 128, bf16 operands, fp32 accumulation / softmax
// (FlashAttention-2's forward, the paper's attention kernel, §5
// setup P:L169; math: SURVEY §8c.1 "Attention", O = softmax(QK^T/sqrt(d) +
// causal) V, lse = log sum exp of each score row).
//
// One CTA = one 128-row query tile of one head; heavy tiles first across the
// whole grid (blockIdx.x = head, blockIdx.y = 0 is the last query tile, which
// sees every key tile).  384 threads:
//   warp 0      TMA producer (Q once; K_j, V_j double-buffered)
//   warp 1      MMA issuer, all lanes converged, one elected lane per
//               tcgen05 op: S_j = Q K_j^T into TMEM (two S buffers), then
//               O_h += P_h(j-1) V_{j-1}[64h..64h+63] per half h
//   warp 2      TMEM allocator (512 columns: O_0 | O_1 | S0 | S1)
//   warps 4-11  softmax, two warps per query row: half h = (warp - 4) / 4
//               owns key columns [64h, 64h + 64) of every S tile, keeps its
//               OWN running max / sum and its OWN O accumulator O_h (no
//               per-tile exchange between the halves), writes P_h (bf16
//               pairs) over the S columns it just read (A operand of PV from
//               TMEM), rescales O_h in TMEM only when its max grows by more
//               than 2^8 (exact: the stale max is used for P and the sum
//               alike).  The halves combine once at the end:
//               m = max(m_0, m_1), O = sum_h O_h 2^(m_h - m),
//               l = sum_h l_h 2^(m_h - m).
// The softmax warps are ALU-issue-bound: scale-and-subtract and the row sums
// run on packed fp32 pairs (FFMA2 / FADD2), the row max with 3-input max.
#include <cudaTypedefs.h>

#include <cmath>

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

struct FwdArgs {
  int s, nq, nkv;
  int dh;      // head dim: 128 (LM) or 80 (ViT); heads with dh < 128 are zero-padded to 128 by TMA
  int causal;  // 1: causal mask (LM); 0: bidirectional (ViT)
  int64_t ldo;
  void* o;
  float* lse;
  float scale_log2;  // log2(e) / sqrt(d)
};

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

constexpr int FWD_THREADS = 384;
constexpr int FWD_SMEM = 1024 + 5 * TILE_BYTES + 4 * T * 4 + 256;  // Q, K[2], V[2], (m, l) x 2 halves, barriers

__global__ void __launch_bounds__(FWD_THREADS, 1)
    attn_fwd_sm100(const __grid_constant__ CUtensorMap tm_qkv, const FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by a pointer offset (not an integer round trip), so every
  // pointer derived from it keeps the shared state space: LDS / STS, not generic LD / ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;      // [2]
  uint8_t* sV = smem + 3 * TILE_BYTES;  // [2]
  float* sml = reinterpret_cast<float*>(smem + 5 * TILE_BYTES);  // [2 halves][m, l][T]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sml + 4 * T);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;   // [2]
  uint64_t* p_full = bar + 11;  // [2 buffers][2 halves]
  uint64_t* o_done = bar + 15;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x;
  const int qt = gridDim.y - 1 - blockIdx.y;  // longest (most key tiles) first
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = a.causal ? qt + 1 : (a.s + T - 1) / T;  // causal: key tiles 0..qt
  const int kh = a.nq + g, vh = a.nq + a.nkv + g;          // head indices in the [q | k | v] row

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(o_done + i, 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(p_full + i, 128);
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem, tS0 = tmem + 256;  // O_h at tO + 128h; S buffer b at tS0 + 128b

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, TILE_BYTES);
      tma_load_3d(sQ, &tm_qkv, q_full, 0, h, qt * T);
      tma_load_3d(sQ + ATOM, &tm_qkv, q_full, 64, h, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait_wd(k_empty + b, ph ^ 1, 321, a.s, h, qt);
        mbar_arrive_expect_tx(k_full + b, TILE_BYTES);
        tma_load_3d(sK + b * TILE_BYTES, &tm_qkv, k_full + b, 0, kh, j * T);
        tma_load_3d(sK + b * TILE_BYTES + ATOM, &tm_qkv, k_full + b, 64, kh, j * T);
        mbar_wait_wd(v_empty + b, ph ^ 1, 322, a.s, h, qt);
        mbar_arrive_expect_tx(v_full + b, TILE_BYTES);
        tma_load_3d(sV + b * TILE_BYTES, &tm_qkv, v_full + b, 0, vh, j * T);
        tma_load_3d(sV + b * TILE_BYTES + ATOM, &tm_qkv, v_full + b, 64, vh, j * T);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idS = make_idesc_bf16(T, T, false, false);  // S = Q K^T (both K-major)
    const uint32_t idO = make_idesc_bf16(T, a.dh, false, true);    // O += P V (V MN-major, N = dh)
    const int nk = a.dh / 16;                                       // QK^T K-steps (zero padding skipped)
    const uint64_t dQ = make_sw128_desc(smem_u32(sQ), 16, 1024);
    const uint64_t dK0 = make_sw128_desc(smem_u32(sK), 16, 1024);
    const uint64_t dV0 = make_sw128_desc(smem_u32(sV), ATOM, 1024);
    mbar_wait_wd(q_full, 0, 323, a.s, h, qt);
    auto issue_pv = [&](int jj) {
      const int b = jj & 1;
      mbar_wait_wd(v_full + b, (jj >> 1) & 1, 325, a.s, h, qt);
      const uint64_t vd = dV0 + (uint64_t)((b * TILE_BYTES) >> 4);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        mbar_wait_wd(p_full + b * 2 + hf, (jj >> 1) & 1, 324, a.s, h, qt);
        tc_fence_after();
        // O_hf += P_hf (TMEM, keys 64hf..64hf+63: 32 packed columns) . V_j[64hf.., :]
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_f16_ts_el(tO + hf * 128, tS0 + b * 128 + hf * 64 + kk * 8, vd + (uint64_t)((hf * 4 + kk) * 128), idO,
                        (jj > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit_el(v_empty + b);
      mma_commit_el(o_done + b);
    };
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      mbar_wait_wd(k_full + b, ph, 326, a.s, h, qt);
      // buffer b last held P(j-2), consumed by PV(j-2), issued before this S(j) (in-order pipe)
      tc_fence_after();
      const uint64_t kd = dK0 + (uint64_t)((b * TILE_BYTES) >> 4);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        if (kk >= nk) break;
        const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
        mma_f16_ss_el(tS0 + b * 128, dQ + off, kd + off, idS, kk > 0 ? 1u : 0u);
      }
      mma_commit_el(k_empty + b);
      mma_commit_el(s_full + b);
      if (j > 0) issue_pv(j - 1);
    }
    issue_pv(n_kv - 1);
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2;          // key columns [64*half, 64*half + 64) of every S tile
    const int quad = warp & 3;                 // TMEM lanes 32*quad ..
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int qrow = qt * T + r;
    const float sl2 = a.scale_log2;
    const uint32_t tOh = tO + half * 128;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      mbar_wait_wd(s_full + b, (j >> 1) & 1, 328, a.s, h, qt);
      tc_fence_after();
      uint32_t u[64];
      tmem_ld_32x32b_x32(tS0 + b * 128 + half * 64 + lane_off, u);
      tmem_ld_32x32b_x32(tS0 + b * 128 + half * 64 + 32 + lane_off, u + 32);
      tmem_wait_ld();
      float sv[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) sv[i] = __uint_as_float(u[i]);
      const int cbase = j * T + half * 64;
      if ((a.causal && j == qt) || cbase + 64 > a.s) {  // diagonal or ragged tile: causal / length mask
        const int lim = a.causal ? min(qrow + 1, a.s) : a.s;
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (cbase + i >= lim) sv[i] = -INFINITY;
      }
      // row max as a 3-ary tree (depth 4) instead of a 31-deep dependent chain:
      // the softmax warps are latency-bound (two per scheduler)
      float m1[22];
#pragma unroll
      for (int i = 0; i < 21; ++i) m1[i] = fmax3(sv[3 * i], sv[3 * i + 1], sv[3 * i + 2]);
      m1[21] = sv[63];
      float m2[8];
#pragma unroll
      for (int i = 0; i < 7; ++i) m2[i] = fmax3(m1[3 * i], m1[3 * i + 1], m1[3 * i + 2]);
      m2[7] = m1[21];
      float mx = fmaxf(fmax3(m2[0], m2[1], m2[2]), fmax3(m2[3], m2[4], fmax3(m2[5], m2[6], m2[7]))) * sl2;
      const bool need = mx > m + 8.f;
      if (__any_sync(0xffffffffu, need)) {
        float alpha = 1.f;
        if (need) {
          alpha = (m == -INFINITY) ? 0.f : ex2(m - mx);
          l *= alpha;
          m = mx;
        }
        if (j > 0) {  // O_half holds PV(0..j-1): wait for PV(j-1), rescale all 128 columns
          mbar_wait_wd(o_done + ((j - 1) & 1), ((j - 1) >> 1) & 1, 329, a.s, h, qt);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            const uint32_t ta = tOh + c * 32 + lane_off;
            tmem_ld_32x32b_x32(ta, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(ta, v);
          }
          tmem_wait_st();
        }
      }
      // m == -inf (every key of this half masked so far): exponent -inf -> P = 0
      const float nm = (m == -INFINITY) ? -INFINITY : -m;
      const uint64_t sc2 = pk2f(sl2, sl2), nm2 = pk2f(nm, nm);
      uint64_t lacc[4] = {pk2f(0.f, 0.f), pk2f(0.f, 0.f), pk2f(0.f, 0.f), pk2f(0.f, 0.f)};  // 4 chains of 8
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        float t0, t1;
        up2f(ffma2(pk2f(sv[i], sv[i + 1]), sc2, nm2), t0, t1);
        const float p0 = ex2(t0), p1 = ex2(t1);
        lacc[(i >> 1) & 3] = fadd2(lacc[(i >> 1) & 3], pk2f(p0, p1));
        pk[i >> 1] = pack2(p0, p1);
      }
      {
        float l0, l1;
        up2f(fadd2(fadd2(lacc[0], lacc[1]), fadd2(lacc[2], lacc[3])), l0, l1);
        l += l0 + l1;
      }
      // P_half over the first 32 of this half's 64 S columns (already read above)
      tmem_st_32x32b_x32(tS0 + b * 128 + half * 64 + lane_off, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full + b * 2 + half);
    }
    // combine the halves: exchange (m, l) once
    sml[(half * 2 + 0) * T + r] = m;
    sml[(half * 2 + 1) * T + r] = l;
    named_bar_sync(2, 256);
    const float m0 = sml[0 * T + r], l0 = sml[1 * T + r], m1 = sml[2 * T + r], l1 = sml[3 * T + r];
    const float mt = fmaxf(m0, m1);
    const float f0 = (m0 == -INFINITY) ? 0.f : ex2(m0 - mt), f1 = (m1 == -INFINITY) ? 0.f : ex2(m1 - mt);
    const float lt = l0 * f0 + l1 * f1;
    mbar_wait_wd(o_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1, 331, a.s, h, qt);
    tc_fence_after();
    const bool valid = qrow < a.s;
    const float inv = 1.f / lt;
    const float c0 = f0 * inv, c1 = f1 * inv;
    bf16* orow = reinterpret_cast<bf16*>(a.o) + (int64_t)(valid ? qrow : 0) * a.ldo + (int64_t)h * a.dh + half * 64;
    const int ncol = min(64, a.dh - half * 64);  // columns of [64 half, 64 half + 64) inside the head
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {  // this half writes output columns [64 half, 64 half + 64)
      if (c * 32 >= ncol) break;
      uint32_t v0[32], v1[32];
      tmem_ld_32x32b_x32(tO + half * 64 + c * 32 + lane_off, v0);
      tmem_ld_32x32b_x32(tO + 128 + half * 64 + c * 32 + lane_off, v1);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          if (c * 32 + i >= ncol) break;
          float o8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) o8[e] = __uint_as_float(v0[i + e]) * c0 + __uint_as_float(v1[i + e]) * c1;
          uint4 q;
          q.x = pack2(o8[0], o8[1]);
          q.y = pack2(o8[2], o8[3]);
          q.z = pack2(o8[4], o8[5]);
          q.w = pack2(o8[6], o8[7]);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = q;
        }
      }
    }
    if (valid && half == 0) a.lse[(int64_t)h * a.s + qrow] = (mt + log2f(lt)) * 0.69314718055994530942f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

// d = 128 or 80, bf16, fused [q | k | v] row layout (row stride ld); causal
// (LM) or bidirectional (ViT).
stp_status attn_fwd_sm100_launch(int s, int nq, int nkv, int dh, int causal, const void* qkv_base, int64_t ld,
                                 void* o, int64_t ldo, float* lse, cudaStream_t st) {
  static unsigned long long attr_mask = 0;
  STP_TRY(set_max_smem_once((const void*)attn_fwd_sm100, FWD_SMEM, &attr_mask));
  CUtensorMap tm;
  STP_TRY(tensor_map_heads(&tm, qkv_base, dh, nq + 2 * nkv, s, ld, T));
  FwdArgs a;
  a.dh = dh;
  a.causal = causal;
  a.s = s;
  a.nq = nq;
  a.nkv = nkv;
  a.ldo = ldo;
  a.o = o;
  a.lse = lse;
  a.scale_log2 = LOG2E / sqrtf((float)dh);
  attn_fwd_sm100<<<dim3(nq, (s + T - 1) / T), FWD_THREADS, FWD_SMEM, st>>>(tm, a);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

}  // namespace stp
