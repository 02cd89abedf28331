// Causal GQA attention forward on the 5th-generation tensor cores (sm_100a):
// tcgen05.mma with TMEM accumulators, operands staged by TMA (128-byte
// swizzle).  Used for head_dim 128 in bf16 (the Qwen2 shapes of the hot
// path); other head dims use the mma.sync kernels in attention.cu.
//
// One CTA = one 128-row query tile of one head, 256 threads:
//   warp 0      TMA producer (Q once; K_j, V_j double-buffered)
//   warp 1      MMA issuer (one lane): S_j = Q K_j^T into TMEM (two S
//               buffers), then O += P_{j-1} V_{j-1} (O in TMEM)
//   warp 2      TMEM allocator (512 columns: O | S0 | S1)
//   warps 4-7   softmax: thread r owns query row r; reads S_j from TMEM,
//               online softmax in the log2 domain, writes P_j (bf16) to smem
//               in the UMMA K-major SW128 layout, rescales O in TMEM only
//               when the running max grows by more than 2^8 (exact: the same
//               stale max is used for P and for the row sum), finally
//               normalises O and writes O and the LSE.
#include <cudaTypedefs.h>

#include "common.h"
#include "prof.h"
#include "sm100.h"

namespace stp {

stp_status tensor_map_bf16(CUtensorMap* out, const void* ptr, int64_t d0, int64_t d1, int64_t ld, int b0, int b1);

namespace {

using namespace sm100;

constexpr int T = 128;             // query rows per CTA = key rows per tile
constexpr int D = 128;             // head dim
constexpr int TILE_BYTES = T * D * 2;  // 32 KB: two 16 KB SW128 atoms (64 columns each)
constexpr int ATOM = T * 64 * 2;       // 16 KB
constexpr int SMEM_BYTES = 1024 + 7 * TILE_BYTES + 256;  // Q, K0, K1, V0, V1, P0, P1 + barriers

struct FwdArgs {
  int s, nq, nkv;
  int64_t ldo;
  void* o;
  float* lse;
  float scale_log2;  // log2(e) / sqrt(d)
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pair arithmetic of sm_100 (FFMA2 / FADD2 / FMUL2: two lanes of
// fp32 per instruction) and the 3-input max (FMNMX3): the softmax warps are
// issue-bound, so halving the per-element ALU instruction count matters.
__device__ __forceinline__ uint64_t pk2f(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2f(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// 2^x on the FMA pipe (FA4-style MUFU offload): round-to-nearest split
// x = i + f (magic-number add, f in [-0.5, 0.5]), degree-4 polynomial for 2^f
// (max rel. error ~4e-6 on [-0.5, 0.5]), 2^i by exponent-field add.  x < -126
// flushes to 0 like ex2.approx.ftz.
__device__ __forceinline__ float ex2_fma(float x) {
  x = fmaxf(x, -127.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: integer part lands in the mantissa
  const int i = __float_as_int(t) - 0x4B400000;
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.0013333558f, 0.0096181291f);
  p = fmaf(p, f, 0.0555041087f);
  p = fmaf(p, f, 0.2402265070f);
  p = fmaf(p, f, 0.6931471806f);
  p = fmaf(p, f, 1.0f);
  return x <= -126.f ? 0.f : __int_as_float(__float_as_int(p) + (i << 23));
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void __launch_bounds__(256, 1)
    attn_fwd_sm100(const __grid_constant__ CUtensorMap tm_qkv, const FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;          // 2 buffers
  uint8_t* sV = smem + 3 * TILE_BYTES;      // 2 buffers
  uint8_t* sP = smem + 5 * TILE_BYTES;      // 2 buffers
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 7 * TILE_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;   // [2]
  uint64_t* s_empty = bar + 11; // [2]
  uint64_t* p_full = bar + 13;  // [2]
  uint64_t* o_done = bar + 15;  // [2]: PV of tiles with j % 2 == b done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = gridDim.x;
  const int qt = nqt - 1 - blockIdx.x;  // longest (most key tiles) first
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = qt + 1;              // causal: key tiles 0..qt
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 128);
      mbar_init(p_full + i, 128);
      mbar_init(o_done + i, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem, tS0 = tmem + 128;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, q_full, qcol, qt * T);
      tma_load_2d(sQ + ATOM, &tm_qkv, q_full, qcol + 64, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(k_empty + b, ph ^ 1);
        mbar_arrive_expect_tx(k_full + b, TILE_BYTES);
        tma_load_2d(sK + b * TILE_BYTES, &tm_qkv, k_full + b, kcol, j * T);
        tma_load_2d(sK + b * TILE_BYTES + ATOM, &tm_qkv, k_full + b, kcol + 64, j * T);
        mbar_wait(v_empty + b, ph ^ 1);
        mbar_arrive_expect_tx(v_full + b, TILE_BYTES);
        tma_load_2d(sV + b * TILE_BYTES, &tm_qkv, v_full + b, vcol, j * T);
        tma_load_2d(sV + b * TILE_BYTES + ATOM, &tm_qkv, v_full + b, vcol + 64, j * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_bf16(T, T, false, false);  // S = Q K^T
      constexpr uint32_t idO = make_idesc_bf16(T, D, false, true);   // O += P V (V MN-major)
      const uint32_t q_addr = smem_u32(sQ), p_addr = smem_u32(sP);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int jj) {
        const int b = jj & 1;
        mbar_wait(p_full + b, (jj >> 1) & 1);
        mbar_wait(v_full + b, (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + b * TILE_BYTES);
        const uint32_t pb_addr = p_addr + b * TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          const uint64_t ad = make_sw128_desc(pb_addr + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = make_sw128_desc(v_addr + kk * 2048, ATOM, 1024);
          mma_f16_ss(tO, ad, bd, idO, (jj > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(v_empty + b);
        mma_commit(o_done + b);
      };
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(k_full + b, ph);
        mbar_wait(s_empty + b, ph ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES);
        const uint32_t tS = tS0 + b * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = make_sw128_desc(q_addr + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = make_sw128_desc(k_addr + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
          mma_f16_ss(tS, ad, bd, idS, kk > 0 ? 1u : 0u);
        }
        mma_commit(k_empty + b);
        mma_commit(s_full + b);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_kv - 1);
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;       // query row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int qrow = qt * T + r;
    float m = -INFINITY, l = 0.f;
    uint8_t* prow0 = sP + (r >> 3) * 1024 + (r & 7) * 128;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      mbar_wait(s_full + b, (j >> 1) & 1);
      tc_fence_after();
      float sv[T];
      {
        uint32_t v[T];
#pragma unroll
        for (int c = 0; c < T / 32; ++c) tmem_ld_32x32b_x32(tS0 + b * 128 + lane_off + c * 32, v + c * 32);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < T; ++i) sv[i] = __uint_as_float(v[i]);
      }
      tc_fence_before();
      mbar_arrive(s_empty + b);
      // scale to the log2 domain, causal / length mask, row max
      float mx = -INFINITY;
      const int kbase = j * T;
      const bool diag = (j == qt);
#pragma unroll
      for (int i = 0; i < T; ++i) {
        float x = sv[i] * a.scale_log2;
        if ((diag && kbase + i > qrow) || kbase + i >= a.s) x = -INFINITY;
        sv[i] = x;
        mx = fmaxf(mx, x);
      }
      // rescale O and l to a new max only when it grew by > 2^8 (first tile:
      // m = -inf); tcgen05.ld/st are warp-collective, so the branch is
      // warp-uniform and rows that keep their max use alpha = 1
      const bool need = mx > m + 8.f;
      if (__any_sync(0xffffffffu, need)) {
        float alpha = 1.f;
        if (need) {
          alpha = (m == -INFINITY) ? 0.f : ex2(m - mx);
          l *= alpha;
          m = mx;
        }
        if (j > 0) {
          // O must be stable: every PV up to j-1 has completed
          mbar_wait(o_done + ((j - 1) & 1), ((j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tO + lane_off + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(tO + lane_off + c * 32, v);
          }
          tmem_wait_st();
        }
      } else if (j >= 2) {
        mbar_wait(o_done + b, ((j - 2) >> 1) & 1);  // P buffer b free (PV j-2 done)
      }
      // P = exp2(x - m) -> bf16, K-major SW128 smem layout (two 64-col atoms)
      uint8_t* prow = prow0 + b * TILE_BYTES;
#pragma unroll
      for (int c = 0; c < T / 8; ++c) {
        float p[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          p[i] = ex2(sv[c * 8 + i] - m);
          l += p[i];
        }
        uint4 u;
        u.x = pack2(p[0], p[1]);
        u.y = pack2(p[2], p[3]);
        u.z = pack2(p[4], p[5]);
        u.w = pack2(p[6], p[7]);
        const int atom = c >> 3, ch = c & 7;
        *reinterpret_cast<uint4*>(prow + atom * ATOM + ((ch ^ (r & 7)) << 4)) = u;
      }
      fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
      tc_fence_before();
      mbar_arrive(p_full + b);
    }
    // epilogue: O / l once the last PV (and therefore all) completed
    mbar_wait(o_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1);
    tc_fence_after();
    // every lane loads (tcgen05.ld is warp-collective); rows >= s skip the store
    const bool valid = qrow < a.s;
    const float inv = 1.f / l;
    bf16* orow = reinterpret_cast<bf16*>(a.o) + (int64_t)(valid ? qrow : 0) * a.ldo + (int64_t)h * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tO + lane_off + c * 32, v);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          u.x = pack2(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv);
          u.y = pack2(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv);
          u.z = pack2(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv);
          u.w = pack2(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = u;
        }
      }
    }
    if (valid) a.lse[(int64_t)h * a.s + qrow] = (m + log2f(l)) * 0.69314718055994530942f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}


// Forward, version 2: P in TMEM (A operand of PV, tcgen05 ts-mode), three K/V
// stages in the freed shared memory.
constexpr int KV_ST = 3;
constexpr int SMEM_BYTES_V2 = 1024 + (1 + 2 * KV_ST) * TILE_BYTES + 256;

__global__ void __launch_bounds__(256, 1)
    attn_fwd_sm100_v2(const __grid_constant__ CUtensorMap tm_qkv, const FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;          // KV_ST buffers
  uint8_t* sV = smem + (1 + KV_ST) * TILE_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (1 + 2 * KV_ST) * TILE_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;            // [KV_ST]
  uint64_t* k_empty = k_full + KV_ST;    // [KV_ST]
  uint64_t* v_full = k_empty + KV_ST;    // [KV_ST]
  uint64_t* v_empty = v_full + KV_ST;    // [KV_ST]
  uint64_t* s_full = v_empty + KV_ST;    // [2]
  uint64_t* s_empty = s_full + 2;        // [2]
  uint64_t* p_full = s_empty + 2;        // [2]
  uint64_t* o_done = p_full + 2;         // [2]: PV of tiles with j % 2 == b done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = gridDim.x;
  const int qt = nqt - 1 - blockIdx.x;  // longest (most key tiles) first
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = qt + 1;              // causal: key tiles 0..qt
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KV_ST; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 128);
      mbar_init(p_full + i, 128);
      mbar_init(o_done + i, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem, tS0 = tmem + 128, tP0 = tmem + 384;  // P0 | P1: 64 columns each

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, q_full, qcol, qt * T);
      tma_load_2d(sQ + ATOM, &tm_qkv, q_full, qcol + 64, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j % KV_ST;
        const uint32_t ph = (j / KV_ST) & 1;
        mbar_wait(k_empty + b, ph ^ 1);
        mbar_arrive_expect_tx(k_full + b, TILE_BYTES);
        tma_load_2d(sK + b * TILE_BYTES, &tm_qkv, k_full + b, kcol, j * T);
        tma_load_2d(sK + b * TILE_BYTES + ATOM, &tm_qkv, k_full + b, kcol + 64, j * T);
        mbar_wait(v_empty + b, ph ^ 1);
        mbar_arrive_expect_tx(v_full + b, TILE_BYTES);
        tma_load_2d(sV + b * TILE_BYTES, &tm_qkv, v_full + b, vcol, j * T);
        tma_load_2d(sV + b * TILE_BYTES + ATOM, &tm_qkv, v_full + b, vcol + 64, j * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_bf16(T, T, false, false);  // S = Q K^T
      constexpr uint32_t idO = make_idesc_bf16(T, D, false, true);   // O += P V (V MN-major)
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int jj) {
        const int pb = jj & 1, vb = jj % KV_ST;
        mbar_wait(p_full + pb, (jj >> 1) & 1);
        mbar_wait(v_full + vb, (jj / KV_ST) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + vb * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          const uint64_t bd = make_sw128_desc(v_addr + kk * 2048, ATOM, 1024);
          mma_f16_ts(tO, tP0 + pb * 64 + kk * 8, bd, idO, (jj > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(v_empty + vb);
        mma_commit(o_done + pb);
      };
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1, kb = j % KV_ST;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(k_full + kb, (j / KV_ST) & 1);
        mbar_wait(s_empty + b, ph ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + kb * TILE_BYTES);
        const uint32_t tS = tS0 + b * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = make_sw128_desc(q_addr + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = make_sw128_desc(k_addr + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
          mma_f16_ss(tS, ad, bd, idS, kk > 0 ? 1u : 0u);
        }
        mma_commit(k_empty + kb);
        mma_commit(s_full + b);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_kv - 1);
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;       // query row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int qrow = qt * T + r;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      mbar_wait(s_full + b, (j >> 1) & 1);
      tc_fence_after();
      float sv[T];
      {
        uint32_t v[T];
#pragma unroll
        for (int c = 0; c < T / 32; ++c) tmem_ld_32x32b_x32(tS0 + b * 128 + lane_off + c * 32, v + c * 32);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < T; ++i) sv[i] = __uint_as_float(v[i]);
      }
      tc_fence_before();
      mbar_arrive(s_empty + b);
      // scale to the log2 domain, causal / length mask, row max
      float mx = -INFINITY;
      const int kbase = j * T;
      const bool diag = (j == qt);
#pragma unroll
      for (int i = 0; i < T; ++i) {
        float x = sv[i] * a.scale_log2;
        if ((diag && kbase + i > qrow) || kbase + i >= a.s) x = -INFINITY;
        sv[i] = x;
        mx = fmaxf(mx, x);
      }
      // rescale O and l to a new max only when it grew by > 2^8 (first tile:
      // m = -inf); tcgen05.ld/st are warp-collective, so the branch is
      // warp-uniform and rows that keep their max use alpha = 1
      const bool need = mx > m + 8.f;
      if (__any_sync(0xffffffffu, need)) {
        float alpha = 1.f;
        if (need) {
          alpha = (m == -INFINITY) ? 0.f : ex2(m - mx);
          l *= alpha;
          m = mx;
        }
        if (j > 0) {
          // O must be stable: every PV up to j-1 has completed
          mbar_wait(o_done + ((j - 1) & 1), ((j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tO + lane_off + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(tO + lane_off + c * 32, v);
          }
          tmem_wait_st();
        }
      } else if (j >= 2) {
        mbar_wait(o_done + b, ((j - 2) >> 1) & 1);  // P buffer b free (PV j-2 done)
      }
      // P = exp2(x - m) -> bf16 pairs into TMEM buffer b (A operand of PV)
      uint32_t pk[T / 2];
#pragma unroll
      for (int i = 0; i < T; i += 2) {
        const float p0 = ex2(sv[i] - m), p1 = ex2(sv[i + 1] - m);
        l += p0 + p1;
        pk[i >> 1] = pack2(p0, p1);
      }
      tmem_st_32x32b_x32(tP0 + b * 64 + lane_off, pk);
      tmem_st_32x32b_x32(tP0 + b * 64 + lane_off + 32, pk + 32);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full + b);
    }
    // epilogue: O / l once the last PV (and therefore all) completed
    mbar_wait(o_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1);
    tc_fence_after();
    // every lane loads (tcgen05.ld is warp-collective); rows >= s skip the store
    const bool valid = qrow < a.s;
    const float inv = 1.f / l;
    bf16* orow = reinterpret_cast<bf16*>(a.o) + (int64_t)(valid ? qrow : 0) * a.ldo + (int64_t)h * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tO + lane_off + c * 32, v);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          u.x = pack2(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv);
          u.y = pack2(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv);
          u.z = pack2(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv);
          u.w = pack2(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = u;
        }
      }
    }
    if (valid) a.lse[(int64_t)h * a.s + qrow] = (m + log2f(l)) * 0.69314718055994530942f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}



// Forward, version 3: 8 softmax warps (two per row: warp w covers TMEM lanes
// 32(w%4).. and S columns 64*half..), the softmax scale folded into one FFMA
// per element (p = ex2(s*scale_log2 - m)), masking only on the diagonal /
// ragged tile, P in TMEM (ts-mode PV), two K/V stages.  The two halves of a
// row exchange their partial max through shared memory once per tile.
constexpr int FWD3_THREADS = 384;
constexpr int SMEM_BYTES_V3 = 1024 + 5 * TILE_BYTES + 3 * 2 * T * 4 + 256;

template <bool POLY>
__global__ void __launch_bounds__(FWD3_THREADS, 1)
    attn_fwd_sm100_v3(const __grid_constant__ CUtensorMap tm_qkv, const FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;      // [2]
  uint8_t* sV = smem + 3 * TILE_BYTES;  // [2]
  float* smax = reinterpret_cast<float*>(smem + 5 * TILE_BYTES);  // [2 tiles][2 halves][T]
  float* ssum = smax + 4 * T;                                      // [2 halves][T]
  uint64_t* bar = reinterpret_cast<uint64_t*>(ssum + 2 * T);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;   // [2]
  uint64_t* s_empty = bar + 11; // [2]
  uint64_t* p_full = bar + 13;  // [2]
  uint64_t* o_done = bar + 15;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = gridDim.x;
  const int qt = nqt - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = qt + 1;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 256);
      mbar_init(p_full + i, 256);
      mbar_init(o_done + i, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem, tS0 = tmem + 128, tP0 = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, q_full, qcol, qt * T);
      tma_load_2d(sQ + ATOM, &tm_qkv, q_full, qcol + 64, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait_wd(k_empty + b, ph ^ 1, 301, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(k_full + b, TILE_BYTES);
        tma_load_2d(sK + b * TILE_BYTES, &tm_qkv, k_full + b, kcol, j * T);
        tma_load_2d(sK + b * TILE_BYTES + ATOM, &tm_qkv, k_full + b, kcol + 64, j * T);
        mbar_wait_wd(v_empty + b, ph ^ 1, 302, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(v_full + b, TILE_BYTES);
        tma_load_2d(sV + b * TILE_BYTES, &tm_qkv, v_full + b, vcol, j * T);
        tma_load_2d(sV + b * TILE_BYTES + ATOM, &tm_qkv, v_full + b, vcol + 64, j * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_bf16(T, T, false, false);
      constexpr uint32_t idO = make_idesc_bf16(T, D, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait_wd(q_full, 0, 303, a.s, a.nq, (int)blockIdx.y);
      auto issue_pv = [&](int jj) {
        const int b = jj & 1;
        mbar_wait_wd(p_full + b, (jj >> 1) & 1, 304, a.s, a.nq, (int)blockIdx.y);
        mbar_wait_wd(v_full + b, (jj >> 1) & 1, 305, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)
          mma_f16_ts(tO, tP0 + b * 64 + kk * 8, make_sw128_desc(v_addr + kk * 2048, ATOM, 1024), idO,
                     (jj > 0 || kk > 0) ? 1u : 0u);
        mma_commit(v_empty + b);
        mma_commit(o_done + b);
      };
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait_wd(k_full + b, ph, 306, a.s, a.nq, (int)blockIdx.y);
        mbar_wait_wd(s_empty + b, ph ^ 1, 307, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tS0 + b * 128, make_sw128_desc(q_addr + off, 16, 1024), make_sw128_desc(k_addr + off, 16, 1024),
                     idS, kk > 0 ? 1u : 0u);
        }
        mma_commit(k_empty + b);
        mma_commit(s_full + b);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_kv - 1);
    }
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2;          // S / O columns [64*half, 64*half + 64)
    const int quad = warp & 3;                 // TMEM lanes 32*quad ..
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int qrow = qt * T + r;
    const float sl2 = a.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      mbar_wait_wd(s_full + b, (j >> 1) & 1, 308, a.s, a.nq, (int)blockIdx.y);
      tc_fence_after();
      uint32_t u[64];
      tmem_ld_32x32b_x32(tS0 + b * 128 + half * 64 + lane_off, u);
      tmem_ld_32x32b_x32(tS0 + b * 128 + half * 64 + 32 + lane_off, u + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_empty + b);
      float sv[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) sv[i] = __uint_as_float(u[i]);
      const int cbase = j * T + half * 64;
      if (j == qt || cbase + 64 > a.s) {  // diagonal or ragged tile: causal / length mask
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (cbase + i > qrow || cbase + i >= a.s) sv[i] = -INFINITY;
      }
      float mx = fmax3(sv[0], sv[1], sv[2]);
#pragma unroll
      for (int i = 3; i < 63; i += 2) mx = fmax3(mx, sv[i], sv[i + 1]);
      mx = fmaxf(mx, sv[63]);
      smax[(b * 2 + half) * T + r] = mx;
      named_bar(2, 256);
      mx = fmaxf(smax[(b * 2) * T + r], smax[(b * 2 + 1) * T + r]) * sl2;
      const bool need = mx > m + 8.f;
      if (__any_sync(0xffffffffu, need)) {
        float alpha = 1.f;
        if (need) {
          alpha = (m == -INFINITY) ? 0.f : ex2(m - mx);
          l *= alpha;
          m = mx;
        }
        if (j > 0) {
          mbar_wait_wd(o_done + ((j - 1) & 1), ((j - 1) >> 1) & 1, 309, a.s, a.nq, (int)blockIdx.y);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t v[32];
            const uint32_t ta = tO + half * 64 + c * 32 + lane_off;
            tmem_ld_32x32b_x32(ta, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(ta, v);
          }
          tmem_wait_st();
        }
      } else if (j >= 2) {
        mbar_wait_wd(o_done + b, ((j - 2) >> 1) & 1, 310, a.s, a.nq, (int)blockIdx.y);
      }
      const float nm = -m;
      const uint64_t sc2 = pk2f(sl2, sl2), nm2 = pk2f(nm, nm);
      uint64_t lacc = pk2f(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        float t0, t1;
        up2f(ffma2(pk2f(sv[i], sv[i + 1]), sc2, nm2), t0, t1);
        const float p0 = ex2(t0);
        const float p1 = POLY ? ex2_fma(t1) : ex2(t1);
        lacc = fadd2(lacc, pk2f(p0, p1));
        u[i >> 1] = pack2(p0, p1);
      }
      {
        float l0, l1;
        up2f(lacc, l0, l1);
        l += l0 + l1;
      }
      tmem_st_32x32b_x32(tP0 + b * 64 + half * 32 + lane_off, u);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full + b);
    }
    ssum[half * T + r] = l;
    named_bar(2, 256);
    const float lt = ssum[r] + ssum[T + r];
    mbar_wait_wd(o_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1, 311, a.s, a.nq, (int)blockIdx.y);
    tc_fence_after();
    const bool valid = qrow < a.s;
    const float inv = 1.f / lt;
    bf16* orow = reinterpret_cast<bf16*>(a.o) + (int64_t)(valid ? qrow : 0) * a.ldo + (int64_t)h * D + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tO + half * 64 + c * 32 + lane_off, v);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 q;
          q.x = pack2(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv);
          q.y = pack2(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv);
          q.z = pack2(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv);
          q.w = pack2(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = q;
        }
      }
    }
    if (valid && half == 0) a.lse[(int64_t)h * a.s + qrow] = (m + log2f(lt)) * 0.69314718055994530942f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Forward, version 4: like v3 (8 softmax warps, two per row, 64 key columns
// each) but each half keeps its OWN running max / sum and its OWN O
// accumulator (O_0 | O_1 | S0 | S1 = 4 x 128 TMEM columns): no per-tile
// max exchange / 256-thread barrier between the halves; PV is two K = 64
// MMAs (half h: O_h += P_h V_j[64h .. 64h+63]); P_h is written over the
// S columns the same half just read.  The halves combine once at the end:
// m = max(m_0, m_1), O = sum_h O_h 2^(m_h - m), l = sum_h l_h 2^(m_h - m).
constexpr int SMEM_BYTES_V4 = 1024 + 5 * TILE_BYTES + 4 * T * 4 + 256;

__global__ void __launch_bounds__(FWD3_THREADS, 1)
    attn_fwd_sm100_v4(const __grid_constant__ CUtensorMap tm_qkv, const FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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
  const int nqt = gridDim.x;
  const int qt = nqt - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = qt + 1;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

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
      tma_load_2d(sQ, &tm_qkv, q_full, qcol, qt * T);
      tma_load_2d(sQ + ATOM, &tm_qkv, q_full, qcol + 64, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait_wd(k_empty + b, ph ^ 1, 321, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(k_full + b, TILE_BYTES);
        tma_load_2d(sK + b * TILE_BYTES, &tm_qkv, k_full + b, kcol, j * T);
        tma_load_2d(sK + b * TILE_BYTES + ATOM, &tm_qkv, k_full + b, kcol + 64, j * T);
        mbar_wait_wd(v_empty + b, ph ^ 1, 322, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(v_full + b, TILE_BYTES);
        tma_load_2d(sV + b * TILE_BYTES, &tm_qkv, v_full + b, vcol, j * T);
        tma_load_2d(sV + b * TILE_BYTES + ATOM, &tm_qkv, v_full + b, vcol + 64, j * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_bf16(T, T, false, false);
      constexpr uint32_t idO = make_idesc_bf16(T, D, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait_wd(q_full, 0, 323, a.s, a.nq, (int)blockIdx.y);
      auto issue_pv = [&](int jj) {
        const int b = jj & 1;
        mbar_wait_wd(v_full + b, (jj >> 1) & 1, 325, a.s, a.nq, (int)blockIdx.y);
        const uint32_t v_addr = smem_u32(sV + b * TILE_BYTES);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          mbar_wait_wd(p_full + b * 2 + hf, (jj >> 1) & 1, 324, a.s, a.nq, (int)blockIdx.y);
          tc_fence_after();
          // O_hf += P_hf (TMEM, keys 64hf..64hf+63: 32 packed columns) . V_j[64hf.., :]
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_f16_ts(tO + hf * 128, tS0 + b * 128 + hf * 64 + kk * 8,
                       make_sw128_desc(v_addr + (hf * 4 + kk) * 2048, ATOM, 1024), idO, (jj > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(v_empty + b);
        mma_commit(o_done + b);
      };
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait_wd(k_full + b, ph, 326, a.s, a.nq, (int)blockIdx.y);
        // buffer b last held P(j-2), consumed by PV(j-2), issued before this S(j) (in-order pipe)
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tS0 + b * 128, make_sw128_desc(q_addr + off, 16, 1024), make_sw128_desc(k_addr + off, 16, 1024),
                     idS, kk > 0 ? 1u : 0u);
        }
        mma_commit(k_empty + b);
        mma_commit(s_full + b);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_kv - 1);
    }
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
      mbar_wait_wd(s_full + b, (j >> 1) & 1, 328, a.s, a.nq, (int)blockIdx.y);
      tc_fence_after();
      uint32_t u[64];
      tmem_ld_32x32b_x32(tS0 + b * 128 + half * 64 + lane_off, u);
      tmem_ld_32x32b_x32(tS0 + b * 128 + half * 64 + 32 + lane_off, u + 32);
      tmem_wait_ld();
      float sv[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) sv[i] = __uint_as_float(u[i]);
      const int cbase = j * T + half * 64;
      if (j == qt || cbase + 64 > a.s) {  // diagonal or ragged tile: causal / length mask
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (cbase + i > qrow || cbase + i >= a.s) sv[i] = -INFINITY;
      }
      float mx = fmax3(sv[0], sv[1], sv[2]);
#pragma unroll
      for (int i = 3; i < 63; i += 2) mx = fmax3(mx, sv[i], sv[i + 1]);
      mx = fmaxf(mx, sv[63]) * sl2;
      const bool need = mx > m + 8.f;
      if (__any_sync(0xffffffffu, need)) {
        float alpha = 1.f;
        if (need) {
          alpha = (m == -INFINITY) ? 0.f : ex2(m - mx);
          l *= alpha;
          m = mx;
        }
        if (j > 0) {  // O_half holds PV(0..j-1): wait for PV(j-1), rescale all 128 columns
          mbar_wait_wd(o_done + ((j - 1) & 1), ((j - 1) >> 1) & 1, 329, a.s, a.nq, (int)blockIdx.y);
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
      uint64_t lacc = pk2f(0.f, 0.f);
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        float t0, t1;
        up2f(ffma2(pk2f(sv[i], sv[i + 1]), sc2, nm2), t0, t1);
        const float p0 = ex2(t0), p1 = ex2(t1);
        lacc = fadd2(lacc, pk2f(p0, p1));
        pk[i >> 1] = pack2(p0, p1);
      }
      {
        float l0, l1;
        up2f(lacc, l0, l1);
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
    named_bar(2, 256);
    const float m0 = sml[0 * T + r], l0 = sml[1 * T + r], m1 = sml[2 * T + r], l1 = sml[3 * T + r];
    const float mt = fmaxf(m0, m1);
    const float f0 = (m0 == -INFINITY) ? 0.f : ex2(m0 - mt), f1 = (m1 == -INFINITY) ? 0.f : ex2(m1 - mt);
    const float lt = l0 * f0 + l1 * f1;
    mbar_wait_wd(o_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1, 331, a.s, a.nq, (int)blockIdx.y);
    tc_fence_after();
    const bool valid = qrow < a.s;
    const float inv = 1.f / lt;
    const float c0 = f0 * inv, c1 = f1 * inv;
    bf16* orow = reinterpret_cast<bf16*>(a.o) + (int64_t)(valid ? qrow : 0) * a.ldo + (int64_t)h * D + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {  // this half writes output columns [64 half, 64 half + 64)
      uint32_t v0[32], v1[32];
      tmem_ld_32x32b_x32(tO + half * 64 + c * 32 + lane_off, v0);
      tmem_ld_32x32b_x32(tO + 128 + half * 64 + c * 32 + lane_off, v1);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
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

// ---------------------------------------------------------------- backward
// dQ kernel: one CTA per (query tile, head); loop over key tiles j <= i:
//   S = Q K_j^T, dP = dO V_j^T (TMEM), dS = P * (dP - D) (softmax warps,
//   bf16 -> smem), dQ += dS K_j (TMEM).  dQ = scale * dQ at the end.
constexpr int DQ_SMEM = 1024 + 7 * TILE_BYTES + 256;  // Q, dO, K[2], V[2], dS

struct BwdArgs {
  int s, nq, nkv;
  const float* lse;  // [nq, s] natural log
  const float* Dl;   // [nq, s]
  void* dq;          // bf16 [s, ldd] (q columns)
  int64_t ldd;
  float* dk_part;    // fp32 [nq, s, D]
  float* dv_part;    // fp32 [nq, s, D]
  float scale_log2, scale;
};


__global__ void __launch_bounds__(256, 1)
    attn_bwd_dq_sm100(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                      const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sdO = smem + TILE_BYTES;
  uint8_t* sK = smem + 2 * TILE_BYTES;  // [2]
  uint8_t* sV = smem + 4 * TILE_BYTES;  // [2]
  uint8_t* sdS = smem + 6 * TILE_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 7 * TILE_BYTES);
  uint64_t* qdo_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* sdp_full = bar + 9;
  uint64_t* sdp_empty = bar + 10;
  uint64_t* ds_full = bar + 11;
  uint64_t* dq_done = bar + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = qt + 1;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(qdo_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(sdp_empty, 128);
    mbar_init(ds_full, 128);
    mbar_init(dq_done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tQ = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qdo_full, 2 * TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, qdo_full, qcol, qt * T);
      tma_load_2d(sQ + ATOM, &tm_qkv, qdo_full, qcol + 64, qt * T);
      tma_load_2d(sdO, &tm_do, qdo_full, h * D, qt * T);
      tma_load_2d(sdO + ATOM, &tm_do, qdo_full, h * D + 64, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(k_empty + b, ph ^ 1);
        mbar_arrive_expect_tx(k_full + b, TILE_BYTES);
        tma_load_2d(sK + b * TILE_BYTES, &tm_qkv, k_full + b, kcol, j * T);
        tma_load_2d(sK + b * TILE_BYTES + ATOM, &tm_qkv, k_full + b, kcol + 64, j * T);
        mbar_wait(v_empty + b, ph ^ 1);
        mbar_arrive_expect_tx(v_full + b, TILE_BYTES);
        tma_load_2d(sV + b * TILE_BYTES, &tm_qkv, v_full + b, vcol, j * T);
        tma_load_2d(sV + b * TILE_BYTES + ATOM, &tm_qkv, v_full + b, vcol + 64, j * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idKK = make_idesc_bf16(T, T, false, false);  // S, dP: both operands K-major
      constexpr uint32_t idQ = make_idesc_bf16(T, D, false, true);    // dQ += dS K (K MN-major)
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sdO), ds_addr = smem_u32(sdS);
      mbar_wait(qdo_full, 0);
      auto issue_sdp = [&](int j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(k_full + b, ph);
        mbar_wait(v_full + b, ph);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES), v_addr = smem_u32(sV + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(q_addr + off, 16, 1024), make_sw128_desc(k_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(do_addr + off, 16, 1024), make_sw128_desc(v_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(v_empty + b);
        mma_commit(sdp_full);
      };
      issue_sdp(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {
          mbar_wait(sdp_empty, j & 1);  // softmax has read S/dP of tile j
          issue_sdp(j + 1);
        }
        mbar_wait(ds_full, j & 1);
        tc_fence_after();
        const int b = j & 1;
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          const uint64_t ad = make_sw128_desc(ds_addr + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = make_sw128_desc(k_addr + kk * 2048, ATOM, 1024);
          mma_f16_ss(tQ, ad, bd, idQ, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(k_empty + b);
        mma_commit(dq_done);
      }
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int qrow = qt * T + r;
    const bool vrow = qrow < a.s;
    const float lse2 = vrow ? a.lse[(int64_t)h * a.s + qrow] * 1.4426950408889634f : 0.f;
    const float Dv = vrow ? a.Dl[(int64_t)h * a.s + qrow] : 0.f;
    uint8_t* drow = sdS + (r >> 3) * 1024 + (r & 7) * 128;
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(sdp_full, j & 1);
      tc_fence_after();
      uint32_t pk[T / 2];
      const int kbase = j * T;
      const bool diag = (j == qt);
#pragma unroll
      for (int c = 0; c < T / 32; ++c) {
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(tS + lane_off + c * 32, sv);
        tmem_ld_32x32b_x32(tP + lane_off + c * 32, dv);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float d2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = kbase + c * 32 + i + e;
            float p = ex2(__uint_as_float(sv[i + e]) * a.scale_log2 - lse2);
            if ((diag && col > qrow) || col >= a.s || !vrow) p = 0.f;
            d2[e] = p * (__uint_as_float(dv[i + e]) - Dv);
          }
          pk[(c * 32 + i) >> 1] = pack2(d2[0], d2[1]);
        }
      }
      tc_fence_before();
      mbar_arrive(sdp_empty);
      if (j > 0) mbar_wait(dq_done, (j - 1) & 1);  // previous dQ MMA done reading dS smem
#pragma unroll
      for (int c = 0; c < T / 8; ++c) {
        uint4 u = make_uint4(pk[c * 4], pk[c * 4 + 1], pk[c * 4 + 2], pk[c * 4 + 3]);
        const int atom = c >> 3, ch = c & 7;
        *reinterpret_cast<uint4*>(drow + atom * ATOM + ((ch ^ (r & 7)) << 4)) = u;
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(dq_done, (n_kv - 1) & 1);
    tc_fence_after();
    bf16* orow = reinterpret_cast<bf16*>(a.dq) + (int64_t)(vrow ? qrow : 0) * a.ldd + (int64_t)h * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tQ + lane_off + c * 32, v);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          u.x = pack2(__uint_as_float(v[i]) * a.scale, __uint_as_float(v[i + 1]) * a.scale);
          u.y = pack2(__uint_as_float(v[i + 2]) * a.scale, __uint_as_float(v[i + 3]) * a.scale);
          u.z = pack2(__uint_as_float(v[i + 4]) * a.scale, __uint_as_float(v[i + 5]) * a.scale);
          u.w = pack2(__uint_as_float(v[i + 6]) * a.scale, __uint_as_float(v[i + 7]) * a.scale);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = u;
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

// dQ kernel, version 2: dS double-buffered in TMEM (A operand of dQ += dS K).
constexpr int DQ2_SMEM = 1024 + 6 * TILE_BYTES + 256;

__global__ void __launch_bounds__(256, 1)
    attn_bwd_dq_sm100_v2(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                      const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sdO = smem + TILE_BYTES;
  uint8_t* sK = smem + 2 * TILE_BYTES;  // [2]
  uint8_t* sV = smem + 4 * TILE_BYTES;  // [2]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 6 * TILE_BYTES);
  uint64_t* qdo_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* sdp_full = bar + 9;
  uint64_t* sdp_empty = bar + 10;
  uint64_t* ds_full = bar + 11;   // [2]
  uint64_t* dq_done = bar + 13;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = qt + 1;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(qdo_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(sdp_empty, 128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(ds_full + i, 128);
      mbar_init(dq_done + i, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tQ = tmem + 256, tdS0 = tmem + 384;  // dS0 | dS1 (64 cols)

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qdo_full, 2 * TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, qdo_full, qcol, qt * T);
      tma_load_2d(sQ + ATOM, &tm_qkv, qdo_full, qcol + 64, qt * T);
      tma_load_2d(sdO, &tm_do, qdo_full, h * D, qt * T);
      tma_load_2d(sdO + ATOM, &tm_do, qdo_full, h * D + 64, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(k_empty + b, ph ^ 1);
        mbar_arrive_expect_tx(k_full + b, TILE_BYTES);
        tma_load_2d(sK + b * TILE_BYTES, &tm_qkv, k_full + b, kcol, j * T);
        tma_load_2d(sK + b * TILE_BYTES + ATOM, &tm_qkv, k_full + b, kcol + 64, j * T);
        mbar_wait(v_empty + b, ph ^ 1);
        mbar_arrive_expect_tx(v_full + b, TILE_BYTES);
        tma_load_2d(sV + b * TILE_BYTES, &tm_qkv, v_full + b, vcol, j * T);
        tma_load_2d(sV + b * TILE_BYTES + ATOM, &tm_qkv, v_full + b, vcol + 64, j * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idKK = make_idesc_bf16(T, T, false, false);  // S, dP: both operands K-major
      constexpr uint32_t idQ = make_idesc_bf16(T, D, false, true);    // dQ += dS K (K MN-major)
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sdO);
      mbar_wait(qdo_full, 0);
      auto issue_sdp = [&](int j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(k_full + b, ph);
        mbar_wait(v_full + b, ph);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES), v_addr = smem_u32(sV + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(q_addr + off, 16, 1024), make_sw128_desc(k_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(do_addr + off, 16, 1024), make_sw128_desc(v_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(v_empty + b);
        mma_commit(sdp_full);
      };
      issue_sdp(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {
          mbar_wait(sdp_empty, j & 1);  // softmax has read S/dP of tile j
          issue_sdp(j + 1);
        }
        const int b = j & 1;
        mbar_wait(ds_full + b, (j >> 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          const uint64_t bd = make_sw128_desc(k_addr + kk * 2048, ATOM, 1024);
          mma_f16_ts(tQ, tdS0 + b * 64 + kk * 8, bd, idQ, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(k_empty + b);
        mma_commit(dq_done + b);
      }
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int qrow = qt * T + r;
    const bool vrow = qrow < a.s;
    const float lse2 = vrow ? a.lse[(int64_t)h * a.s + qrow] * 1.4426950408889634f : 0.f;
    const float Dv = vrow ? a.Dl[(int64_t)h * a.s + qrow] : 0.f;
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(sdp_full, j & 1);
      tc_fence_after();
      uint32_t pk[T / 2];
      const int kbase = j * T;
      const bool diag = (j == qt);
#pragma unroll
      for (int c = 0; c < T / 32; ++c) {
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(tS + lane_off + c * 32, sv);
        tmem_ld_32x32b_x32(tP + lane_off + c * 32, dv);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float d2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = kbase + c * 32 + i + e;
            float p = ex2(__uint_as_float(sv[i + e]) * a.scale_log2 - lse2);
            if ((diag && col > qrow) || col >= a.s || !vrow) p = 0.f;
            d2[e] = p * (__uint_as_float(dv[i + e]) - Dv);
          }
          pk[(c * 32 + i) >> 1] = pack2(d2[0], d2[1]);
        }
      }
      tc_fence_before();
      mbar_arrive(sdp_empty);
      const int b = j & 1;
      if (j >= 2) mbar_wait(dq_done + b, ((j - 2) >> 1) & 1);  // dQ MMA of tile j-2 done reading dS buffer b
      tmem_st_32x32b_x32(tdS0 + b * 64 + lane_off, pk);
      tmem_st_32x32b_x32(tdS0 + b * 64 + lane_off + 32, pk + 32);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full + b);
    }
    mbar_wait(dq_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1);
    tc_fence_after();
    bf16* orow = reinterpret_cast<bf16*>(a.dq) + (int64_t)(vrow ? qrow : 0) * a.ldd + (int64_t)h * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tQ + lane_off + c * 32, v);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          u.x = pack2(__uint_as_float(v[i]) * a.scale, __uint_as_float(v[i + 1]) * a.scale);
          u.y = pack2(__uint_as_float(v[i + 2]) * a.scale, __uint_as_float(v[i + 3]) * a.scale);
          u.z = pack2(__uint_as_float(v[i + 4]) * a.scale, __uint_as_float(v[i + 5]) * a.scale);
          u.w = pack2(__uint_as_float(v[i + 6]) * a.scale, __uint_as_float(v[i + 7]) * a.scale);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = u;
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

// dK/dV kernel: one CTA per (key tile, query head); loop over query tiles
// i >= j: S^T = K Q_i^T, dP^T = V dO_i^T (TMEM); P^T, dS^T = P^T (dP^T - D)
// (bf16 -> smem, one thread per key row); dV += P^T dO_i, dK += dS^T Q_i
// (TMEM).  fp32 partials per query head; attn_bwd_reduce sums the group.
constexpr int KV_SMEM = 1024 + 6 * TILE_BYTES + 2 * T * 4 + 256;  // K, V, Q, dO, P^T, dS^T, lse/D tiles

__global__ void __launch_bounds__(256, 1)
    attn_bwd_dkdv_sm100(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                        const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE_BYTES;
  uint8_t* sQ = smem + 2 * TILE_BYTES;
  uint8_t* sdO = smem + 3 * TILE_BYTES;
  uint8_t* sP = smem + 4 * TILE_BYTES;
  uint8_t* sdS = smem + 5 * TILE_BYTES;
  float* s_lse = reinterpret_cast<float*>(smem + 6 * TILE_BYTES);
  float* s_D = s_lse + T;
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_D + T);
  uint64_t* kv_full = bar + 0;
  uint64_t* qdo_full = bar + 1;
  uint64_t* qdo_empty = bar + 2;
  uint64_t* sdp_full = bar + 3;
  uint64_t* sdp_empty = bar + 4;
  uint64_t* pds_full = bar + 5;
  uint64_t* pds_free = bar + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (a.s + T - 1) / T;
  const int kt = gridDim.x - 1 - blockIdx.x;  // key tile; low tiles (most query tiles) first
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_q = nt - kt;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(qdo_full, 1);
    mbar_init(qdo_empty, 1);
    mbar_init(sdp_full, 1);
    mbar_init(sdp_empty, 128);
    mbar_init(pds_full, 128);
    mbar_init(pds_free, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tdV = tmem, tdK = tmem + 128, tS = tmem + 256, tP = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE_BYTES);
      tma_load_2d(sK, &tm_qkv, kv_full, kcol, kt * T);
      tma_load_2d(sK + ATOM, &tm_qkv, kv_full, kcol + 64, kt * T);
      tma_load_2d(sV, &tm_qkv, kv_full, vcol, kt * T);
      tma_load_2d(sV + ATOM, &tm_qkv, kv_full, vcol + 64, kt * T);
      for (int it = 0; it < n_q; ++it) {
        const int qi = kt + it;
        mbar_wait(qdo_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(qdo_full, 2 * TILE_BYTES);
        tma_load_2d(sQ, &tm_qkv, qdo_full, qcol, qi * T);
        tma_load_2d(sQ + ATOM, &tm_qkv, qdo_full, qcol + 64, qi * T);
        tma_load_2d(sdO, &tm_do, qdo_full, h * D, qi * T);
        tma_load_2d(sdO + ATOM, &tm_do, qdo_full, h * D + 64, qi * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idKK = make_idesc_bf16(T, T, false, false);
      constexpr uint32_t idMN = make_idesc_bf16(T, D, false, true);
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV), q_addr = smem_u32(sQ), do_addr = smem_u32(sdO);
      const uint32_t p_addr = smem_u32(sP), ds_addr = smem_u32(sdS);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_q; ++it) {
        mbar_wait(qdo_full, it & 1);
        mbar_wait(sdp_empty, (it & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(k_addr + off, 16, 1024), make_sw128_desc(q_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(v_addr + off, 16, 1024), make_sw128_desc(do_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(sdp_full);
        mbar_wait(pds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {  // K dim = query rows of the tile
          const uint32_t aoff = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tdV, make_sw128_desc(p_addr + aoff, 16, 1024), make_sw128_desc(do_addr + kk * 2048, ATOM, 1024),
                     idMN, (it > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          const uint32_t aoff = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tdK, make_sw128_desc(ds_addr + aoff, 16, 1024), make_sw128_desc(q_addr + kk * 2048, ATOM, 1024),
                     idMN, (it > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(qdo_empty);
        mma_commit(pds_free);
      }
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;  // key row within the tile
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int krow = kt * T + r;
    const bool vrow = krow < a.s;
    uint8_t* prow = sP + (r >> 3) * 1024 + (r & 7) * 128;
    uint8_t* drow = sdS + (r >> 3) * 1024 + (r & 7) * 128;
    for (int it = 0; it < n_q; ++it) {
      const int qi = kt + it;
      const int qbase = qi * T;
      named_bar(1, 128);  // everyone is done reading the previous tile's lse / D
      {
        const int q = qbase + r;
        s_lse[r] = q < a.s ? a.lse[(int64_t)h * a.s + q] * 1.4426950408889634f : INFINITY;
        s_D[r] = q < a.s ? a.Dl[(int64_t)h * a.s + q] : 0.f;
      }
      named_bar(1, 128);
      mbar_wait(sdp_full, it & 1);
      tc_fence_after();
      uint32_t pp[T / 2], pd[T / 2];
      const bool diag = (qi == kt);
#pragma unroll
      for (int c = 0; c < T / 32; ++c) {
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(tS + lane_off + c * 32, sv);
        tmem_ld_32x32b_x32(tP + lane_off + c * 32, dv);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float p2[2], d2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int qc = c * 32 + i + e;
            float p = ex2(__uint_as_float(sv[i + e]) * a.scale_log2 - s_lse[qc]);
            if ((diag && qbase + qc < krow) || !vrow) p = 0.f;
            p2[e] = p;
            d2[e] = p * (__uint_as_float(dv[i + e]) - s_D[qc]);
          }
          pp[(c * 32 + i) >> 1] = pack2(p2[0], p2[1]);
          pd[(c * 32 + i) >> 1] = pack2(d2[0], d2[1]);
        }
      }
      tc_fence_before();
      mbar_arrive(sdp_empty);
      if (it > 0) mbar_wait(pds_free, (it - 1) & 1);
#pragma unroll
      for (int c = 0; c < T / 8; ++c) {
        const int atom = c >> 3, ch = c & 7;
        const int off = atom * ATOM + ((ch ^ (r & 7)) << 4);
        *reinterpret_cast<uint4*>(prow + off) = make_uint4(pp[c * 4], pp[c * 4 + 1], pp[c * 4 + 2], pp[c * 4 + 3]);
        *reinterpret_cast<uint4*>(drow + off) = make_uint4(pd[c * 4], pd[c * 4 + 1], pd[c * 4 + 2], pd[c * 4 + 3]);
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(pds_full);
    }
    mbar_wait(pds_free, (n_q - 1) & 1);
    tc_fence_after();
    float* kr = a.dk_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D;
    float* vr = a.dv_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32], k[32];
      tmem_ld_32x32b_x32(tdV + lane_off + c * 32, v);
      tmem_ld_32x32b_x32(tdK + lane_off + c * 32, k);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          *reinterpret_cast<float4*>(vr + c * 32 + i) =
              make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                          __uint_as_float(v[i + 3]));
          *reinterpret_cast<float4*>(kr + c * 32 + i) =
              make_float4(__uint_as_float(k[i]) * a.scale, __uint_as_float(k[i + 1]) * a.scale,
                          __uint_as_float(k[i + 2]) * a.scale, __uint_as_float(k[i + 3]) * a.scale);
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


// dK/dV kernel, version 2: P^T and dS^T stay in TMEM (written over the S^T /
// dP^T accumulators once read) and feed tcgen05.mma as the A operand, so the
// freed shared memory double-buffers Q_i / dO_i: the loads of tile i+1
// overlap the MMAs and softmax of tile i.  Relies on tcgen05.mma executing
// in issue order (dV/dK of tile i read P^T/dS^T before S^T/dP^T of tile i+1
// overwrite them).
constexpr int KV2_SMEM = 1024 + 6 * TILE_BYTES + 4 * T * 4 + 256;  // K, V, Q[2], dO[2], lse/D[2]

__global__ void __launch_bounds__(256, 1)
    attn_bwd_dkdv_sm100_v2(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                           const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE_BYTES;
  uint8_t* sQ = smem + 2 * TILE_BYTES;   // [2]
  uint8_t* sdO = smem + 4 * TILE_BYTES;  // [2]
  float* s_lse = reinterpret_cast<float*>(smem + 6 * TILE_BYTES);  // [2][T]
  float* s_D = s_lse + 2 * T;                                       // [2][T]
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_D + 2 * T);
  uint64_t* kv_full = bar + 0;
  uint64_t* qdo_full = bar + 1;   // [2]
  uint64_t* qdo_empty = bar + 3;  // [2]
  uint64_t* sdp_full = bar + 5;
  uint64_t* pds_full = bar + 6;
  uint64_t* done = bar + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (a.s + T - 1) / T;
  const int kt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_q = nt - kt;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(qdo_full + i, 1);
      mbar_init(qdo_empty + i, 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(pds_full, 128);
    mbar_init(done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tdV = tmem, tdK = tmem + 128, tS = tmem + 256, tP = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE_BYTES);
      tma_load_2d(sK, &tm_qkv, kv_full, kcol, kt * T);
      tma_load_2d(sK + ATOM, &tm_qkv, kv_full, kcol + 64, kt * T);
      tma_load_2d(sV, &tm_qkv, kv_full, vcol, kt * T);
      tma_load_2d(sV + ATOM, &tm_qkv, kv_full, vcol + 64, kt * T);
      for (int it = 0; it < n_q; ++it) {
        const int b = it & 1, qi = kt + it;
        mbar_wait(qdo_empty + b, ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(qdo_full + b, 2 * TILE_BYTES);
        uint8_t* q = sQ + b * TILE_BYTES;
        uint8_t* o = sdO + b * TILE_BYTES;
        tma_load_2d(q, &tm_qkv, qdo_full + b, qcol, qi * T);
        tma_load_2d(q + ATOM, &tm_qkv, qdo_full + b, qcol + 64, qi * T);
        tma_load_2d(o, &tm_do, qdo_full + b, h * D, qi * T);
        tma_load_2d(o + ATOM, &tm_do, qdo_full + b, h * D + 64, qi * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idKK = make_idesc_bf16(T, T, false, false);
      constexpr uint32_t idMN = make_idesc_bf16(T, D, false, true);
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_q; ++it) {
        const int b = it & 1;
        const uint32_t q_addr = smem_u32(sQ + b * TILE_BYTES), do_addr = smem_u32(sdO + b * TILE_BYTES);
        mbar_wait(qdo_full + b, (it >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(k_addr + off, 16, 1024), make_sw128_desc(q_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(v_addr + off, 16, 1024), make_sw128_desc(do_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(sdp_full);
        mbar_wait(pds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)  // dV += P^T dO_i   (P^T from TMEM, 8 columns per k16)
          mma_f16_ts(tdV, tS + kk * 8, make_sw128_desc(do_addr + kk * 2048, ATOM, 1024), idMN,
                     (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)  // dK += dS^T Q_i
          mma_f16_ts(tdK, tP + kk * 8, make_sw128_desc(q_addr + kk * 2048, ATOM, 1024), idMN,
                     (it > 0 || kk > 0) ? 1u : 0u);
        mma_commit(qdo_empty + b);
      }
      mma_commit(done);
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int krow = kt * T + r;
    const bool vrow = krow < a.s;
    for (int it = 0; it < n_q; ++it) {
      const int b = it & 1, qi = kt + it;
      const int qbase = qi * T;
      {
        const int q = qbase + r;
        s_lse[b * T + r] = q < a.s ? a.lse[(int64_t)h * a.s + q] * 1.4426950408889634f : INFINITY;
        s_D[b * T + r] = q < a.s ? a.Dl[(int64_t)h * a.s + q] : 0.f;
      }
      named_bar(1, 128);
      const float* lse_t = s_lse + b * T;
      const float* D_t = s_D + b * T;
      mbar_wait(sdp_full, it & 1);
      tc_fence_after();
      uint32_t pp[T / 2], pd[T / 2];
      const bool diag = (qi == kt);
#pragma unroll
      for (int c = 0; c < T / 32; ++c) {
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(tS + lane_off + c * 32, sv);
        tmem_ld_32x32b_x32(tP + lane_off + c * 32, dv);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float p2[2], d2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int qc = c * 32 + i + e;
            float p = ex2(__uint_as_float(sv[i + e]) * a.scale_log2 - lse_t[qc]);
            if ((diag && qbase + qc < krow) || !vrow) p = 0.f;
            p2[e] = p;
            d2[e] = p * (__uint_as_float(dv[i + e]) - D_t[qc]);
          }
          pp[(c * 32 + i) >> 1] = pack2(p2[0], p2[1]);
          pd[(c * 32 + i) >> 1] = pack2(d2[0], d2[1]);
        }
      }
      // P^T over the S^T columns, dS^T over the dP^T columns (bf16 pairs)
      tmem_st_32x32b_x32(tS + lane_off, pp);
      tmem_st_32x32b_x32(tS + lane_off + 32, pp + 32);
      tmem_st_32x32b_x32(tP + lane_off, pd);
      tmem_st_32x32b_x32(tP + lane_off + 32, pd + 32);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(pds_full);
    }
    mbar_wait(done, 0);
    tc_fence_after();
    float* kr = a.dk_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D;
    float* vr = a.dv_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32], k[32];
      tmem_ld_32x32b_x32(tdV + lane_off + c * 32, v);
      tmem_ld_32x32b_x32(tdK + lane_off + c * 32, k);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          *reinterpret_cast<float4*>(vr + c * 32 + i) =
              make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                          __uint_as_float(v[i + 3]));
          *reinterpret_cast<float4*>(kr + c * 32 + i) =
              make_float4(__uint_as_float(k[i]) * a.scale, __uint_as_float(k[i + 1]) * a.scale,
                          __uint_as_float(k[i + 2]) * a.scale, __uint_as_float(k[i + 3]) * a.scale);
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

// Backward version 3: dQ and dK/dV kernels with 8 softmax warps (two per
// row, 64 columns each), FFMA-folded exponent, masking only on edge tiles.
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_sm100_v3(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                      const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sdO = smem + TILE_BYTES;
  uint8_t* sK = smem + 2 * TILE_BYTES;  // [2]
  uint8_t* sV = smem + 4 * TILE_BYTES;  // [2]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 6 * TILE_BYTES);
  uint64_t* qdo_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* sdp_full = bar + 9;
  uint64_t* sdp_empty = bar + 10;
  uint64_t* ds_full = bar + 11;   // [2]
  uint64_t* dq_done = bar + 13;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = qt + 1;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(qdo_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(sdp_empty, 256);
    for (int i = 0; i < 2; ++i) {
      mbar_init(ds_full + i, 256);
      mbar_init(dq_done + i, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tQ = tmem + 256, tdS0 = tmem + 384;  // dS0 | dS1 (64 cols)

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qdo_full, 2 * TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, qdo_full, qcol, qt * T);
      tma_load_2d(sQ + ATOM, &tm_qkv, qdo_full, qcol + 64, qt * T);
      tma_load_2d(sdO, &tm_do, qdo_full, h * D, qt * T);
      tma_load_2d(sdO + ATOM, &tm_do, qdo_full, h * D + 64, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait_wd(k_empty + b, ph ^ 1, 201, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(k_full + b, TILE_BYTES);
        tma_load_2d(sK + b * TILE_BYTES, &tm_qkv, k_full + b, kcol, j * T);
        tma_load_2d(sK + b * TILE_BYTES + ATOM, &tm_qkv, k_full + b, kcol + 64, j * T);
        mbar_wait_wd(v_empty + b, ph ^ 1, 202, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(v_full + b, TILE_BYTES);
        tma_load_2d(sV + b * TILE_BYTES, &tm_qkv, v_full + b, vcol, j * T);
        tma_load_2d(sV + b * TILE_BYTES + ATOM, &tm_qkv, v_full + b, vcol + 64, j * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idKK = make_idesc_bf16(T, T, false, false);  // S, dP: both operands K-major
      constexpr uint32_t idQ = make_idesc_bf16(T, D, false, true);    // dQ += dS K (K MN-major)
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sdO);
      mbar_wait_wd(qdo_full, 0, 203, a.s, a.nq, (int)blockIdx.y);
      auto issue_sdp = [&](int j) {
        const int b = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait_wd(k_full + b, ph, 204, a.s, a.nq, (int)blockIdx.y);
        mbar_wait_wd(v_full + b, ph, 205, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES), v_addr = smem_u32(sV + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(q_addr + off, 16, 1024), make_sw128_desc(k_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(do_addr + off, 16, 1024), make_sw128_desc(v_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(v_empty + b);
        mma_commit(sdp_full);
      };
      issue_sdp(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {
          mbar_wait_wd(sdp_empty, j & 1, 206, a.s, a.nq, (int)blockIdx.y);  // softmax has read S/dP of tile j
          issue_sdp(j + 1);
        }
        const int b = j & 1;
        mbar_wait_wd(ds_full + b, (j >> 1) & 1, 207, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          const uint64_t bd = make_sw128_desc(k_addr + kk * 2048, ATOM, 1024);
          mma_f16_ts(tQ, tdS0 + b * 64 + kk * 8, bd, idQ, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(k_empty + b);
        mma_commit(dq_done + b);
      }
    }
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int qrow = qt * T + r;
    const bool vrow = qrow < a.s;
    const float nlse2 = vrow ? -a.lse[(int64_t)h * a.s + qrow] * 1.4426950408889634f : 0.f;
    const float Dv = vrow ? a.Dl[(int64_t)h * a.s + qrow] : 0.f;
    const float sl2 = a.scale_log2;
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait_wd(sdp_full, j & 1, 208, a.s, a.nq, (int)blockIdx.y);
      tc_fence_after();
      uint32_t sv[64], dv[64];
      tmem_ld_32x32b_x32(tS + half * 64 + lane_off, sv);
      tmem_ld_32x32b_x32(tS + half * 64 + 32 + lane_off, sv + 32);
      tmem_ld_32x32b_x32(tP + half * 64 + lane_off, dv);
      tmem_ld_32x32b_x32(tP + half * 64 + 32 + lane_off, dv + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(sdp_empty);
      const int cbase = j * T + half * 64;
      const bool edge = (j == qt) || cbase + 64 > a.s || !vrow;
      uint32_t pk[32];
      const uint64_t sc2 = pk2f(sl2, sl2), nl2 = pk2f(nlse2, nlse2), D2 = pk2f(Dv, Dv);
#pragma unroll
      for (int i = 0; i < 64; i += 2) {  // packed fp32 pairs (FFMA2 / FADD2 / FMUL2)
        float t0, t1;
        up2f(ffma2(pk2f(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), sc2, nl2), t0, t1);
        float p0 = ex2(t0), p1 = ex2(t1);
        if (edge) {
          if (cbase + i > qrow || cbase + i >= a.s || !vrow) p0 = 0.f;
          if (cbase + i + 1 > qrow || cbase + i + 1 >= a.s || !vrow) p1 = 0.f;
        }
        float d0, d1;
        up2f(fmul2(pk2f(p0, p1), fsub2(pk2f(__uint_as_float(dv[i]), __uint_as_float(dv[i + 1])), D2)), d0, d1);
        pk[i >> 1] = pack2(d0, d1);
      }
      const int b = j & 1;
      if (j >= 2) mbar_wait_wd(dq_done + b, ((j - 2) >> 1) & 1, 209, a.s, a.nq, (int)blockIdx.y);
      tmem_st_32x32b_x32(tdS0 + b * 64 + half * 32 + lane_off, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full + b);
    }
    mbar_wait_wd(dq_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1, 210, a.s, a.nq, (int)blockIdx.y);
    tc_fence_after();
    bf16* orow = reinterpret_cast<bf16*>(a.dq) + (int64_t)(vrow ? qrow : 0) * a.ldd + (int64_t)h * D + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tQ + half * 64 + c * 32 + lane_off, v);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          u.x = pack2(__uint_as_float(v[i]) * a.scale, __uint_as_float(v[i + 1]) * a.scale);
          u.y = pack2(__uint_as_float(v[i + 2]) * a.scale, __uint_as_float(v[i + 3]) * a.scale);
          u.z = pack2(__uint_as_float(v[i + 4]) * a.scale, __uint_as_float(v[i + 5]) * a.scale);
          u.w = pack2(__uint_as_float(v[i + 6]) * a.scale, __uint_as_float(v[i + 7]) * a.scale);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = u;
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

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_sm100_v3(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                           const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE_BYTES;
  uint8_t* sQ = smem + 2 * TILE_BYTES;   // [2]
  uint8_t* sdO = smem + 4 * TILE_BYTES;  // [2]
  float* s_lse = reinterpret_cast<float*>(smem + 6 * TILE_BYTES);  // [2][T]
  float* s_D = s_lse + 2 * T;                                       // [2][T]
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_D + 2 * T);
  uint64_t* kv_full = bar + 0;
  uint64_t* qdo_full = bar + 1;   // [2]
  uint64_t* qdo_empty = bar + 3;  // [2]
  uint64_t* sdp_full = bar + 5;
  uint64_t* pds_full = bar + 6;
  uint64_t* done = bar + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (a.s + T - 1) / T;
  const int kt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_q = nt - kt;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(qdo_full + i, 1);
      mbar_init(qdo_empty + i, 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(pds_full, 256);
    mbar_init(done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tdV = tmem, tdK = tmem + 128, tS = tmem + 256, tP = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE_BYTES);
      tma_load_2d(sK, &tm_qkv, kv_full, kcol, kt * T);
      tma_load_2d(sK + ATOM, &tm_qkv, kv_full, kcol + 64, kt * T);
      tma_load_2d(sV, &tm_qkv, kv_full, vcol, kt * T);
      tma_load_2d(sV + ATOM, &tm_qkv, kv_full, vcol + 64, kt * T);
      for (int it = 0; it < n_q; ++it) {
        const int b = it & 1, qi = kt + it;
        mbar_wait_wd(qdo_empty + b, ((it >> 1) & 1) ^ 1, 211, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(qdo_full + b, 2 * TILE_BYTES);
        uint8_t* q = sQ + b * TILE_BYTES;
        uint8_t* o = sdO + b * TILE_BYTES;
        tma_load_2d(q, &tm_qkv, qdo_full + b, qcol, qi * T);
        tma_load_2d(q + ATOM, &tm_qkv, qdo_full + b, qcol + 64, qi * T);
        tma_load_2d(o, &tm_do, qdo_full + b, h * D, qi * T);
        tma_load_2d(o + ATOM, &tm_do, qdo_full + b, h * D + 64, qi * T);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idKK = make_idesc_bf16(T, T, false, false);
      constexpr uint32_t idMN = make_idesc_bf16(T, D, false, true);
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV);
      mbar_wait_wd(kv_full, 0, 212, a.s, a.nq, (int)blockIdx.y);
      for (int it = 0; it < n_q; ++it) {
        const int b = it & 1;
        const uint32_t q_addr = smem_u32(sQ + b * TILE_BYTES), do_addr = smem_u32(sdO + b * TILE_BYTES);
        mbar_wait_wd(qdo_full + b, (it >> 1) & 1, 213, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(k_addr + off, 16, 1024), make_sw128_desc(q_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(v_addr + off, 16, 1024), make_sw128_desc(do_addr + off, 16, 1024), idKK,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(sdp_full);
        mbar_wait_wd(pds_full, it & 1, 214, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)  // dV += P^T dO_i   (P^T from TMEM, 8 columns per k16)
          mma_f16_ts(tdV, tS + kk * 8, make_sw128_desc(do_addr + kk * 2048, ATOM, 1024), idMN,
                     (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)  // dK += dS^T Q_i
          mma_f16_ts(tdK, tP + kk * 8, make_sw128_desc(q_addr + kk * 2048, ATOM, 1024), idMN,
                     (it > 0 || kk > 0) ? 1u : 0u);
        mma_commit(qdo_empty + b);
      }
      mma_commit(done);
    }
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;           // key row
    const int tid = threadIdx.x - 128;        // 0..255
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int krow = kt * T + r;
    const bool vrow = krow < a.s;
    const float sl2 = a.scale_log2;
    for (int it = 0; it < n_q; ++it) {
      const int b = it & 1, qi = kt + it;
      const int qbase = qi * T;
      {  // threads 0-127 stage -lse*log2e, threads 128-255 stage D, for the 128 query rows
        const int q = qbase + (tid & 127);
        if (tid < 128) s_lse[b * T + tid] = q < a.s ? -a.lse[(int64_t)h * a.s + q] * 1.4426950408889634f : -INFINITY;
        else s_D[b * T + tid - 128] = q < a.s ? a.Dl[(int64_t)h * a.s + q] : 0.f;
      }
      named_bar(1, 256);
      const float* nl = s_lse + b * T + half * 64;
      const float* Dq = s_D + b * T + half * 64;
      mbar_wait_wd(sdp_full, it & 1, 215, a.s, a.nq, (int)blockIdx.y);
      tc_fence_after();
      uint32_t sv[64], dv[64];
      tmem_ld_32x32b_x32(tS + half * 64 + lane_off, sv);
      tmem_ld_32x32b_x32(tS + half * 64 + 32 + lane_off, sv + 32);
      tmem_ld_32x32b_x32(tP + half * 64 + lane_off, dv);
      tmem_ld_32x32b_x32(tP + half * 64 + 32 + lane_off, dv + 32);
      tmem_wait_ld();
      const bool diag = (qi == kt);
      uint32_t pp[32], pd[32];
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        const float4 l4 = *reinterpret_cast<const float4*>(nl + i);
        const float4 d4 = *reinterpret_cast<const float4*>(Dq + i);
        const float la[4] = {l4.x, l4.y, l4.z, l4.w}, da[4] = {d4.x, d4.y, d4.z, d4.w};
        float p[4], d[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          p[e] = ex2(fmaf(__uint_as_float(sv[i + e]), sl2, la[e]));
          if (diag && qbase + half * 64 + i + e < krow) p[e] = 0.f;
          d[e] = p[e] * (__uint_as_float(dv[i + e]) - da[e]);
        }
        if (!vrow) p[0] = p[1] = p[2] = p[3] = d[0] = d[1] = d[2] = d[3] = 0.f;
        pp[i >> 1] = pack2(p[0], p[1]);
        pp[(i >> 1) + 1] = pack2(p[2], p[3]);
        pd[i >> 1] = pack2(d[0], d[1]);
        pd[(i >> 1) + 1] = pack2(d[2], d[3]);
      }
      // P^T over the S^T columns, dS^T over the dP^T columns (bf16 pairs)
      tmem_st_32x32b_x32(tS + half * 32 + lane_off, pp);
      tmem_st_32x32b_x32(tP + half * 32 + lane_off, pd);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(pds_full);
    }
    mbar_wait_wd(done, 0, 216, a.s, a.nq, (int)blockIdx.y);
    tc_fence_after();
    float* kr = a.dk_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D + half * 64;
    float* vr = a.dv_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32], k[32];
      tmem_ld_32x32b_x32(tdV + half * 64 + c * 32 + lane_off, v);
      tmem_ld_32x32b_x32(tdK + half * 64 + c * 32 + lane_off, k);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          *reinterpret_cast<float4*>(vr + c * 32 + i) =
              make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                          __uint_as_float(v[i + 3]));
          *reinterpret_cast<float4*>(kr + c * 32 + i) =
              make_float4(__uint_as_float(k[i]) * a.scale, __uint_as_float(k[i + 1]) * a.scale,
                          __uint_as_float(k[i + 2]) * a.scale, __uint_as_float(k[i + 3]) * a.scale);
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

// dK/dV kernel, version 4: query tiles of 64 rows so that S^T / dP^T are
// DOUBLE-BUFFERED in TMEM (dV 128 | dK 128 | S0 64 | dP0 64 | S1 64 | dP1 64
// columns): the MMA warp issues S^T/dP^T of tile i+1 before waiting for the
// softmax warps' P^T/dS^T of tile i, so the tensor pipe computes tile i+1
// (and then dV/dK of tile i) while the softmax warps work on tile i.  In v3
// the single S/dP buffer serialises the two.  Q_i / dO_i: 4-stage TMA ring of
// 64-row tiles.  tcgen05.mma executes in issue order, so S^T(i+2) (issued
// after dV/dK(i)) cannot overwrite P^T/dS^T(i) before they are consumed.
constexpr int QT = 64;                          // query rows per tile
constexpr int QT_BYTES = QT * D * 2;            // 16 KB
constexpr int QATOM = QT * 64 * 2;              // 8 KB
constexpr int KV4_STAGES = 4;
constexpr int KV4_SMEM = 1024 + 2 * TILE_BYTES + 2 * KV4_STAGES * QT_BYTES + 4 * QT * 4 + 256;
constexpr int KV5_SMEM = 1024 + 2 * TILE_BYTES + 2 * KV4_STAGES * QT_BYTES + 8 * QT * 4 + 256;

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_sm100_v4(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q64,
                           const __grid_constant__ CUtensorMap tm_do64, const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE_BYTES;
  uint8_t* sQ = smem + 2 * TILE_BYTES;                          // [STAGES]
  uint8_t* sdO = sQ + KV4_STAGES * QT_BYTES;                    // [STAGES]
  float* s_lse = reinterpret_cast<float*>(sdO + KV4_STAGES * QT_BYTES);  // [2][QT]
  float* s_D = s_lse + 2 * QT;                                           // [2][QT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_D + 2 * QT);
  uint64_t* kv_full = bar + 0;
  uint64_t* qdo_full = bar + 1;                  // [STAGES]
  uint64_t* qdo_empty = bar + 1 + KV4_STAGES;    // [STAGES]
  uint64_t* sdp_full = bar + 1 + 2 * KV4_STAGES;  // [2]
  uint64_t* pds_full = sdp_full + 2;              // [2]
  uint64_t* done = pds_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (a.s + T - 1) / T;
  const int nq64 = (a.s + QT - 1) / QT;
  const int kt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int q0 = 2 * kt;           // first query tile that sees this key tile
  const int n_q = nq64 - q0;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;
  (void)nt;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < KV4_STAGES; ++i) {
      mbar_init(qdo_full + i, 1);
      mbar_init(qdo_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(sdp_full + i, 1);
      mbar_init(pds_full + i, 256);
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
  const uint32_t tdV = tmem, tdK = tmem + 128, tSP = tmem + 256;  // buffer b: S at tSP + 128b, dP at +64

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE_BYTES);
      tma_load_2d(sK, &tm_kv, kv_full, kcol, kt * T);
      tma_load_2d(sK + ATOM, &tm_kv, kv_full, kcol + 64, kt * T);
      tma_load_2d(sV, &tm_kv, kv_full, vcol, kt * T);
      tma_load_2d(sV + ATOM, &tm_kv, kv_full, vcol + 64, kt * T);
      for (int it = 0; it < n_q; ++it) {
        const int st = it % KV4_STAGES, qi = q0 + it;
        mbar_wait_wd(qdo_empty + st, ((it / KV4_STAGES) & 1) ^ 1, 217, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(qdo_full + st, 2 * QT_BYTES);
        uint8_t* q = sQ + st * QT_BYTES;
        uint8_t* o = sdO + st * QT_BYTES;
        tma_load_2d(q, &tm_q64, qdo_full + st, qcol, qi * QT);
        tma_load_2d(q + QATOM, &tm_q64, qdo_full + st, qcol + 64, qi * QT);
        tma_load_2d(o, &tm_do64, qdo_full + st, h * D, qi * QT);
        tma_load_2d(o + QATOM, &tm_do64, qdo_full + st, h * D + 64, qi * QT);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_bf16(T, QT, false, false);  // S^T, dP^T: M = 128 keys, N = 64 queries
      constexpr uint32_t idMN = make_idesc_bf16(T, D, false, true);   // dV, dK: N = d, B (dO_i, Q_i) MN-major
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV);
      mbar_wait_wd(kv_full, 0, 218, a.s, a.nq, (int)blockIdx.y);
      auto issue_sdp = [&](int it) {
        const int st = it % KV4_STAGES, b = it & 1;
        const uint32_t q_addr = smem_u32(sQ + st * QT_BYTES), do_addr = smem_u32(sdO + st * QT_BYTES);
        mbar_wait_wd(qdo_full + st, (it / KV4_STAGES) & 1, 219, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
        const uint32_t tS = tSP + b * 128, tP = tS + 64;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ka = (kk >> 2) * ATOM + (kk & 3) * 32, qa = (kk >> 2) * QATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(k_addr + ka, 16, 1024), make_sw128_desc(q_addr + qa, 16, 1024), idS,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ka = (kk >> 2) * ATOM + (kk & 3) * 32, qa = (kk >> 2) * QATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(v_addr + ka, 16, 1024), make_sw128_desc(do_addr + qa, 16, 1024), idS,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(sdp_full + b);
      };
      issue_sdp(0);
      for (int it = 0; it < n_q; ++it) {
        if (it + 1 < n_q) issue_sdp(it + 1);
        const int st = it % KV4_STAGES, b = it & 1;
        const uint32_t q_addr = smem_u32(sQ + st * QT_BYTES), do_addr = smem_u32(sdO + st * QT_BYTES);
        const uint32_t tS = tSP + b * 128, tP = tS + 64;
        mbar_wait_wd(pds_full + b, (it >> 1) & 1, 220, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)  // dV += P^T dO_i   (P^T from TMEM, 8 columns per k16)
          mma_f16_ts(tdV, tS + kk * 8, make_sw128_desc(do_addr + kk * 2048, QATOM, 1024), idMN,
                     (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)  // dK += dS^T Q_i
          mma_f16_ts(tdK, tP + kk * 8, make_sw128_desc(q_addr + kk * 2048, QATOM, 1024), idMN,
                     (it > 0 || kk > 0) ? 1u : 0u);
        mma_commit(qdo_empty + st);
      }
      mma_commit(done);
    }
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2, quad = warp & 3;  // half: query columns [32 half, 32 half + 32)
    const int r = quad * 32 + lane;                     // key row
    const int tid = threadIdx.x - 128;                  // 0..255
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int krow = kt * T + r;
    const bool vrow = krow < a.s;
    const float sl2 = a.scale_log2;
    for (int it = 0; it < n_q; ++it) {
      const int b = it & 1, qi = q0 + it;
      const int qbase = qi * QT;
      if (tid < 2 * QT) {  // threads 0-63 stage -lse*log2e, 64-127 stage D, for the 64 query rows
        const int q = qbase + (tid & (QT - 1));
        if (tid < QT) s_lse[b * QT + tid] = q < a.s ? -a.lse[(int64_t)h * a.s + q] * 1.4426950408889634f : -INFINITY;
        else s_D[b * QT + tid - QT] = q < a.s ? a.Dl[(int64_t)h * a.s + q] : 0.f;
      }
      named_bar(1, 256);
      const float* nl = s_lse + b * QT + half * 32;
      const float* Dq = s_D + b * QT + half * 32;
      const uint32_t tS = tSP + b * 128, tP = tS + 64;
      mbar_wait_wd(sdp_full + b, (it >> 1) & 1, 221, a.s, a.nq, (int)blockIdx.y);
      tc_fence_after();
      uint32_t sv[32], dv[32];
      tmem_ld_32x32b_x32(tS + half * 32 + lane_off, sv);
      tmem_ld_32x32b_x32(tP + half * 32 + lane_off, dv);
      tmem_wait_ld();
      const bool diag = qbase < krow + 1 && it < 2;  // tiles overlapping the key tile need the causal mask
      uint32_t pp[16], pd[16];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 l4 = *reinterpret_cast<const float4*>(nl + i);
        const float4 d4 = *reinterpret_cast<const float4*>(Dq + i);
        const float la[4] = {l4.x, l4.y, l4.z, l4.w}, da[4] = {d4.x, d4.y, d4.z, d4.w};
        float p[4], d[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          p[e] = ex2(fmaf(__uint_as_float(sv[i + e]), sl2, la[e]));
          if (diag && qbase + half * 32 + i + e < krow) p[e] = 0.f;
          d[e] = p[e] * (__uint_as_float(dv[i + e]) - da[e]);
        }
        if (!vrow) p[0] = p[1] = p[2] = p[3] = d[0] = d[1] = d[2] = d[3] = 0.f;
        pp[i >> 1] = pack2(p[0], p[1]);
        pp[(i >> 1) + 1] = pack2(p[2], p[3]);
        pd[i >> 1] = pack2(d[0], d[1]);
        pd[(i >> 1) + 1] = pack2(d[2], d[3]);
      }
      // P^T over the S^T columns, dS^T over the dP^T columns (bf16 pairs)
      tmem_st_32x32b_x16(tS + half * 16 + lane_off, pp);
      tmem_st_32x32b_x16(tP + half * 16 + lane_off, pd);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(pds_full + b);
    }
    mbar_wait_wd(done, 0, 222, a.s, a.nq, (int)blockIdx.y);
    tc_fence_after();
    float* kr = a.dk_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D + half * 64;
    float* vr = a.dv_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32], k[32];
      tmem_ld_32x32b_x32(tdV + half * 64 + c * 32 + lane_off, v);
      tmem_ld_32x32b_x32(tdK + half * 64 + c * 32 + lane_off, k);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          *reinterpret_cast<float4*>(vr + c * 32 + i) =
              make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                          __uint_as_float(v[i + 3]));
          *reinterpret_cast<float4*>(kr + c * 32 + i) =
              make_float4(__uint_as_float(k[i]) * a.scale, __uint_as_float(k[i + 1]) * a.scale,
                          __uint_as_float(k[i + 2]) * a.scale, __uint_as_float(k[i + 3]) * a.scale);
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

// dK/dV kernel, version 5: v4 with ping-pong softmax warp groups (one key row
// per thread, alternate query tiles per group).
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_sm100_v5(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q64,
                           const __grid_constant__ CUtensorMap tm_do64, const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE_BYTES;
  uint8_t* sQ = smem + 2 * TILE_BYTES;                          // [STAGES]
  uint8_t* sdO = sQ + KV4_STAGES * QT_BYTES;                    // [STAGES]
  // per warp group, double-buffered by (it >> 1) & 1: a group's threads sync only
  // at their own per-tile barrier, so a fast thread may stage tile it + 2 while a
  // slow one still reads tile it's rows
  float* s_lse = reinterpret_cast<float*>(sdO + KV4_STAGES * QT_BYTES);  // [2 groups][2][QT]
  float* s_D = s_lse + 4 * QT;                                           // [2 groups][2][QT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_D + 4 * QT);
  uint64_t* kv_full = bar + 0;
  uint64_t* qdo_full = bar + 1;                  // [STAGES]
  uint64_t* qdo_empty = bar + 1 + KV4_STAGES;    // [STAGES]
  uint64_t* sdp_full = bar + 1 + 2 * KV4_STAGES;  // [2]
  uint64_t* pds_full = sdp_full + 2;              // [2]
  uint64_t* done = pds_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (a.s + T - 1) / T;
  const int nq64 = (a.s + QT - 1) / QT;
  const int kt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int q0 = 2 * kt;           // first query tile that sees this key tile
  const int n_q = nq64 - q0;
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;
  (void)nt;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < KV4_STAGES; ++i) {
      mbar_init(qdo_full + i, 1);
      mbar_init(qdo_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(sdp_full + i, 1);
      mbar_init(pds_full + i, 128);
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
  const uint32_t tdV = tmem, tdK = tmem + 128, tSP = tmem + 256;  // buffer b: S at tSP + 128b, dP at +64

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE_BYTES);
      tma_load_2d(sK, &tm_kv, kv_full, kcol, kt * T);
      tma_load_2d(sK + ATOM, &tm_kv, kv_full, kcol + 64, kt * T);
      tma_load_2d(sV, &tm_kv, kv_full, vcol, kt * T);
      tma_load_2d(sV + ATOM, &tm_kv, kv_full, vcol + 64, kt * T);
      for (int it = 0; it < n_q; ++it) {
        const int st = it % KV4_STAGES, qi = q0 + it;
        mbar_wait_wd(qdo_empty + st, ((it / KV4_STAGES) & 1) ^ 1, 217, a.s, a.nq, (int)blockIdx.y);
        mbar_arrive_expect_tx(qdo_full + st, 2 * QT_BYTES);
        uint8_t* q = sQ + st * QT_BYTES;
        uint8_t* o = sdO + st * QT_BYTES;
        tma_load_2d(q, &tm_q64, qdo_full + st, qcol, qi * QT);
        tma_load_2d(q + QATOM, &tm_q64, qdo_full + st, qcol + 64, qi * QT);
        tma_load_2d(o, &tm_do64, qdo_full + st, h * D, qi * QT);
        tma_load_2d(o + QATOM, &tm_do64, qdo_full + st, h * D + 64, qi * QT);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_bf16(T, QT, false, false);  // S^T, dP^T: M = 128 keys, N = 64 queries
      constexpr uint32_t idMN = make_idesc_bf16(T, D, false, true);   // dV, dK: N = d, B (dO_i, Q_i) MN-major
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV);
      mbar_wait_wd(kv_full, 0, 218, a.s, a.nq, (int)blockIdx.y);
      auto issue_sdp = [&](int it) {
        const int st = it % KV4_STAGES, b = it & 1;
        const uint32_t q_addr = smem_u32(sQ + st * QT_BYTES), do_addr = smem_u32(sdO + st * QT_BYTES);
        mbar_wait_wd(qdo_full + st, (it / KV4_STAGES) & 1, 219, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
        const uint32_t tS = tSP + b * 128, tP = tS + 64;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ka = (kk >> 2) * ATOM + (kk & 3) * 32, qa = (kk >> 2) * QATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(k_addr + ka, 16, 1024), make_sw128_desc(q_addr + qa, 16, 1024), idS,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ka = (kk >> 2) * ATOM + (kk & 3) * 32, qa = (kk >> 2) * QATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(v_addr + ka, 16, 1024), make_sw128_desc(do_addr + qa, 16, 1024), idS,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(sdp_full + b);
      };
      issue_sdp(0);
      for (int it = 0; it < n_q; ++it) {
        if (it + 1 < n_q) issue_sdp(it + 1);
        const int st = it % KV4_STAGES, b = it & 1;
        const uint32_t q_addr = smem_u32(sQ + st * QT_BYTES), do_addr = smem_u32(sdO + st * QT_BYTES);
        const uint32_t tS = tSP + b * 128, tP = tS + 64;
        mbar_wait_wd(pds_full + b, (it >> 1) & 1, 220, a.s, a.nq, (int)blockIdx.y);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)  // dV += P^T dO_i   (P^T from TMEM, 8 columns per k16)
          mma_f16_ts(tdV, tS + kk * 8, make_sw128_desc(do_addr + kk * 2048, QATOM, 1024), idMN,
                     (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)  // dK += dS^T Q_i
          mma_f16_ts(tdK, tP + kk * 8, make_sw128_desc(q_addr + kk * 2048, QATOM, 1024), idMN,
                     (it > 0 || kk > 0) ? 1u : 0u);
        mma_commit(qdo_empty + st);
      }
      mma_commit(done);
    }
  } else if (warp >= 4) {
    // ping-pong: warp group grp (4 warps, one key row per thread) converts
    // the query tiles with it % 2 == grp, all 64 columns in two 32-column
    // chunks; the two groups run independently (own named barrier / lse-D
    // staging), so one group's TMEM / global-load latency hides behind the
    // other's work.
    const int grp = (warp - 4) >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;                     // key row
    const int gtid = threadIdx.x - 128 - grp * 128;     // 0..127 within the group
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int krow = kt * T + r;
    const bool vrow = krow < a.s;
    const float sl2 = a.scale_log2;
    for (int it = grp; it < n_q; it += 2) {
      const int b = it & 1, qi = q0 + it;
      const int qbase = qi * QT;
      const int sb = grp * 2 + ((it >> 1) & 1);  // this group's staging buffer for tile it
      {  // threads 0-63 of the group stage -lse*log2e, 64-127 stage D, for the 64 query rows
        const int q = qbase + (gtid & (QT - 1));
        if (gtid < QT) s_lse[sb * QT + gtid] = q < a.s ? -a.lse[(int64_t)h * a.s + q] * 1.4426950408889634f : -INFINITY;
        else s_D[sb * QT + gtid - QT] = q < a.s ? a.Dl[(int64_t)h * a.s + q] : 0.f;
      }
      named_bar(1 + grp, 128);
      const uint32_t tS = tSP + b * 128, tP = tS + 64;
      mbar_wait_wd(sdp_full + b, (it >> 1) & 1, 251, a.s, a.nq, h);
      tc_fence_after();
      const bool diag = it < 2;  // tiles overlapping the key tile need the causal mask
#pragma unroll 1
      for (int ch = 0; ch < 2; ++ch) {
        const float* nl = s_lse + sb * QT + ch * 32;
        const float* Dq = s_D + sb * QT + ch * 32;
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(tS + ch * 32 + lane_off, sv);
        tmem_ld_32x32b_x32(tP + ch * 32 + lane_off, dv);
        tmem_wait_ld();
        uint32_t pp[16], pd[16];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(nl + i);
          const float4 d4 = *reinterpret_cast<const float4*>(Dq + i);
          float pv[4], dd[4];
          const uint64_t sc2 = pk2f(sl2, sl2);
#pragma unroll
          for (int e = 0; e < 4; e += 2) {  // packed fp32 pairs (FFMA2 / FADD2 / FMUL2)
            const uint64_t la2 = e ? pk2f(l4.z, l4.w) : pk2f(l4.x, l4.y);
            const uint64_t da2 = e ? pk2f(d4.z, d4.w) : pk2f(d4.x, d4.y);
            float t0, t1;
            up2f(ffma2(pk2f(__uint_as_float(sv[i + e]), __uint_as_float(sv[i + e + 1])), sc2, la2), t0, t1);
            pv[e] = ex2(t0);
            pv[e + 1] = ex2(t1);
            if (diag) {
              if (qbase + ch * 32 + i + e < krow) pv[e] = 0.f;
              if (qbase + ch * 32 + i + e + 1 < krow) pv[e + 1] = 0.f;
            }
            up2f(fmul2(pk2f(pv[e], pv[e + 1]),
                       fsub2(pk2f(__uint_as_float(dv[i + e]), __uint_as_float(dv[i + e + 1])), da2)),
                 dd[e], dd[e + 1]);
          }
          if (!vrow) pv[0] = pv[1] = pv[2] = pv[3] = dd[0] = dd[1] = dd[2] = dd[3] = 0.f;
          pp[i >> 1] = pack2(pv[0], pv[1]);
          pp[(i >> 1) + 1] = pack2(pv[2], pv[3]);
          pd[i >> 1] = pack2(dd[0], dd[1]);
          pd[(i >> 1) + 1] = pack2(dd[2], dd[3]);
        }
        // P^T / dS^T (bf16 pairs) over columns [16 ch, 16 ch + 16) of S^T / dP^T:
        // chunk 1 reads S^T columns 32-63, which chunk 0's stores do not touch
        tmem_st_32x32b_x16(tS + ch * 16 + lane_off, pp);
        tmem_st_32x32b_x16(tP + ch * 16 + lane_off, pd);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(pds_full + b);
    }
    const int half = grp;
    mbar_wait_wd(done, 0, 222, a.s, a.nq, (int)blockIdx.y);
    tc_fence_after();
    float* kr = a.dk_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D + half * 64;
    float* vr = a.dv_part + ((int64_t)h * a.s + (vrow ? krow : 0)) * D + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32], k[32];
      tmem_ld_32x32b_x32(tdV + half * 64 + c * 32 + lane_off, v);
      tmem_ld_32x32b_x32(tdK + half * 64 + c * 32 + lane_off, k);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          *reinterpret_cast<float4*>(vr + c * 32 + i) =
              make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                          __uint_as_float(v[i + 3]));
          *reinterpret_cast<float4*>(kr + c * 32 + i) =
              make_float4(__uint_as_float(k[i]) * a.scale, __uint_as_float(k[i + 1]) * a.scale,
                          __uint_as_float(k[i + 2]) * a.scale, __uint_as_float(k[i + 3]) * a.scale);
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

// dQ kernel, version 4: key tiles of 64 rows so that S / dP are
// DOUBLE-BUFFERED in TMEM (dQ 128 | S0 64 | dP0 64 | S1 64 | dP1 64 | dS0 32 |
// dS1 32 columns): the MMA warp issues S/dP of tile j+1 as soon as the
// softmax warps have read buffer (j+1)&1 (tile j-1), so the tensor pipe
// computes the next tile while the softmax warps convert this one.  K_j / V_j:
// 4-stage TMA ring of 64-row tiles.
constexpr int DQ4_STAGES = 4;
constexpr int DQ4_SMEM = 1024 + 2 * TILE_BYTES + 2 * DQ4_STAGES * QT_BYTES + 256;

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_sm100_v4(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_kv64,
                         const __grid_constant__ CUtensorMap tm_do, const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sdO = smem + TILE_BYTES;
  uint8_t* sK = smem + 2 * TILE_BYTES;            // [STAGES] 64-row tiles
  uint8_t* sV = sK + DQ4_STAGES * QT_BYTES;       // [STAGES]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + DQ4_STAGES * QT_BYTES);
  uint64_t* qdo_full = bar + 0;
  uint64_t* kv_full = bar + 1;                    // [STAGES]
  uint64_t* kv_empty = kv_full + DQ4_STAGES;      // [STAGES]
  uint64_t* sdp_full = kv_empty + DQ4_STAGES;     // [2]
  uint64_t* sdp_empty = sdp_full + 2;             // [2]
  uint64_t* ds_full = sdp_empty + 2;              // [2]
  uint64_t* dq_done = ds_full + 2;                // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = 2 * (qt + 1);  // 64-row key tiles with keys <= the tile's last query row
  const int qcol = h * D, kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(qdo_full, 1);
    for (int i = 0; i < DQ4_STAGES; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(sdp_full + i, 1);
      mbar_init(sdp_empty + i, 256);
      mbar_init(ds_full + i, 256);
      mbar_init(dq_done + i, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_kv64);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tQ = tmem, tSP = tmem + 128, tdS = tmem + 384;  // buffer b: S at tSP + 128b, dP at +64; dS at tdS + 32b

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qdo_full, 2 * TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, qdo_full, qcol, qt * T);
      tma_load_2d(sQ + ATOM, &tm_qkv, qdo_full, qcol + 64, qt * T);
      tma_load_2d(sdO, &tm_do, qdo_full, h * D, qt * T);
      tma_load_2d(sdO + ATOM, &tm_do, qdo_full, h * D + 64, qt * T);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % DQ4_STAGES;
        mbar_wait_wd(kv_empty + st, ((j / DQ4_STAGES) & 1) ^ 1, 401, a.s, a.nq, h);
        mbar_arrive_expect_tx(kv_full + st, 2 * QT_BYTES);
        uint8_t* k = sK + st * QT_BYTES;
        uint8_t* v = sV + st * QT_BYTES;
        tma_load_2d(k, &tm_kv64, kv_full + st, kcol, j * QT);
        tma_load_2d(k + QATOM, &tm_kv64, kv_full + st, kcol + 64, j * QT);
        tma_load_2d(v, &tm_kv64, kv_full + st, vcol, j * QT);
        tma_load_2d(v + QATOM, &tm_kv64, kv_full + st, vcol + 64, j * QT);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_bf16(T, QT, false, false);  // S, dP: M = 128 queries, N = 64 keys
      constexpr uint32_t idQ = make_idesc_bf16(T, D, false, true);    // dQ += dS K_j (K_j MN-major)
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sdO);
      mbar_wait_wd(qdo_full, 0, 402, a.s, a.nq, h);
      auto issue_sdp = [&](int j) {
        const int st = j % DQ4_STAGES, b = j & 1;
        mbar_wait_wd(kv_full + st, (j / DQ4_STAGES) & 1, 403, a.s, a.nq, h);
        if (j >= 2) mbar_wait_wd(sdp_empty + b, ((j - 2) >> 1) & 1, 404, a.s, a.nq, h);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * QT_BYTES), v_addr = smem_u32(sV + st * QT_BYTES);
        const uint32_t tS = tSP + b * 128, tP = tS + 64;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t qa = (kk >> 2) * ATOM + (kk & 3) * 32, ka = (kk >> 2) * QATOM + (kk & 3) * 32;
          mma_f16_ss(tS, make_sw128_desc(q_addr + qa, 16, 1024), make_sw128_desc(k_addr + ka, 16, 1024), idS,
                     kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t qa = (kk >> 2) * ATOM + (kk & 3) * 32, ka = (kk >> 2) * QATOM + (kk & 3) * 32;
          mma_f16_ss(tP, make_sw128_desc(do_addr + qa, 16, 1024), make_sw128_desc(v_addr + ka, 16, 1024), idS,
                     kk > 0 ? 1u : 0u);
        }
        mma_commit(sdp_full + b);
      };
      issue_sdp(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) issue_sdp(j + 1);
        const int st = j % DQ4_STAGES, b = j & 1;
        mbar_wait_wd(ds_full + b, (j >> 1) & 1, 405, a.s, a.nq, h);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * QT_BYTES);
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)  // dQ += dS K_j   (dS from TMEM, 8 columns per k16)
          mma_f16_ts(tQ, tdS + b * 32 + kk * 8, make_sw128_desc(k_addr + kk * 2048, QATOM, 1024), idQ,
                     (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(kv_empty + st);
        mma_commit(dq_done + b);
      }
    }
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2, quad = warp & 3;  // half: key columns [32 half, 32 half + 32) of the tile
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int qrow = qt * T + r;
    const bool vrow = qrow < a.s;
    const float nlse2 = vrow ? -a.lse[(int64_t)h * a.s + qrow] * 1.4426950408889634f : 0.f;
    const float Dv = vrow ? a.Dl[(int64_t)h * a.s + qrow] : 0.f;
    const float sl2 = a.scale_log2;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      const uint32_t tS = tSP + b * 128, tP = tS + 64;
      mbar_wait_wd(sdp_full + b, (j >> 1) & 1, 406, a.s, a.nq, h);
      tc_fence_after();
      uint32_t sv[32], dv[32];
      tmem_ld_32x32b_x32(tS + half * 32 + lane_off, sv);
      tmem_ld_32x32b_x32(tP + half * 32 + lane_off, dv);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(sdp_empty + b);
      const int cbase = j * QT + half * 32;
      const bool edge = j >= 2 * qt || cbase + 32 > a.s || !vrow;
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float d2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float p = ex2(fmaf(__uint_as_float(sv[i + e]), sl2, nlse2));
          if (edge && (cbase + i + e > qrow || cbase + i + e >= a.s || !vrow)) p = 0.f;
          d2[e] = p * (__uint_as_float(dv[i + e]) - Dv);
        }
        pk[i >> 1] = pack2(d2[0], d2[1]);
      }
      if (j >= 2) mbar_wait_wd(dq_done + b, ((j - 2) >> 1) & 1, 407, a.s, a.nq, h);
      tmem_st_32x32b_x16(tdS + b * 32 + half * 16 + lane_off, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full + b);
    }
    mbar_wait_wd(dq_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1, 408, a.s, a.nq, h);
    tc_fence_after();
    bf16* orow = reinterpret_cast<bf16*>(a.dq) + (int64_t)(vrow ? qrow : 0) * a.ldd + (int64_t)h * D + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tQ + half * 64 + c * 32 + lane_off, v);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          u.x = pack2(__uint_as_float(v[i]) * a.scale, __uint_as_float(v[i + 1]) * a.scale);
          u.y = pack2(__uint_as_float(v[i + 2]) * a.scale, __uint_as_float(v[i + 3]) * a.scale);
          u.z = pack2(__uint_as_float(v[i + 4]) * a.scale, __uint_as_float(v[i + 5]) * a.scale);
          u.w = pack2(__uint_as_float(v[i + 6]) * a.scale, __uint_as_float(v[i + 7]) * a.scale);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = u;
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

// dQ kernel, version 5: Q and dO live in TMEM (bf16 pairs, loaded once per
// CTA by the softmax warps) and feed S = Q K_j^T and dP = dO V_j^T as the A
// operand, so shared memory only streams the 64-row K_j / V_j tiles (the A
// operand was 2/3 of the smem operand traffic of those MMAs).  TMEM: dQ 128 |
// S 64 | dP 64 | dS[2] 2x32 | Q 64 | dO 64 = 448 columns; S/dP single-buffered
// (released as soon as the softmax warps have loaded them).
constexpr int DQ5_SMEM = 1024 + 2 * DQ4_STAGES * QT_BYTES + 256;

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_sm100_v5(const __grid_constant__ CUtensorMap tm_kv64, const BwdArgs a, const bf16* __restrict__ qkv,
                         int64_t ld, const bf16* __restrict__ dout, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;                             // [STAGES] 64-row tiles
  uint8_t* sV = sK + DQ4_STAGES * QT_BYTES;       // [STAGES]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + DQ4_STAGES * QT_BYTES);
  uint64_t* ops_ready = bar + 0;                  // Q / dO in TMEM (256 softmax threads)
  uint64_t* kv_full = bar + 1;                    // [STAGES]
  uint64_t* kv_empty = kv_full + DQ4_STAGES;      // [STAGES]
  uint64_t* sdp_full = kv_empty + DQ4_STAGES;
  uint64_t* sdp_empty = sdp_full + 1;
  uint64_t* ds_full = sdp_empty + 1;              // [2]
  uint64_t* dq_done = ds_full + 2;                // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y;
  const int grp = a.nq / a.nkv, g = h / grp;
  const int n_kv = 2 * (qt + 1);
  const int kcol = a.nq * D + g * D, vcol = (a.nq + a.nkv) * D + g * D;

  if (threadIdx.x == 0) {
    mbar_init(ops_ready, 256);
    for (int i = 0; i < DQ4_STAGES; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(sdp_empty, 256);
    for (int i = 0; i < 2; ++i) {
      mbar_init(ds_full + i, 256);
      mbar_init(dq_done + i, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm_kv64);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tQ = tmem, tS = tmem + 128, tP = tmem + 192, tdS = tmem + 256, tQa = tmem + 320, tdOa = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % DQ4_STAGES;
        mbar_wait_wd(kv_empty + st, ((j / DQ4_STAGES) & 1) ^ 1, 501, a.s, a.nq, h);
        mbar_arrive_expect_tx(kv_full + st, 2 * QT_BYTES);
        uint8_t* k = sK + st * QT_BYTES;
        uint8_t* v = sV + st * QT_BYTES;
        tma_load_2d(k, &tm_kv64, kv_full + st, kcol, j * QT);
        tma_load_2d(k + QATOM, &tm_kv64, kv_full + st, kcol + 64, j * QT);
        tma_load_2d(v, &tm_kv64, kv_full + st, vcol, j * QT);
        tma_load_2d(v + QATOM, &tm_kv64, kv_full + st, vcol + 64, j * QT);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = make_idesc_bf16(T, QT, false, false);  // S, dP: M = 128 queries, N = 64 keys
      constexpr uint32_t idQ = make_idesc_bf16(T, D, false, true);    // dQ += dS K_j (K_j MN-major)
      mbar_wait_wd(ops_ready, 0, 502, a.s, a.nq, h);
      tc_fence_after();
      auto issue_sdp = [&](int j) {
        const int st = j % DQ4_STAGES;
        mbar_wait_wd(kv_full + st, (j / DQ4_STAGES) & 1, 503, a.s, a.nq, h);
        if (j >= 1) mbar_wait_wd(sdp_empty, (j - 1) & 1, 504, a.s, a.nq, h);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * QT_BYTES), v_addr = smem_u32(sV + st * QT_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ka = (kk >> 2) * QATOM + (kk & 3) * 32;
          mma_f16_ts(tS, tQa + kk * 8, make_sw128_desc(k_addr + ka, 16, 1024), idS, kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ka = (kk >> 2) * QATOM + (kk & 3) * 32;
          mma_f16_ts(tP, tdOa + kk * 8, make_sw128_desc(v_addr + ka, 16, 1024), idS, kk > 0 ? 1u : 0u);
        }
        mma_commit(sdp_full);
      };
      issue_sdp(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) issue_sdp(j + 1);
        const int st = j % DQ4_STAGES, b = j & 1;
        mbar_wait_wd(ds_full + b, (j >> 1) & 1, 505, a.s, a.nq, h);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * QT_BYTES);
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)  // dQ += dS K_j   (dS from TMEM, 8 columns per k16)
          mma_f16_ts(tQ, tdS + b * 32 + kk * 8, make_sw128_desc(k_addr + kk * 2048, QATOM, 1024), idQ,
                     (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(kv_empty + st);
        mma_commit(dq_done + b);
      }
    }
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int qrow = qt * T + r;
    const bool vrow = qrow < a.s;
    {  // this row's half (64 of 128 d) of Q and dO -> TMEM (bf16 pairs: 32 columns each)
      uint32_t u[32];
      const uint4* qs = reinterpret_cast<const uint4*>(qkv + (int64_t)(vrow ? qrow : 0) * ld + (int64_t)h * D + half * 64);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint4 x = vrow ? qs[i] : make_uint4(0, 0, 0, 0);
        u[4 * i] = x.x; u[4 * i + 1] = x.y; u[4 * i + 2] = x.z; u[4 * i + 3] = x.w;
      }
      tmem_st_32x32b_x32(tQa + half * 32 + lane_off, u);
      const uint4* ds_ = reinterpret_cast<const uint4*>(dout + (int64_t)(vrow ? qrow : 0) * ldo + (int64_t)h * D + half * 64);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint4 x = vrow ? ds_[i] : make_uint4(0, 0, 0, 0);
        u[4 * i] = x.x; u[4 * i + 1] = x.y; u[4 * i + 2] = x.z; u[4 * i + 3] = x.w;
      }
      tmem_st_32x32b_x32(tdOa + half * 32 + lane_off, u);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ops_ready);
    }
    const float nlse2 = vrow ? -a.lse[(int64_t)h * a.s + qrow] * 1.4426950408889634f : 0.f;
    const float Dv = vrow ? a.Dl[(int64_t)h * a.s + qrow] : 0.f;
    const float sl2 = a.scale_log2;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      mbar_wait_wd(sdp_full, j & 1, 506, a.s, a.nq, h);
      tc_fence_after();
      uint32_t sv[32], dv[32];
      tmem_ld_32x32b_x32(tS + half * 32 + lane_off, sv);
      tmem_ld_32x32b_x32(tP + half * 32 + lane_off, dv);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(sdp_empty);
      const int cbase = j * QT + half * 32;
      const bool edge = j >= 2 * qt || cbase + 32 > a.s || !vrow;
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float d2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float p = ex2(fmaf(__uint_as_float(sv[i + e]), sl2, nlse2));
          if (edge && (cbase + i + e > qrow || cbase + i + e >= a.s || !vrow)) p = 0.f;
          d2[e] = p * (__uint_as_float(dv[i + e]) - Dv);
        }
        pk[i >> 1] = pack2(d2[0], d2[1]);
      }
      if (j >= 2) mbar_wait_wd(dq_done + b, ((j - 2) >> 1) & 1, 507, a.s, a.nq, h);
      tmem_st_32x32b_x16(tdS + b * 32 + half * 16 + lane_off, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full + b);
    }
    mbar_wait_wd(dq_done + ((n_kv - 1) & 1), ((n_kv - 1) >> 1) & 1, 508, a.s, a.nq, h);
    tc_fence_after();
    bf16* orow = reinterpret_cast<bf16*>(a.dq) + (int64_t)(vrow ? qrow : 0) * a.ldd + (int64_t)h * D + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tQ + half * 64 + c * 32 + lane_off, v);
      tmem_wait_ld();
      if (vrow) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u4;
          u4.x = pack2(__uint_as_float(v[i]) * a.scale, __uint_as_float(v[i + 1]) * a.scale);
          u4.y = pack2(__uint_as_float(v[i + 2]) * a.scale, __uint_as_float(v[i + 3]) * a.scale);
          u4.z = pack2(__uint_as_float(v[i + 4]) * a.scale, __uint_as_float(v[i + 5]) * a.scale);
          u4.w = pack2(__uint_as_float(v[i + 6]) * a.scale, __uint_as_float(v[i + 7]) * a.scale);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = u4;
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

// dk/dv (bf16, kv-head columns of dqkv) = sum over the group's query heads.
__global__ void attn_bwd_reduce(int s, int nq, int nkv, const float* __restrict__ dk_part,
                                const float* __restrict__ dv_part, bf16* dk, bf16* dv, int64_t ldd) {
  const int grp = nq / nkv;
  const int64_t total = (int64_t)s * nkv * (D / 4);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % (D / 4)) * 4;
    const int64_t t2 = i / (D / 4);
    const int g = (int)(t2 % nkv);
    const int64_t row = t2 / nkv;
    float4 sk = make_float4(0.f, 0.f, 0.f, 0.f), sv = sk;
    for (int hh = 0; hh < grp; ++hh) {
      const int64_t off = ((int64_t)(g * grp + hh) * s + row) * D + c4;
      const float4 a = *reinterpret_cast<const float4*>(dk_part + off);
      const float4 b = *reinterpret_cast<const float4*>(dv_part + off);
      sk.x += a.x; sk.y += a.y; sk.z += a.z; sk.w += a.w;
      sv.x += b.x; sv.y += b.y; sv.z += b.z; sv.w += b.w;
    }
    bf16* kd = dk + row * ldd + (int64_t)g * D + c4;
    bf16* vd = dv + row * ldd + (int64_t)g * D + c4;
    *reinterpret_cast<uint2*>(kd) = make_uint2(pack2(sk.x, sk.y), pack2(sk.z, sk.w));
    *reinterpret_cast<uint2*>(vd) = make_uint2(pack2(sv.x, sv.y), pack2(sv.z, sv.w));
  }
}

}  // namespace

// Tuning knob (stp_set_option "attn_fwd"): 1 = P via smem, 2 = P in TMEM.
int& attn_fwd_version_ref() {
  static int v = [] {
    const char* e = getenv("STP_ATTN_FWD");
    return e ? atoi(e) : 4;  // runtime.cpp kAttnFwdDefault
  }();
  return v;
}

// Used by attention.cu for d == 128, bf16.
stp_status attn_fwd_sm100_launch(int s, int nq, int nkv, const void* qkv_base, int64_t ld, void* o, int64_t ldo,
                                 float* lse, cudaStream_t st) {
  CUtensorMap tm;
  STP_TRY_STATUS(tensor_map_bf16(&tm, qkv_base, ld, s, ld, 64, T));
  static bool attr = false;
  if (!attr) {
    STP_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr = true;
  }
  FwdArgs a;
  a.s = s;
  a.nq = nq;
  a.nkv = nkv;
  a.ldo = ldo;
  a.o = o;
  a.lse = lse;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  dim3 grid((s + T - 1) / T, nq);
  if (attn_fwd_version_ref() == 4) {
    static bool attr4 = false;
    if (!attr4) {
      STP_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_sm100_v4, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES_V4));
      attr4 = true;
    }
    attn_fwd_sm100_v4<<<grid, FWD3_THREADS, SMEM_BYTES_V4, st>>>(tm, a);
  } else if (attn_fwd_version_ref() == 3 || attn_fwd_version_ref() == 5) {
    static bool attr3 = false;
    if (!attr3) {
      STP_CUDA_TRY(
          cudaFuncSetAttribute(attn_fwd_sm100_v3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES_V3));
      STP_CUDA_TRY(
          cudaFuncSetAttribute(attn_fwd_sm100_v3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES_V3));
      attr3 = true;
    }
    if (attn_fwd_version_ref() == 5) attn_fwd_sm100_v3<true><<<grid, FWD3_THREADS, SMEM_BYTES_V3, st>>>(tm, a);
    else attn_fwd_sm100_v3<false><<<grid, FWD3_THREADS, SMEM_BYTES_V3, st>>>(tm, a);
  } else if (attn_fwd_version_ref() == 2) {
    static bool attr2 = false;
    if (!attr2) {
      STP_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_sm100_v2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES_V2));
      attr2 = true;
    }
    attn_fwd_sm100_v2<<<grid, 256, SMEM_BYTES_V2, st>>>(tm, a);
  } else {
    attn_fwd_sm100<<<grid, 256, SMEM_BYTES, st>>>(tm, a);
  }
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

}  // namespace stp

namespace stp {
// Tuning knob (stp_set_option "attn_bwd"): 1 = smem P^T/dS^T dK/dV kernel,
// 2 = TMEM-resident P^T/dS^T with double-buffered Q/dO, 3 = 8 softmax warps,
// 4 = 64-row query tiles with double-buffered S^T/dP^T, 5 = v4 +
// the dQ kernel with 64-row key tiles and double-buffered S/dP, 6 = v4 + the
// dQ kernel with Q / dO as TMEM-resident A operands, 7 = v4 with ping-pong
// softmax warp groups in the dK/dV kernel + the v3 dQ kernel (default).
int& attn_bwd_version_ref() {
  static int v = [] {
    const char* e = getenv("STP_ATTN_BWD");
    return e ? atoi(e) : 7;  // runtime.cpp kAttnBwdDefault
  }();
  return v;
}
// dq/dk/dv for d == 128 bf16 with the fused [q | k | v] layout; ws: fp32
// [nq*s] D (already computed) followed by dk/dv partials [2, nq, s, 128].
stp_status attn_bwd_sm100_launch(int s, int nq, int nkv, const void* qkv_base, int64_t ld, const void* dout,
                                 int64_t ldo, const float* lse, const float* Dl, void* dq_base, int64_t ldd,
                                 float* part, cudaStream_t st) {
  CUtensorMap tq, td;
  STP_TRY(tensor_map_bf16(&tq, qkv_base, ld, s, ld, 64, T));
  STP_TRY(tensor_map_bf16(&td, dout, ldo, s, ldo, 64, T));
  static bool attr = false;
  if (!attr) {
    STP_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dq_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, DQ_SMEM));
    STP_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dkdv_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, KV_SMEM));
    STP_CUDA_TRY(
        cudaFuncSetAttribute(attn_bwd_dkdv_sm100_v2, cudaFuncAttributeMaxDynamicSharedMemorySize, KV2_SMEM));
    STP_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dq_sm100_v2, cudaFuncAttributeMaxDynamicSharedMemorySize, DQ2_SMEM));
    STP_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dq_sm100_v3, cudaFuncAttributeMaxDynamicSharedMemorySize, DQ2_SMEM));
    STP_CUDA_TRY(
        cudaFuncSetAttribute(attn_bwd_dkdv_sm100_v3, cudaFuncAttributeMaxDynamicSharedMemorySize, KV2_SMEM));
    attr = true;
  }
  BwdArgs a;
  a.s = s;
  a.nq = nq;
  a.nkv = nkv;
  a.lse = lse;
  a.Dl = Dl;
  a.dq = dq_base;
  a.ldd = ldd;
  a.dk_part = part;
  a.dv_part = part + (int64_t)nq * s * D;
  a.scale = 1.f / sqrtf((float)D);
  a.scale_log2 = 1.4426950408889634f * a.scale;
  const int nt = (s + T - 1) / T;
  if (attn_bwd_version_ref() >= 4) {
    const bool v5 = attn_bwd_version_ref() == 7;
    CUtensorMap tq64, td64;
    STP_TRY(tensor_map_bf16(&tq64, qkv_base, ld, s, ld, 64, QT));
    STP_TRY(tensor_map_bf16(&td64, dout, ldo, s, ldo, 64, QT));
    static bool attr4 = false;
    if (!attr4) {
      STP_CUDA_TRY(
          cudaFuncSetAttribute(attn_bwd_dkdv_sm100_v4, cudaFuncAttributeMaxDynamicSharedMemorySize, KV4_SMEM));
      attr4 = true;
    }
    static bool attr7 = false;
    if (v5 && !attr7) {
      STP_CUDA_TRY(
          cudaFuncSetAttribute(attn_bwd_dkdv_sm100_v5, cudaFuncAttributeMaxDynamicSharedMemorySize, KV5_SMEM));
      attr7 = true;
    }
    if (v5) attn_bwd_dkdv_sm100_v5<<<dim3(nt, nq), 384, KV5_SMEM, st>>>(tq, tq64, td64, a);
    else attn_bwd_dkdv_sm100_v4<<<dim3(nt, nq), 384, KV4_SMEM, st>>>(tq, tq64, td64, a);
  } else if (attn_bwd_version_ref() == 3) attn_bwd_dkdv_sm100_v3<<<dim3(nt, nq), 384, KV2_SMEM, st>>>(tq, td, a);
  else if (attn_bwd_version_ref() == 2) attn_bwd_dkdv_sm100_v2<<<dim3(nt, nq), 256, KV2_SMEM, st>>>(tq, td, a);
  else attn_bwd_dkdv_sm100<<<dim3(nt, nq), 256, KV_SMEM, st>>>(tq, td, a);
  count_launch();
  STP_LAUNCH_CHECK();
  if (attn_bwd_version_ref() == 6) {
    CUtensorMap tkv64;
    STP_TRY(tensor_map_bf16(&tkv64, qkv_base, ld, s, ld, 64, QT));
    static bool attr6 = false;
    if (!attr6) {
      STP_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dq_sm100_v5, cudaFuncAttributeMaxDynamicSharedMemorySize, DQ5_SMEM));
      attr6 = true;
    }
    attn_bwd_dq_sm100_v5<<<dim3(nt, nq), 384, DQ5_SMEM, st>>>(tkv64, a, (const bf16*)qkv_base, ld, (const bf16*)dout,
                                                              ldo);
  } else if (attn_bwd_version_ref() == 5) {
    CUtensorMap tkv64;
    STP_TRY(tensor_map_bf16(&tkv64, qkv_base, ld, s, ld, 64, QT));
    static bool attr5 = false;
    if (!attr5) {
      STP_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dq_sm100_v4, cudaFuncAttributeMaxDynamicSharedMemorySize, DQ4_SMEM));
      attr5 = true;
    }
    attn_bwd_dq_sm100_v4<<<dim3(nt, nq), 384, DQ4_SMEM, st>>>(tq, tkv64, td, a);
  } else if (attn_bwd_version_ref() >= 3) attn_bwd_dq_sm100_v3<<<dim3(nt, nq), 384, DQ2_SMEM, st>>>(tq, td, a);
  else if (attn_bwd_version_ref() == 2) attn_bwd_dq_sm100_v2<<<dim3(nt, nq), 256, DQ2_SMEM, st>>>(tq, td, a);
  else attn_bwd_dq_sm100<<<dim3(nt, nq), 256, DQ_SMEM, st>>>(tq, td, a);
  count_launch();
  STP_LAUNCH_CHECK();
  bf16* dk = reinterpret_cast<bf16*>(dq_base) + (int64_t)nq * D;
  bf16* dv = dk + (int64_t)nkv * D;
  const int64_t total = (int64_t)s * nkv * (D / 4);
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 16 * num_sms());
  attn_bwd_reduce<<<grid, 256, 0, st>>>(s, nq, nkv, a.dk_part, a.dv_part, dk, dv, ldd);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}
}  // namespace stp
