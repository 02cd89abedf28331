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
constexpr int SMEM_BYTES = 1024 + 6 * TILE_BYTES + 256;  // Q, K0, K1, V0, V1, P + barriers

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

__global__ void __launch_bounds__(256, 1)
    attn_fwd_sm100(const __grid_constant__ CUtensorMap tm_qkv, const FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;          // 2 buffers
  uint8_t* sV = smem + 3 * TILE_BYTES;      // 2 buffers
  uint8_t* sP = smem + 5 * TILE_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 6 * TILE_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;   // [2]
  uint64_t* s_empty = bar + 11; // [2]
  uint64_t* p_full = bar + 13;
  uint64_t* o_done = bar + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

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
    }
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
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
        mbar_wait(p_full, jj & 1);
        mbar_wait(v_full + b, (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + b * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          const uint64_t ad = make_sw128_desc(p_addr + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = make_sw128_desc(v_addr + kk * 2048, ATOM, 1024);
          mma_f16_ss(tO, ad, bd, idO, (jj > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(v_empty + b);
        mma_commit(o_done);
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
    uint8_t* prow = sP + (r >> 3) * 1024 + (r & 7) * 128;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      mbar_wait(s_full + b, (j >> 1) & 1);
      tc_fence_after();
      float sv[T];
#pragma unroll
      for (int c = 0; c < T / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tS0 + b * 128 + lane_off + c * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(v[i]);
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
      // P_{j-1} consumed and O stable before touching P smem / O
      if (j > 0) mbar_wait(o_done, (j - 1) & 1);
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
      }
      // P = exp2(x - m) -> bf16, K-major SW128 smem layout (two 64-col atoms)
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
      mbar_arrive(p_full);
    }
    // epilogue: O / l
    mbar_wait(o_done, (n_kv - 1) & 1);
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

}  // namespace

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
  attn_fwd_sm100<<<grid, 256, SMEM_BYTES, st>>>(tm, a);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

}  // namespace stp
