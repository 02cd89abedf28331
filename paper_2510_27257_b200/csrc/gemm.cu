// TP-sharded linear-layer GEMMs (the paper's
// Column/RowParallelLinear matmuls, Fig. 2).
//
// bf16: persistent warp-specialised tcgen05 kernel.  One CTA per SM, 256
// threads: warp 0 = TMA producer, warp 1 = MMA issuer (one elected lane),
// warp 2 = TMEM allocator, warps 4-7 = epilogue (TMEM -> registers ->
// global).  Tile 128 x BN x 64, BN in {128, 192, 256}, a ring of smem stages
// (128-byte swizzle, filled by TMA, released by tcgen05.commit), two TMEM
// accumulators so the epilogue of tile i overlaps the main loop of tile i+1;
// a 2-SM variant (cta_group::2, 256 x 256 tiles) for the large shapes.
// Operands may be K-major or MN-major (descriptor transpose bits) so forward
// (X W^T), dgrad (dY W) and wgrad (dY^T X) all run without transposes.
// The epilogue indexes the accumulator registers with compile-time indices
// only (a runtime index puts the chunk in local memory: DESIGN.md §7c).
//
// fp32: true-fp32 SIMT FMA GEMM (no TF32) for the fp32 parity mode.
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.h"
#include "prof.h"
#include "sm100.h"

namespace stp {

stp_status set_max_smem_once(const void* func, int bytes, unsigned long long* mask);
namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kSmemBudget = 192 * 1024;

struct GemmArgs {
  int* tile_ctr;  // dynamic tile scheduler counter (0 at launch; reset by the last fetch)
  int M, N, K;
  int num_m_blk, num_n_blk, num_k_blk;
  int n_fast;  // tile raster: 0 = m-block fastest (A re-swept per n-block), 1 = n-block fastest
  int epilogue;
  void* C;
  int64_t ldc;
  const void* bias;
  const void* R;
  int64_t ldr;
  // STP_EPI_STORE_CE (LM head): fp32 cross-entropy row statistics of the
  // accumulator before rounding, per 128-column block (ce_part [M][ce_nblk]
  // x (max, sum exp(z - max))) and the target logit (ce_tl [M])
  const int32_t* ce_tgt;
  int64_t ce_v0;
  float* ce_part;
  float* ce_tl;
  int ce_nblk;
  // push mode (STORE / BIAS epilogues): row m goes to push[m / push_rows] at
  // row push_off + m % push_rows -- the reduce-scatter of a row-parallel
  // GEMM's partial done by the epilogue's NVLink stores into each TP peer's
  // receive buffer (stp_gemm_push_targets)
  void* push[8];
  int64_t push_rows, push_off;
};

// Running (max, sum exp) of one row over 32 fp32 accumulator columns; the
// target logit is written by the one thread whose chunk holds it.
__device__ __forceinline__ void ce_update(const GemmArgs& p, int row, int col, const uint32_t* v, float& m, float& l) {
  const int nv = min(32, p.N - col);
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j < nv) mx = fmaxf(mx, __uint_as_float(v[j]));
  const float mn = fmaxf(m, mx);
  float acc = (m == -INFINITY) ? 0.f : l * __expf(m - mn);
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j < nv) acc += __expf(__uint_as_float(v[j]) - mn);
  m = mn;
  l = acc;
  const int64_t tl = (int64_t)p.ce_tgt[row] - p.ce_v0 - col;
  // compile-time indices only: a runtime v[tl] would put the accumulator chunk in local memory
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j == tl && j < nv) p.ce_tl[row] = __uint_as_float(v[j]);
}
__device__ __forceinline__ void ce_flush(const GemmArgs& p, int row, int col, float& m, float& l) {
  float* q = p.ce_part + ((int64_t)row * p.ce_nblk + col / 128) * 2;
  q[0] = m;
  q[1] = l;
  m = -INFINITY;
  l = 0.f;
}

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGES = kSmemBudget / (A_BYTES + B_BYTES);
  static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + 1024 + 512;
  static constexpr int TMEM_COLS = BN == 192 ? 512 : 2 * BN;  // tcgen05.alloc takes powers of two
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// 256-bit global accesses (sm_100 STG.256 / LDG.256): one thread writes a whole
// 32-byte sector per instruction.  The epilogue's threads each own one row, so
// a warp's 16-byte stores wrote half sectors (ncu: 2x the sectors of the
// bytes) -- the drain of a short-K GEMM's tiles was store-bound.
__device__ __forceinline__ void st256(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e, uint32_t f,
                                      uint32_t g, uint32_t h) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
               "r"(e), "r"(f), "r"(g), "r"(h)
               : "memory");
}
__device__ __forceinline__ void ld256(const void* p, float* o) {
  asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
               : "l"(p));
}
__device__ __forceinline__ bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }

// Epilogue for 32 consecutive columns of one row.
__device__ __forceinline__ void epilogue_row32(const GemmArgs& p, int row, int col, const uint32_t* v) {
  float f[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
  const bool full = (col + 32 <= p.N);
  if (p.epilogue == STP_EPI_ACCUM_F32) {
    float* c = reinterpret_cast<float*>(p.C) + (int64_t)row * p.ldc + col;
    if (full && aligned32(c)) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float o[8];
        ld256(c + j, o);
        st256(c + j, __float_as_uint(o[0] + f[j]), __float_as_uint(o[1] + f[j + 1]), __float_as_uint(o[2] + f[j + 2]),
              __float_as_uint(o[3] + f[j + 3]), __float_as_uint(o[4] + f[j + 4]), __float_as_uint(o[5] + f[j + 5]),
              __float_as_uint(o[6] + f[j + 6]), __float_as_uint(o[7] + f[j + 7]));
      }
    } else if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o = *reinterpret_cast<float4*>(c + j);
        o.x += f[j];
        o.y += f[j + 1];
        o.z += f[j + 2];
        o.w += f[j + 3];
        *reinterpret_cast<float4*>(c + j) = o;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < p.N) c[j] += f[j];
    }
    return;
  }
  if (p.epilogue == STP_EPI_SWIGLU_BWD) {  // C = [G | U] (ldc >= 2N), overwritten by [dG | dU]
    bf16* gp = reinterpret_cast<bf16*>(p.C) + (int64_t)row * p.ldc + col;
    bf16* up = gp + p.N;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 gv = *reinterpret_cast<const uint4*>(gp + j), uv = *reinterpret_cast<const uint4*>(up + j);
        const bf16* g8 = reinterpret_cast<const bf16*>(&gv);
        const bf16* u8 = reinterpret_cast<const bf16*>(&uv);
        float dg[8], du[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float z = __bfloat162float(g8[q]), sg = 1.f / (1.f + __expf(-z)), dh = f[j + q];
          du[q] = dh * z * sg;
          dg[q] = dh * __bfloat162float(u8[q]) * sg * (1.f + z * (1.f - sg));
        }
        *reinterpret_cast<uint4*>(gp + j) = make_uint4(pack_bf16x2(dg[0], dg[1]), pack_bf16x2(dg[2], dg[3]),
                                                       pack_bf16x2(dg[4], dg[5]), pack_bf16x2(dg[6], dg[7]));
        *reinterpret_cast<uint4*>(up + j) = make_uint4(pack_bf16x2(du[0], du[1]), pack_bf16x2(du[2], du[3]),
                                                       pack_bf16x2(du[4], du[5]), pack_bf16x2(du[6], du[7]));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (col + j >= p.N) continue;
        const float z = __bfloat162float(gp[j]), sg = 1.f / (1.f + __expf(-z)), dh = f[j];
        const float u = __bfloat162float(up[j]);
        up[j] = __float2bfloat16_rn(dh * z * sg);
        gp[j] = __float2bfloat16_rn(dh * u * sg * (1.f + z * (1.f - sg)));
      }
    }
    return;
  }
  if (p.epilogue == STP_EPI_BIAS) {
    const bf16* b = reinterpret_cast<const bf16*>(p.bias) + col;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (full || col + j < p.N) f[j] += __bfloat162float(b[j]);
  } else if (p.epilogue == STP_EPI_RESID) {
    const bf16* r = reinterpret_cast<const bf16*>(p.R) + (int64_t)row * p.ldr + col;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 u = *reinterpret_cast<const uint4*>(r + j);
        const bf16* h = reinterpret_cast<const bf16*>(&u);
#pragma unroll
        for (int q = 0; q < 8; ++q) f[j + q] += __bfloat162float(h[q]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < p.N) f[j] += __bfloat162float(r[j]);
    }
  }
  bf16* c = p.push_rows > 0 ? reinterpret_cast<bf16*>(p.push[row / p.push_rows]) +
                                  (p.push_off + row % p.push_rows) * p.ldc + col
                            : reinterpret_cast<bf16*>(p.C) + (int64_t)row * p.ldc + col;
  if (full && aligned32(c)) {
#pragma unroll
    for (int j = 0; j < 32; j += 16)
      st256(c + j, pack_bf16x2(f[j], f[j + 1]), pack_bf16x2(f[j + 2], f[j + 3]), pack_bf16x2(f[j + 4], f[j + 5]),
            pack_bf16x2(f[j + 6], f[j + 7]), pack_bf16x2(f[j + 8], f[j + 9]), pack_bf16x2(f[j + 10], f[j + 11]),
            pack_bf16x2(f[j + 12], f[j + 13]), pack_bf16x2(f[j + 14], f[j + 15]));
  } else if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 u;
      u.x = pack_bf16x2(f[j], f[j + 1]);
      u.y = pack_bf16x2(f[j + 2], f[j + 3]);
      u.z = pack_bf16x2(f[j + 4], f[j + 5]);
      u.w = pack_bf16x2(f[j + 6], f[j + 7]);
      *reinterpret_cast<uint4*>(c + j) = u;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col + j < p.N) c[j] = __float2bfloat16_rn(f[j]);
  }
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256, 1)
    gemm_bf16_sm100(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmArgs p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ring_full = tempty + 2;   // [4] tile-id ring (dynamic scheduler)
  uint64_t* ring_empty = ring_full + 4;
  int* ring = reinterpret_cast<int*>(ring_empty + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    for (int r = 0; r < 4; ++r) {
      mbar_init(ring_full + r, 1);
      mbar_init(ring_empty + r, 5);  // MMA lane + 4 epilogue warps
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_tiles = p.num_m_blk * p.num_n_blk;
  // Dynamic persistent scheduling: the producer lane fetches tile ids from a
  // global atomic counter and hands them to the MMA and epilogue roles via a
  // 4-deep smem ring.  CTAs that start late (SMs busy with communication
  // kernels of the braid) simply take fewer tiles -- no static tail.
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        const int rs = it & 3;
        mbar_wait_wd(ring_empty + rs, ((it >> 2) & 1) ^ 1, 1, p.M, p.N, p.K);
        const int got = atomicAdd(p.tile_ctr, 1);
        if (got == num_tiles + (int)gridDim.x - 1) atomicExch(p.tile_ctr, 0);  // last fetch of the launch
        const int tile = got < num_tiles ? got : -1;
        ring[rs] = tile;
        mbar_arrive(ring_full + rs);
        if (tile < 0) break;
        const int mb = p.n_fast ? tile / p.num_n_blk : tile % p.num_m_blk;
        const int nb = p.n_fast ? tile % p.num_n_blk : tile / p.num_m_blk;
        for (int kb = 0; kb < p.num_k_blk; ++kb) {
          mbar_wait_wd(empty + stage, phase ^ 1, 2, p.M, p.N, p.K);
          mbar_arrive_expect_tx(full + stage, C::A_BYTES + C::B_BYTES);
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          if (!A_MN) {
            tma_load_2d(a, &tmA, full + stage, kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) tma_load_2d(a + c * 64 * BK * 2, &tmA, full + stage, mb * BM + c * 64, kb * BK);
          }
          if (!B_MN) {
            tma_load_2d(b, &tmB, full + stage, kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) tma_load_2d(b + c * 64 * BK * 2, &tmB, full + stage, nb * BN + c * 64, kb * BK);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      for (int local = 0;; ++local) {
        const int rs = local & 3;
        mbar_wait_wd(ring_full + rs, (local >> 2) & 1, 3, p.M, p.N, p.K);
        const int tile = ring[rs];
        mbar_arrive(ring_empty + rs);
        if (tile < 0) break;
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait_wd(tempty + acc, acc_phase ^ 1, 4, p.M, p.N, p.K);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_k_blk; ++kb) {
          mbar_wait_wd(full + stage, phase, 5, p.M, p.N, p.K);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sw128_desc(a_addr + k * 2048, 64 * BK * 2, 1024)
                                     : make_sw128_desc(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sw128_desc(b_addr + k * 2048, 64 * BK * 2, 1024)
                                     : make_sw128_desc(b_addr + k * 32, 16, 1024);
            mma_f16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit(empty + stage);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(tfull + acc);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp & 3;
    for (int local = 0;; ++local) {
      const int rs = local & 3;
      mbar_wait_wd(ring_full + rs, (local >> 2) & 1, 6, p.M, p.N, p.K);
      const int tile = ring[rs];
      __syncwarp();
      if (lane == 0) mbar_arrive(ring_empty + rs);
      if (tile < 0) break;
      const int mb = p.n_fast ? tile / p.num_n_blk : tile % p.num_m_blk;
      const int nb = p.n_fast ? tile % p.num_n_blk : tile / p.num_m_blk;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait_wd(tfull + acc, acc_phase, 7, p.M, p.N, p.K);
      tc_fence_after();
      const int row = mb * BM + ew * 32 + lane;
      float ce_m = -INFINITY, ce_l = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + c0, v);
        tmem_wait_ld();
        const int col = nb * BN + c0;
        if (row < p.M && col < p.N) {
          epilogue_row32(p, row, col, v);
          if (p.epilogue == STP_EPI_STORE_CE) {
            ce_update(p, row, col, v, ce_m, ce_l);
            if ((c0 & 127) == 96 || col + 32 >= p.N) ce_flush(p, row, col, ce_m, ce_l);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}


// 2-SM variant (tcgen05.mma.cta_group::2): a CTA pair computes a 256 x 256
// tile; each SM stages 128 rows of A and 128 of the 256 B columns, and one
// thread of the even CTA issues M=256 MMAs reading both SMs' shared memory,
// accumulating rows 0-127 in the even CTA's TMEM and 128-255 in the odd one.
// Per SM this halves the shared-memory operand traffic per FLOP (the 1-SM
// 128x256 tile needs ~192 B/clk of smem reads+writes at full tensor rate,
// above the ~128 B/clk the SM provides — ncu: 64% tensor-active).
constexpr int S2_STAGE = 2 * 128 * BK * 2;           // A half + B half per CTA: 32 KB
constexpr int S2_STAGES = kSmemBudget / S2_STAGE;    // 6
constexpr int S2_SMEM = S2_STAGES * S2_STAGE + 1024 + 512;

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256, 1)
    gemm_bf16_sm100_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int HALF = 128 * BK * 2;  // 16 KB
  uint8_t* sA = smem;
  uint8_t* sB = smem + S2_STAGES * HALF;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S2_STAGES * S2_STAGE);
  uint64_t* empty = full + S2_STAGES;
  uint64_t* tfull = empty + S2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ring_full = tempty + 2;  // [4] cluster tile-id ring (dynamic scheduler)
  uint64_t* ring_empty = ring_full + 4;
  int* ring = reinterpret_cast<int*>(ring_empty + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();

  if (threadIdx.x == 0) {
    for (int s = 0; s < S2_STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);  // 4 epilogue warps x 2 CTAs (used on the even CTA)
    }
    for (int r = 0; r < 4; ++r) {
      mbar_init(ring_full + r, 1);
      mbar_init(ring_empty + r, 10);  // even CTA: MMA + 4 epi; odd CTA: producer + 4 epi
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  // The cta_group::2 allocation writes into the peer CTA's reserved shared
  // memory (allocation mailbox + mbarrier): both CTAs must have started before
  // it runs.  Without this cluster barrier the even CTA can race the odd
  // CTA's launch and the pair hangs inside tcgen05.alloc (seen as an
  // intermittent whole-step hang; cuda-gdb: odd CTA's allocator warp in the
  // "alloc after relinquish" trap path).
  cluster_sync();
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_m2 = (p.M + 255) / 256;
  const int num_n2 = (p.N + 255) / 256;
  const int num_tiles = num_m2 * num_n2;
  const int ncl = gridDim.x >> 1;
  const uint32_t ring_empty0 = mapa(smem_u32(ring_empty), 0);
  auto release_slot = [&](int rs) {
    if (rank == 0) mbar_arrive(ring_empty + rs);
    else mbar_arrive_cluster(ring_empty0 + rs * 8);
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = mapa(smem_u32(full), 0);
      for (int it = 0;; ++it) {
        const int rs = it & 3;
        int tile;
        if (rank == 0) {
          mbar_wait_cluster_wd(ring_empty + rs, ((it >> 2) & 1) ^ 1, 101, p.M, p.N, p.K);
          const int got = atomicAdd(p.tile_ctr, 1);
          if (got == num_tiles + ncl - 1) atomicExch(p.tile_ctr, 0);  // last fetch of the launch
          tile = got < num_tiles ? got : -1;
          ring[rs] = tile;
          st_cluster_u32(mapa(smem_u32(ring + rs), 1), (uint32_t)tile);
          mbar_arrive(ring_full + rs);
          mbar_arrive_cluster(mapa(smem_u32(ring_full + rs), 1));
        } else {
          mbar_wait_cluster_wd(ring_full + rs, (it >> 2) & 1, 102, p.M, p.N, p.K);
          tile = ring[rs];
          release_slot(rs);
        }
        if (tile < 0) break;
        const int m0 = (p.n_fast ? tile / num_n2 : tile % num_m2) * 256 + (int)rank * 128;
        const int n0 = (p.n_fast ? tile % num_n2 : tile / num_m2) * 256 + (int)rank * 128;
        for (int kb = 0; kb < p.num_k_blk; ++kb) {
          mbar_wait_wd(empty + stage, phase ^ 1, 103, p.M, p.N, p.K);
          if (rank == 0) mbar_arrive_expect_tx(full + stage, 2 * S2_STAGE);
          const uint32_t fb = full0 + stage * 8;
          uint8_t* a = sA + stage * HALF;
          uint8_t* b = sB + stage * HALF;
          if (!A_MN) {
            tma_load_2d_2sm(a, &tmA, fb, kb * BK, m0);
          } else {
            tma_load_2d_2sm(a, &tmA, fb, m0, kb * BK);
            tma_load_2d_2sm(a + 64 * BK * 2, &tmA, fb, m0 + 64, kb * BK);
          }
          if (!B_MN) {
            tma_load_2d_2sm(b, &tmB, fb, kb * BK, n0);
          } else {
            tma_load_2d_2sm(b, &tmB, fb, n0, kb * BK);
            tma_load_2d_2sm(b + 64 * BK * 2, &tmB, fb, n0 + 64, kb * BK);
          }
          if (++stage == S2_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(256, 256, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      for (int local = 0;; ++local) {
        const int rs = local & 3;
        mbar_wait_cluster_wd(ring_full + rs, (local >> 2) & 1, 104, p.M, p.N, p.K);
        const int tile = ring[rs];
        release_slot(rs);
        if (tile < 0) break;
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait_cluster_wd(tempty + acc, acc_phase ^ 1, 105, p.M, p.N, p.K);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < p.num_k_blk; ++kb) {
          mbar_wait_wd(full + stage, phase, 106, p.M, p.N, p.K);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * HALF);
          const uint32_t b_addr = smem_u32(sB + stage * HALF);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sw128_desc(a_addr + k * 2048, 64 * BK * 2, 1024)
                                     : make_sw128_desc(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sw128_desc(b_addr + k * 2048, 64 * BK * 2, 1024)
                                     : make_sw128_desc(b_addr + k * 32, 16, 1024);
            mma_f16_ss_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit_2sm_mc(empty + stage, 0x3);
          if (++stage == S2_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_2sm_mc(tfull + acc, 0x3);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp & 3;
    const uint32_t tempty0 = mapa(smem_u32(tempty), 0);
    for (int local = 0;; ++local) {
      const int rs = local & 3;
      mbar_wait_cluster_wd(ring_full + rs, (local >> 2) & 1, 107, p.M, p.N, p.K);
      const int tile = ring[rs];
      __syncwarp();
      if (lane == 0) release_slot(rs);
      if (tile < 0) break;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait_wd(tfull + acc, acc_phase, 108, p.M, p.N, p.K);
      tc_fence_after();
      const int row = (p.n_fast ? tile / num_n2 : tile % num_m2) * 256 + (int)rank * 128 + ew * 32 + lane;
      const int nb0 = (p.n_fast ? tile % num_n2 : tile / num_m2) * 256;
      float ce_m = -INFINITY, ce_l = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < 256; c0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * 256 + c0, v);
        tmem_wait_ld();
        const int col = nb0 + c0;
        if (row < p.M && col < p.N) {
          epilogue_row32(p, row, col, v);
          if (p.epilogue == STP_EPI_STORE_CE) {
            ce_update(p, row, col, v, ce_m, ce_l);
            if ((c0 & 127) == 96 || col + 32 >= p.N) ce_flush(p, row, col, ce_m, ce_l);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem_base);
  }
}

// ------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  int64_t d0, d1, ld;
  int b0, b1;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && d0 == o.d0 && d1 == o.d1 && ld == o.ld && b0 == o.b0 && b1 == o.b1;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    h ^= std::hash<int64_t>()(k.d0 * 1000003 + k.d1) + 0x9e3779b9 + (h << 6) + (h >> 2);
    h ^= std::hash<int64_t>()(k.ld * 131 + k.b0 * 7 + k.b1) + 0x9e3779b9 + (h << 6) + (h >> 2);
    return h;
  }
};

// 2-D bf16 tensor map: inner dim d0 (contiguous), outer dim d1, row stride ld
// elements, box b0 x b1, 128-byte swizzle, OOB -> zero.  Cached per thread.
stp_status tensor_map(CUtensorMap* out, const void* ptr, int64_t d0, int64_t d1, int64_t ld, int b0, int b1) {
  thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, d0, d1, ld, b0, b1};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return STP_OK;
  }
  auto enc = get_encode();
  if (!enc) return fail(STP_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)d0, (cuuint64_t)d1};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)b0, (cuuint32_t)b1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): d0=%lld d1=%lld ld=%lld box=%dx%d", (int)r, (long long)d0,
              (long long)d1, (long long)ld, b0, b1);
    return STP_ECUDA;
  }
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return STP_OK;
}

// 3-D bf16 tensor map over attention heads: dims {dh (contiguous), heads,
// rows}, strides {dh, ld} elements, box {64, 1, box_rows}, 128-byte swizzle.
// A box at column 64 of a head with dh < 128 reads zeros beyond dh (OOB fill),
// so a d = 80 head lands in shared memory as a zero-padded 128-column tile.
stp_status tensor_map_heads_impl(CUtensorMap* out, const void* ptr, int dh, int heads, int64_t rows, int64_t ld,
                                 int box_rows) {
  thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, -(int64_t)dh, (int64_t)heads * (1ll << 32) + rows, ld, 64, box_rows};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return STP_OK;
  }
  auto enc = get_encode();
  if (!enc) return fail(STP_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)dh, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)dh * 2, (cuuint64_t)(ld * 2)};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (heads) failed (%d): dh=%d heads=%d rows=%lld ld=%lld", (int)r, dh, heads,
              (long long)rows, (long long)ld);
    return STP_ECUDA;
  }
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return STP_OK;
}

// One tile counter per stream (GEMMs on one stream run in order; the last
// fetch of each launch resets its counter to 0).
// Counter blocks are kept per device (a thread that alternates devices
// reuses each device's block instead of reallocating it).
stp_status tile_counter(cudaStream_t st, int** out) {
  struct DevCounters {
    int* base = nullptr;
    std::unordered_map<cudaStream_t, int> slots;
  };
  thread_local std::unordered_map<int, DevCounters> per_dev;
  int dev = 0;
  STP_CUDA_TRY(cudaGetDevice(&dev));
  DevCounters& dc = per_dev[dev];
  int*& base = dc.base;
  auto& slots = dc.slots;
  if (!base) {
    STP_CUDA_TRY(cudaMalloc(&base, 1024 * sizeof(int)));
    STP_CUDA_TRY(cudaMemset(base, 0, 1024 * sizeof(int)));
  }
  auto it = slots.find(st);
  if (it == slots.end()) {
    if (slots.size() >= 1024 / 32) return fail(STP_EUNSUPPORTED, "too many GEMM streams");
    it = slots.emplace(st, (int)slots.size() * 32).first;  // 128-byte apart
  }
  *out = base + it->second;
  return STP_OK;
}

template <int BN, bool A_MN, bool B_MN>
stp_status launch_bf16(const GemmArgs& a, const CUtensorMap& ta, const CUtensorMap& tb, int max_ctas,
                       cudaStream_t st) {
  using C = Cfg<BN>;
  auto kern = gemm_bf16_sm100<BN, A_MN, B_MN>;
  static unsigned long long attr_mask = 0;  // per instantiation, one bit per device
  STP_TRY(set_max_smem_once((const void*)kern, C::SMEM, &attr_mask));
  const int tiles = a.num_m_blk * a.num_n_blk;
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (tiles < grid) grid = tiles;
  kern<<<grid, 256, C::SMEM, st>>>(ta, tb, a);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

}  // namespace

// Tuning knob (stp_set_option "gemm_mc"): 1 = auto (default: 2-SM kernel unless
// its 256x256 wave quantisation is clearly worse than the 1-SM 128xBN one),
// 0 = 1-SM kernel, 3 = 2-SM kernel.  (Round 1's 1-SM cluster variant with B
// multicast, measured slower than the 2-SM kernel, was removed in round 2.)
// Env STP_GEMM_MC sets the default.
int& gemm_mc_mode_ref() {
  static int mode = [] {
    const char* e = getenv("STP_GEMM_MC");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

namespace {

int gemm_mc_mode() { return gemm_mc_mode_ref(); }

template <bool A_MN, bool B_MN>
stp_status launch_bf16_2sm(const GemmArgs& a, const CUtensorMap& ta, const CUtensorMap& tb, int max_ctas,
                           cudaStream_t st) {
  auto kern = gemm_bf16_sm100_2sm<A_MN, B_MN>;
  static unsigned long long attr_mask = 0;  // per instantiation, one bit per device
  STP_TRY(set_max_smem_once((const void*)kern, S2_SMEM, &attr_mask));
  const int tiles = ((a.M + 255) / 256) * ((a.N + 255) / 256);
  int clusters = num_sms() / 2;
  if (max_ctas > 0 && max_ctas / 2 < clusters) clusters = std::max(1, max_ctas / 2);
  if (tiles < clusters) clusters = tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = S2_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  STP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, a));
  count_launch();
  return STP_OK;
}

// Push targets of the next bf16 GEMM on this thread (stp_gemm_push_targets).
struct PushExtra {
  void* ptr[8] = {};
  int n = 0;
  int64_t rows = 0, off = 0;
};
thread_local PushExtra g_push;

// Extra operands of the STORE_CE epilogue (set by lm_head_ce for one call).
struct CeExtra {
  const int32_t* tgt = nullptr;
  int64_t v0 = 0;
  float* part = nullptr;
  float* tl = nullptr;
};
thread_local CeExtra g_ce;

// stats[row] = (M, sum_b l_b exp(m_b - M), target logit) over the 128-column
// blocks of the STORE_CE epilogue (the layout ce_stats produces).
__global__ void ce_part_reduce(int64_t rows, int nblk, const float* __restrict__ part, const float* __restrict__ tl,
                               float* stats) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= rows) return;
  const float* q = part + w * nblk * 2;
  float m = -INFINITY;
  for (int b = lane; b < nblk; b += 32) m = fmaxf(m, q[2 * b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float l = 0.f;
  for (int b = lane; b < nblk; b += 32) l += q[2 * b + 1] * __expf(q[2 * b] - m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if (lane == 0) {
    stats[w * 3 + 0] = m;
    stats[w * 3 + 1] = l;
    stats[w * 3 + 2] = tl[w];
  }
}

stp_status gemm_bf16(int layout, int epi, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                     const void* B, int64_t ldb, void* Cp, int64_t ldc, const void* bias, const void* R,
                     int64_t ldr, int max_ctas, cudaStream_t st) {
  STP_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0 && ldc % 8 == 0, "bf16 GEMM strides must be multiples of 8");
  STP_CHECK_ARG((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
                "bf16 GEMM operands must be 16-byte aligned");
  STP_CHECK_ARG(epi != STP_EPI_RESID || (R != nullptr && ldr % 8 == 0), "RESID epilogue needs R, ldr%8==0");
  STP_CHECK_ARG(epi != STP_EPI_BIAS || bias != nullptr, "BIAS epilogue needs bias");
  const bool a_mn = (layout == STP_GEMM_TN);
  const bool b_mn = (layout == STP_GEMM_NN || layout == STP_GEMM_TN);
  // Kernel / tile choice: maximise (wave efficiency x per-tile throughput).
  // Per-tile tensor-pipe activity measured with ncu on B200 (round 1): 1-SM
  // 128x128 ~0.60, 1-SM 128x256 ~0.80, 2-SM 256x256 ~0.90 of peak (the
  // narrow tiles re-read more operand bytes from shared memory per FLOP).
  const int sms = (max_ctas > 0 && max_ctas < num_sms()) ? max_ctas : num_sms();
  auto eff = [](int64_t tiles, int64_t slots) {
    const int64_t waves = (tiles + slots - 1) / slots;
    return (double)tiles / (double)(waves * slots);
  };
  // useful fraction of the padded N extent (the last n-block of a skinny
  // TP-sharded GEMM can be mostly padding: N = 1152 in 256-wide tiles wastes 10%)
  auto npad = [&](int bn) { return (double)N / (double)(((N + bn - 1) / bn) * bn); };
  auto score1 = [&](int bn) {
    const double tile_eff = bn == 128 ? 0.60 : bn == 192 ? 0.72 : 0.80;
    return eff(((M + BM - 1) / BM) * ((N + bn - 1) / bn), sms) * tile_eff * npad(bn);
  };
  int BNsel = (N <= 128 || score1(128) > score1(256)) ? 128 : 256;
  // 128 x 192 tiles (1-SM) for N a multiple of 192 but not of 256 (not with the
  // CE-statistics epilogue, whose 128-column blocks need 128-aligned tiles)
  if (N % 192 == 0 && N % 256 != 0 && epi != STP_EPI_STORE_CE && score1(192) > score1(BNsel)) BNsel = 192;
  GemmArgs g;
  STP_TRY(tile_counter(st, &g.tile_ctr));
  g.M = (int)M;
  g.N = (int)N;
  g.K = (int)K;
  g.num_m_blk = (int)((M + BM - 1) / BM);
  g.num_n_blk = (int)((N + BNsel - 1) / BNsel);
  g.num_k_blk = (int)((K + BK - 1) / BK);
  // Raster: the operand swept once per block of the other one is re-read
  // from L2 only if it fits; sweep the smaller operand fastest, so the large
  // one streams from HBM once (e.g. the FC1 weight-gradient GEMM: A = dGU^T
  // 466 MB, B = Xn 44 MB -> n-fastest; m-fastest re-read A 14x, 7 GB / call).
  static const int raster_auto = [] {
    const char* e = getenv("STP_GEMM_RASTER");
    return e ? atoi(e) : 1;
  }();
  g.n_fast = (raster_auto && M > N) ? 1 : 0;
  g.epilogue = epi;
  g.C = Cp;
  g.ldc = ldc;
  g.bias = bias;
  g.R = R;
  g.ldr = ldr;
  g.ce_tgt = nullptr;
  g.ce_v0 = 0;
  g.ce_part = nullptr;
  g.ce_tl = nullptr;
  g.ce_nblk = (int)((N + 127) / 128);
  g.push_rows = 0;
  g.push_off = 0;
  if (g_push.n > 0) {
    if (epi != STP_EPI_STORE && epi != STP_EPI_BIAS) return fail(STP_EINVAL, "push targets need a STORE/BIAS epilogue");
    if (M != g_push.rows * g_push.n) return fail(STP_EINVAL, "push targets: M != rows * ranks");
    for (int i = 0; i < g_push.n; ++i) g.push[i] = g_push.ptr[i];
    g.push_rows = g_push.rows;
    g.push_off = g_push.off;
    g_push = PushExtra{};
  }
  if (epi == STP_EPI_STORE_CE) {
    if (!g_ce.tgt || !g_ce.part || !g_ce.tl) return fail(STP_EINVAL, "STORE_CE epilogue needs targets and outputs");
    g.ce_tgt = g_ce.tgt;
    g.ce_v0 = g_ce.v0;
    g.ce_part = g_ce.part;
    g.ce_tl = g_ce.tl;
  }
  CUtensorMap ta, tb;
  stp_status s;
  if (!a_mn) s = tensor_map(&ta, A, K, M, lda, BK, BM);  // A [M, K]
  else s = tensor_map(&ta, A, M, K, lda, 64, BK);         // A^T stored [K, M]
  if (s != STP_OK) return s;
  bool use_2sm = gemm_mc_mode() == 3 && M > 128;
  if (gemm_mc_mode() == 1 && M > 128) {
    const int64_t t2 = ((M + 255) / 256) * ((N + 255) / 256);
    use_2sm = eff(t2, sms / 2) * 0.90 * npad(256) >= score1(BNsel);
  }
  if (use_2sm) {
    // 2-SM: per-CTA boxes of 128 rows (K-major) / 2 x 64 columns (MN-major)
    CUtensorMap ta2, tb2;
    if (!a_mn) s = tensor_map(&ta2, A, K, M, lda, BK, 128);
    else s = tensor_map(&ta2, A, M, K, lda, 64, BK);
    if (s != STP_OK) return s;
    if (!b_mn) s = tensor_map(&tb2, B, K, N, ldb, BK, 128);
    else s = tensor_map(&tb2, B, N, K, ldb, 64, BK);
    if (s != STP_OK) return s;
    if (!a_mn && !b_mn) return launch_bf16_2sm<false, false>(g, ta2, tb2, max_ctas, st);
    if (!a_mn && b_mn) return launch_bf16_2sm<false, true>(g, ta2, tb2, max_ctas, st);
    if (a_mn && b_mn) return launch_bf16_2sm<true, true>(g, ta2, tb2, max_ctas, st);
  }
  if (!b_mn) s = tensor_map(&tb, B, K, N, ldb, BK, BNsel);  // B [N, K]
  else s = tensor_map(&tb, B, N, K, ldb, 64, BK);                              // B [K, N]
  if (s != STP_OK) return s;
#define STP_GEMM_CASE(bn, amn, bmn) \
  if (BNsel == bn && a_mn == amn && b_mn == bmn) return launch_bf16<bn, amn, bmn>(g, ta, tb, max_ctas, st);
  STP_GEMM_CASE(128, false, false)
  STP_GEMM_CASE(256, false, false)
  STP_GEMM_CASE(128, false, true)
  STP_GEMM_CASE(256, false, true)
  STP_GEMM_CASE(128, true, true)
  STP_GEMM_CASE(256, true, true)
  STP_GEMM_CASE(192, false, false)
  STP_GEMM_CASE(192, false, true)
  STP_GEMM_CASE(192, true, true)
#undef STP_GEMM_CASE
  return fail(STP_EUNSUPPORTED, "gemm layout");
}

// -------------------------------------------------------------- fp32 SIMT
// C[m,n] = sum_k A(m,k) B(k,n), A(m,k) = A[m*sam + k*sak], B(k,n) = B[k*sbk + n*sbn].
constexpr int FB = 64, FK = 16;
__global__ void __launch_bounds__(256) gemm_f32_simt(int M, int N, int K, const float* __restrict__ A, int64_t sam,
                                                     int64_t sak, const float* __restrict__ B, int64_t sbk,
                                                     int64_t sbn, float* C, int64_t ldc, int epi,
                                                     const float* __restrict__ bias, const float* __restrict__ R,
                                                     int64_t ldr) {
  __shared__ float As[FK][FB + 1];
  __shared__ float Bs[FK][FB + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * FB, n0 = blockIdx.x * FB;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += FK) {
    for (int i = threadIdx.x; i < FK * FB; i += 256) {
      int kk = i / FB, mm = i % FB;
      int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? A[(int64_t)m * sam + (int64_t)k * sak] : 0.f;
      int n = n0 + mm;
      Bs[kk][mm] = (n < N && k < K) ? B[(int64_t)k * sbk + (int64_t)n * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < FK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      float* c = C + (int64_t)m * ldc + n;
      if (epi == STP_EPI_ACCUM_F32) {
        *c += v;
      } else if (epi == STP_EPI_SWIGLU_BWD) {  // C = [G | U], overwritten by [dG | dU]
        const float z = c[0], u = c[N], sg = 1.f / (1.f + expf(-z));
        c[N] = v * z * sg;
        c[0] = v * u * sg * (1.f + z * (1.f - sg));
      } else {
        if (epi == STP_EPI_BIAS) v += bias[n];
        if (epi == STP_EPI_RESID) v += R[(int64_t)m * ldr + n];
        *c = v;
      }
    }
  }
}

stp_status gemm_f32(int layout, int epi, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                    const float* B, int64_t ldb, float* C, int64_t ldc, const float* bias, const float* R,
                    int64_t ldr, cudaStream_t st) {
  int64_t sam, sak, sbk, sbn;
  if (layout == STP_GEMM_NT) {
    sam = lda; sak = 1; sbk = 1; sbn = ldb;
  } else if (layout == STP_GEMM_NN) {
    sam = lda; sak = 1; sbk = ldb; sbn = 1;
  } else {
    sam = 1; sak = lda; sbk = ldb; sbn = 1;
  }
  dim3 grid((unsigned)((N + FB - 1) / FB), (unsigned)((M + FB - 1) / FB));
  gemm_f32_simt<<<grid, 256, 0, st>>>((int)M, (int)N, (int)K, A, sam, sak, B, sbk, sbn, C, ldc, epi, bias, R, ldr);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

}  // namespace

// 2-D bf16 tensor map with 128-byte swizzle (shared with the attention kernels).
stp_status tensor_map_bf16(CUtensorMap* out, const void* ptr, int64_t d0, int64_t d1, int64_t ld, int b0, int b1) {
  return tensor_map(out, ptr, d0, d1, ld, b0, b1);
}
stp_status tensor_map_heads(CUtensorMap* out, const void* ptr, int dh, int heads, int64_t rows, int64_t ld,
                            int box_rows) {
  return tensor_map_heads_impl(out, ptr, dh, heads, rows, ld, box_rows);
}

stp_status ce_stats(int dtype, int64_t s, int64_t Vl, const void* logits, int64_t ld, const int32_t* tgt, int64_t v0,
                    float* stats, cudaStream_t st);

stp_status gemm_dispatch(int dtype, int layout, int epi, int64_t M, int64_t N, int64_t K, const void* A,
                         int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, const void* bias,
                         const void* R, int64_t ldr, int max_ctas, cudaStream_t st);

// The next bf16 GEMM on this thread stores row m of C into
// ptrs[m / rows] + (off + m % rows) * ldc (n <= 8 targets, C unused): the
// row-parallel GEMM writes its partial directly into the TP peers' receive
// buffers over NVLink (the reduce-scatter's transfer fused into the epilogue).
void gemm_push_targets(void* const* ptrs, int n, int64_t rows, int64_t off) {
  g_push = PushExtra{};
  for (int i = 0; i < n && i < 8; ++i) g_push.ptr[i] = ptrs[i];
  g_push.n = n;
  g_push.rows = rows;
  g_push.off = off;
}

int64_t lm_head_ce_ws_bytes(int64_t s, int64_t Vl) { return (s * ((Vl + 127) / 128) * 2 + s) * 4 + 256; }

// LM head with the vocab-parallel CE statistics of its fp32 accumulators
// (reading Q18: fp32 softmax statistics): logits[s, Vl] = xf W^T (stored in
// the model dtype for the backward) and stats[s, 3] = (row max, sum exp(z -
// max), target logit or 0) of this rank's vocabulary rows [v0, v0 + Vl).
stp_status lm_head_ce(int dtype, int64_t s, int64_t Vl, int64_t h, const void* xf, const void* W, void* logits,
                      const int32_t* tgt, int64_t v0, void* ws, float* stats, int max_ctas, cudaStream_t st) {
  if (s == 0) return STP_OK;
  if (dtype != STP_DTYPE_BF16) {  // fp32 logits are the accumulator: plain store + stats pass
    STP_TRY(gemm_dispatch(dtype, STP_GEMM_NT, STP_EPI_STORE, s, Vl, h, xf, h, W, h, logits, Vl, nullptr, nullptr, 0,
                          max_ctas, st));
    return ce_stats(dtype, s, Vl, logits, Vl, tgt, v0, stats, st);
  }
  const int nblk = (int)((Vl + 127) / 128);
  float* part = (float*)ws;
  float* tl = part + s * nblk * 2;
  STP_CUDA_TRY(cudaMemsetAsync(tl, 0, s * 4, st));
  g_ce.tgt = tgt;
  g_ce.v0 = v0;
  g_ce.part = part;
  g_ce.tl = tl;
  const stp_status r = gemm_dispatch(dtype, STP_GEMM_NT, STP_EPI_STORE_CE, s, Vl, h, xf, h, W, h, logits, Vl, nullptr,
                                     nullptr, 0, max_ctas, st);
  g_ce = CeExtra{};
  STP_TRY(r);
  ce_part_reduce<<<(unsigned)((s + 7) / 8), 256, 0, st>>>(s, nblk, part, tl, stats);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

stp_status gemm_dispatch(int dtype, int layout, int epi, int64_t M, int64_t N, int64_t K, const void* A,
                         int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, const void* bias,
                         const void* R, int64_t ldr, int max_ctas, cudaStream_t st) {
  STP_CHECK_ARG(M >= 0 && N >= 0 && K >= 0, "negative GEMM size");
  STP_CHECK_ARG(layout >= 0 && layout <= 2, "layout");
  STP_CHECK_ARG(epi >= 0 && epi <= 5, "epilogue");
  STP_CHECK_ARG(epi != STP_EPI_SWIGLU_BWD || ldc >= 2 * N, "SWIGLU_BWD epilogue needs ldc >= 2N ([G | U] rows)");
  if (M == 0 || N == 0) return STP_OK;
  const double es = dtype == STP_DTYPE_BF16 ? 2.0 : 4.0;
  const double cbytes = (epi == STP_EPI_ACCUM_F32 ? 8.0 : epi == STP_EPI_SWIGLU_BWD ? 4.0 * es : es) * (double)M * N;
  ProfScope prof(PROF_GEMM, 2.0 * M * N * K, es * ((double)M * K + (double)N * K) + cbytes, st);
  if (dtype == STP_DTYPE_F32)
    return gemm_f32(layout, epi, M, N, K, (const float*)A, lda, (const float*)B, ldb, (float*)C, ldc,
                    (const float*)bias, (const float*)R, ldr, st);
  if (dtype == STP_DTYPE_BF16) {
    if (K == 0) return fail(STP_EUNSUPPORTED, "bf16 GEMM with K == 0");
    return gemm_bf16(layout, epi, M, N, K, A, lda, B, ldb, C, ldc, bias, R, ldr, max_ctas, st);
  }
  return fail(STP_EINVAL, "dtype");
}

}  // namespace stp

extern "C" int64_t stp_op_lm_head_ce_ws_bytes(int64_t s, int64_t Vl) { return stp::lm_head_ce_ws_bytes(s, Vl); }

extern "C" stp_status stp_op_lm_head_ce(int32_t dtype, int64_t s, int64_t Vl, int64_t h, const void* xf, const void* W,
                                        void* logits, const int32_t* tgt, int64_t v0, void* ws, float* stats,
                                        void* stream) {
  return stp::lm_head_ce(dtype, s, Vl, h, xf, W, logits, tgt, v0, ws, stats, 0, (cudaStream_t)stream);
}

extern "C" stp_status stp_op_gemm(int32_t dtype, int32_t layout, int32_t epilogue, int64_t M, int64_t N, int64_t K,
                                  const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                                  const void* bias, const void* R, int64_t ldr, int32_t max_ctas, void* stream) {
  return stp::gemm_dispatch(dtype, layout, epilogue, M, N, K, A, lda, B, ldb, C, ldc, bias, R, ldr, max_ctas,
                            (cudaStream_t)stream);
}
