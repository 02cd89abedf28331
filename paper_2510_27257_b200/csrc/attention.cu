// Causal GQA attention forward / backward (the Attn unit's core; the paper
// runs FlashAttention-2; math: SURVEY §8c.1, oracle
// attention_fwd / attention_bwd) and the bidirectional d = 80 attention of the
// ViT encoder (oracle/vit.py attention_full_fwd / _bwd).  Dispatch: bf16 with
// d in {128, 80} and the fused [q | k | v] row layout runs the tcgen05 kernels
// (attn_fwd_sm100.cu, attn_bwd_sm100.cu); other bf16 head dims (causal only)
// run the mma.sync kernels below; fp32 runs the SIMT kernels.
//
// bf16 mma.sync path (round 1, small-shape / odd-d fallback): FlashAttention-2-style tiling with warp-level
// mma.sync m16n8k16 (bf16 in, fp32 accumulate), online softmax in fp32,
// 64 x 64 tiles, 4 warps x 16 query (or key) rows, padded shared-memory rows
// (conflict-free 32-bit fragment loads).  Backward = a dK/dV kernel (one CTA
// per key block and kv head, looping over the group's query heads and the
// causal query blocks) and a dQ kernel (one CTA per query block and head),
// so no atomics are needed.
//
// fp32 path: straightforward SIMT kernels (one warp per row) used by the
// fp32 parity mode.
#include <algorithm>
#include <cmath>

#include "common.h"
#include "prof.h"

namespace stp {
namespace {

constexpr int BR = 64;   // query rows per CTA
constexpr int BC = 64;   // key rows per tile
constexpr int NW = 4;    // warps per CTA (16 rows each)
constexpr int TL = BC + 8;  // padded row length of transposed tiles

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ uint32_t ld32(const bf16* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// A fragment (16 x 16) of a row-major smem tile X[row][k] with row stride ld.
__device__ __forceinline__ void frag_a(uint32_t* a, const bf16* X, int ld, int r0, int k0, int lane) {
  const int g = lane >> 2, t = lane & 3;
  a[0] = ld32(X + (r0 + g) * ld + k0 + 2 * t);
  a[1] = ld32(X + (r0 + g + 8) * ld + k0 + 2 * t);
  a[2] = ld32(X + (r0 + g) * ld + k0 + 2 * t + 8);
  a[3] = ld32(X + (r0 + g + 8) * ld + k0 + 2 * t + 8);
}
// B fragment (16 x 8, k x n) from a smem tile stored as Y[n][k] (stride ld).
__device__ __forceinline__ void frag_b(uint32_t* b, const bf16* Y, int ld, int n0, int k0, int lane) {
  const int g = lane >> 2, t = lane & 3;
  b[0] = ld32(Y + (n0 + g) * ld + k0 + 2 * t);
  b[1] = ld32(Y + (n0 + g) * ld + k0 + 2 * t + 8);
}
// A fragment (16 rows x 16 k) from two C fragments (n-tiles j, j+1).
__device__ __forceinline__ void c2a(uint32_t* a, const float* c0, const float* c1) {
  a[0] = pack2(c0[0], c0[1]);
  a[1] = pack2(c0[2], c0[3]);
  a[2] = pack2(c1[0], c1[1]);
  a[3] = pack2(c1[2], c1[3]);
}

// Load `rows` x D rows (global row stride ld, element offset col) into smem
// tile S[r][D+8]; optionally also the transpose T[d][TL].  Rows >= nvalid -> 0.
template <int D>
__device__ __forceinline__ void load_tile(bf16* S, bf16* T, const bf16* G, int64_t ld, int64_t row0, int64_t nvalid) {
  constexpr int CH = D / 8;
  for (int idx = threadIdx.x; idx < BC * CH; idx += blockDim.x) {
    const int r = idx / CH, c = (idx % CH) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row0 + r < nvalid) v = *reinterpret_cast<const uint4*>(G + (row0 + r) * ld + c);
    if (S) *reinterpret_cast<uint4*>(S + r * (D + 8) + c) = v;
    if (T) {
      const bf16* e = reinterpret_cast<const bf16*>(&v);
#pragma unroll
      for (int i = 0; i < 8; ++i) T[(c + i) * TL + r] = e[i];
    }
  }
}

// ------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(128) attn_fwd_mma(int s, int nq, int nkv, const bf16* __restrict__ q,
                                                   const bf16* __restrict__ k, const bf16* __restrict__ v,
                                                   int64_t ld, bf16* o, int64_t ldo, float* lse) {
  extern __shared__ __align__(16) uint8_t smem[];
  bf16* Qs = reinterpret_cast<bf16*>(smem);
  bf16* Ks = Qs + BR * (D + 8);
  bf16* Vt = Ks + BC * (D + 8);
  const int nqb = gridDim.x;
  const int qb = nqb - 1 - blockIdx.x;
  const int h = blockIdx.y, grp = nq / nkv, kvh = h / grp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float scale = rsqrtf((float)D);
  load_tile<D>(Qs, nullptr, q + (int64_t)h * D, ld, (int64_t)qb * BR, s);
  __syncthreads();
  const int r0 = warp * 16;
  uint32_t qa[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) frag_a(qa[kk], Qs, D + 8, r0, kk * 16, lane);
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float oacc[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
  const int row_base = qb * BR + r0 + g;
  for (int kb = 0; kb <= qb; ++kb) {
    __syncthreads();
    load_tile<D>(Ks, nullptr, k + (int64_t)kvh * D, ld, (int64_t)kb * BC, s);
    load_tile<D>(nullptr, Vt, v + (int64_t)kvh * D, ld, (int64_t)kb * BC, s);
    __syncthreads();
    float S[BC / 8][4];
#pragma unroll
    for (int j = 0; j < BC / 8; ++j) S[j][0] = S[j][1] = S[j][2] = S[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk)
#pragma unroll
      for (int j = 0; j < BC / 8; ++j) {
        uint32_t b[2];
        frag_b(b, Ks, D + 8, j * 8, kk * 16, lane);
        mma16816(S[j], qa[kk], b);
      }
    float mx[2] = {m[0], m[1]};
#pragma unroll
    for (int j = 0; j < BC / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = kb * BC + j * 8 + 2 * t + (e & 1);
        const int row = row_base + 8 * (e >> 1);
        float x = S[j][e] * scale;
        if (col > row || col >= s) x = -INFINITY;
        S[j][e] = x;
        mx[e >> 1] = fmaxf(mx[e >> 1], x);
      }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
    }
    float alpha[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      alpha[i] = (m[i] == -INFINITY) ? 0.f : __expf(m[i] - mx[i]);
      m[i] = mx[i];
      l[i] *= alpha[i];
    }
#pragma unroll
    for (int j = 0; j < BC / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mm = m[e >> 1];
        const float p = (S[j][e] == -INFINITY) ? 0.f : __expf(S[j][e] - mm);
        S[j][e] = p;
        l[e >> 1] += p;
      }
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      oacc[n][0] *= alpha[0];
      oacc[n][1] *= alpha[0];
      oacc[n][2] *= alpha[1];
      oacc[n][3] *= alpha[1];
    }
#pragma unroll
    for (int kk = 0; kk < BC / 16; ++kk) {
      uint32_t a[4];
      c2a(a, S[2 * kk], S[2 * kk + 1]);
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        uint32_t b[2];
        frag_b(b, Vt, TL, n * 8, kk * 16, lane);
        mma16816(oacc[n], a, b);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    l[i] += __shfl_xor_sync(0xffffffffu, l[i], 1);
    l[i] += __shfl_xor_sync(0xffffffffu, l[i], 2);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = row_base + 8 * i;
    if (row >= s) continue;
    const float inv = 1.f / l[i];
    bf16* orow = o + (int64_t)row * ldo + (int64_t)h * D;
#pragma unroll
    for (int n = 0; n < D / 8; ++n)
      *reinterpret_cast<uint32_t*>(orow + n * 8 + 2 * t) = pack2(oacc[n][2 * i] * inv, oacc[n][2 * i + 1] * inv);
    if (t == 0) lse[(int64_t)h * s + row] = m[i] + logf(l[i]);
  }
}

// Dl[h][row] = sum_d dO * O  (fp32)
template <typename T>
__global__ void attn_bwd_dot(int s, int nq, int D, const T* __restrict__ o, int64_t ldo, const T* __restrict__ dout,
                             float* Dl) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)s * nq) return;
  const int64_t row = w / nq;
  const int h = (int)(w % nq);
  float acc = 0.f;
  for (int d = lane; d < D; d += 32)
    acc += to_f<T>(o[row * ldo + (int64_t)h * D + d]) * to_f<T>(dout[row * ldo + (int64_t)h * D + d]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) Dl[(int64_t)h * s + row] = acc;
}

// dK, dV for one key block and kv head.
template <int D>
__global__ void __launch_bounds__(128) attn_bwd_dkdv_mma(int s, int nq, int nkv, const bf16* __restrict__ q,
                                                        const bf16* __restrict__ k, const bf16* __restrict__ v,
                                                        int64_t ld, const bf16* __restrict__ dout, int64_t ldo,
                                                        const float* __restrict__ lse, const float* __restrict__ Dl,
                                                        bf16* dk, bf16* dv, int64_t ldd) {
  extern __shared__ __align__(16) uint8_t smem[];
  bf16* Ks = reinterpret_cast<bf16*>(smem);
  bf16* Vs = Ks + BC * (D + 8);
  bf16* Qs = Vs + BC * (D + 8);
  bf16* dOs = Qs + BR * (D + 8);
  bf16* Qt = dOs + BR * (D + 8);
  bf16* dOt = Qt + D * TL;
  float* sl = reinterpret_cast<float*>(dOt + D * TL);
  float* sd = sl + BR;
  const int nb = (s + BC - 1) / BC;
  const int kb = blockIdx.x, kvh = blockIdx.y, grp = nq / nkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float scale = rsqrtf((float)D);
  load_tile<D>(Ks, nullptr, k + (int64_t)kvh * D, ld, (int64_t)kb * BC, s);
  load_tile<D>(Vs, nullptr, v + (int64_t)kvh * D, ld, (int64_t)kb * BC, s);
  const int r0 = warp * 16;
  const int kv_base = kb * BC + r0 + g;
  float dka[D / 8][4], dva[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) dka[n][e] = dva[n][e] = 0.f;
  for (int hh = 0; hh < grp; ++hh) {
    const int h = kvh * grp + hh;
    for (int qb = kb; qb < nb; ++qb) {
      __syncthreads();
      load_tile<D>(Qs, Qt, q + (int64_t)h * D, ld, (int64_t)qb * BR, s);
      load_tile<D>(dOs, dOt, dout + (int64_t)h * D, ldo, (int64_t)qb * BR, s);
      for (int i = threadIdx.x; i < BR; i += blockDim.x) {
        const int row = qb * BR + i;
        sl[i] = row < s ? lse[(int64_t)h * s + row] : 0.f;
        sd[i] = row < s ? Dl[(int64_t)h * s + row] : 0.f;
      }
      __syncthreads();
      float P[BR / 8][4];  // P^T: rows = keys, cols = queries
#pragma unroll
      for (int j = 0; j < BR / 8; ++j) P[j][0] = P[j][1] = P[j][2] = P[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        uint32_t a[4];
        frag_a(a, Ks, D + 8, r0, kk * 16, lane);
#pragma unroll
        for (int j = 0; j < BR / 8; ++j) {
          uint32_t b[2];
          frag_b(b, Qs, D + 8, j * 8, kk * 16, lane);
          mma16816(P[j], a, b);
        }
      }
#pragma unroll
      for (int j = 0; j < BR / 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int qc = j * 8 + 2 * t + (e & 1);
          const int qrow = qb * BR + qc;
          const int kvr = kv_base + 8 * (e >> 1);
          P[j][e] = (qrow >= kvr && qrow < s && kvr < s) ? __expf(P[j][e] * scale - sl[qc]) : 0.f;
        }
      // dV += P^T dO
#pragma unroll
      for (int kk = 0; kk < BR / 16; ++kk) {
        uint32_t a[4];
        c2a(a, P[2 * kk], P[2 * kk + 1]);
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          uint32_t b[2];
          frag_b(b, dOt, TL, n * 8, kk * 16, lane);
          mma16816(dva[n], a, b);
        }
      }
      // dP^T = V dO^T
      float dP[BR / 8][4];
#pragma unroll
      for (int j = 0; j < BR / 8; ++j) dP[j][0] = dP[j][1] = dP[j][2] = dP[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        uint32_t a[4];
        frag_a(a, Vs, D + 8, r0, kk * 16, lane);
#pragma unroll
        for (int j = 0; j < BR / 8; ++j) {
          uint32_t b[2];
          frag_b(b, dOs, D + 8, j * 8, kk * 16, lane);
          mma16816(dP[j], a, b);
        }
      }
      // dS^T = P^T * (dP^T - Dl[q])
#pragma unroll
      for (int j = 0; j < BR / 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int qc = j * 8 + 2 * t + (e & 1);
          dP[j][e] = P[j][e] * (dP[j][e] - sd[qc]);
        }
      // dK += dS^T Q
#pragma unroll
      for (int kk = 0; kk < BR / 16; ++kk) {
        uint32_t a[4];
        c2a(a, dP[2 * kk], dP[2 * kk + 1]);
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          uint32_t b[2];
          frag_b(b, Qt, TL, n * 8, kk * 16, lane);
          mma16816(dka[n], a, b);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = kv_base + 8 * i;
    if (row >= s) continue;
    bf16* kr = dk + (int64_t)row * ldd + (int64_t)kvh * D;
    bf16* vr = dv + (int64_t)row * ldd + (int64_t)kvh * D;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      *reinterpret_cast<uint32_t*>(kr + n * 8 + 2 * t) = pack2(dka[n][2 * i] * scale, dka[n][2 * i + 1] * scale);
      *reinterpret_cast<uint32_t*>(vr + n * 8 + 2 * t) = pack2(dva[n][2 * i], dva[n][2 * i + 1]);
    }
  }
}

// dQ for one query block and head.
template <int D>
__global__ void __launch_bounds__(128) attn_bwd_dq_mma(int s, int nq, int nkv, const bf16* __restrict__ q,
                                                      const bf16* __restrict__ k, const bf16* __restrict__ v,
                                                      int64_t ld, const bf16* __restrict__ dout, int64_t ldo,
                                                      const float* __restrict__ lse, const float* __restrict__ Dl,
                                                      bf16* dq, int64_t ldd) {
  extern __shared__ __align__(16) uint8_t smem[];
  bf16* Qs = reinterpret_cast<bf16*>(smem);
  bf16* dOs = Qs + BR * (D + 8);
  bf16* Ks = dOs + BR * (D + 8);
  bf16* Vs = Ks + BC * (D + 8);
  bf16* Kt = Vs + BC * (D + 8);
  const int nqb = gridDim.x;
  const int qb = nqb - 1 - blockIdx.x;
  const int h = blockIdx.y, grp = nq / nkv, kvh = h / grp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float scale = rsqrtf((float)D);
  load_tile<D>(Qs, nullptr, q + (int64_t)h * D, ld, (int64_t)qb * BR, s);
  load_tile<D>(dOs, nullptr, dout + (int64_t)h * D, ldo, (int64_t)qb * BR, s);
  const int r0 = warp * 16;
  const int row_base = qb * BR + r0 + g;
  float myl[2], myd[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = row_base + 8 * i;
    myl[i] = row < s ? lse[(int64_t)h * s + row] : 0.f;
    myd[i] = row < s ? Dl[(int64_t)h * s + row] : 0.f;
  }
  float dqa[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) dqa[n][0] = dqa[n][1] = dqa[n][2] = dqa[n][3] = 0.f;
  for (int kb = 0; kb <= qb; ++kb) {
    __syncthreads();
    load_tile<D>(Ks, Kt, k + (int64_t)kvh * D, ld, (int64_t)kb * BC, s);
    load_tile<D>(Vs, nullptr, v + (int64_t)kvh * D, ld, (int64_t)kb * BC, s);
    __syncthreads();
    float S[BC / 8][4], dP[BC / 8][4];
#pragma unroll
    for (int j = 0; j < BC / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) S[j][e] = dP[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t a[4], a2[4];
      frag_a(a, Qs, D + 8, r0, kk * 16, lane);
      frag_a(a2, dOs, D + 8, r0, kk * 16, lane);
#pragma unroll
      for (int j = 0; j < BC / 8; ++j) {
        uint32_t b[2], b2[2];
        frag_b(b, Ks, D + 8, j * 8, kk * 16, lane);
        mma16816(S[j], a, b);
        frag_b(b2, Vs, D + 8, j * 8, kk * 16, lane);
        mma16816(dP[j], a2, b2);
      }
    }
#pragma unroll
    for (int j = 0; j < BC / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = kb * BC + j * 8 + 2 * t + (e & 1);
        const int row = row_base + 8 * (e >> 1);
        const float p = (col <= row && col < s) ? __expf(S[j][e] * scale - myl[e >> 1]) : 0.f;
        S[j][e] = p * (dP[j][e] - myd[e >> 1]);
      }
#pragma unroll
    for (int kk = 0; kk < BC / 16; ++kk) {
      uint32_t a[4];
      c2a(a, S[2 * kk], S[2 * kk + 1]);
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        uint32_t b[2];
        frag_b(b, Kt, TL, n * 8, kk * 16, lane);
        mma16816(dqa[n], a, b);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = row_base + 8 * i;
    if (row >= s) continue;
    bf16* qr = dq + (int64_t)row * ldd + (int64_t)h * D;
#pragma unroll
    for (int n = 0; n < D / 8; ++n)
      *reinterpret_cast<uint32_t*>(qr + n * 8 + 2 * t) = pack2(dqa[n][2 * i] * scale, dqa[n][2 * i + 1] * scale);
  }
}

// ------------------------------------------------------------ fp32 SIMT
// One warp per (query row, head): online softmax over keys <= row.
__global__ void attn_fwd_f32(int s, int nq, int nkv, int D, int causal, const float* __restrict__ q,
                             const float* __restrict__ k, const float* __restrict__ v, int64_t ld, float* o,
                             int64_t ldo, float* lse) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)s * nq) return;
  const int h = (int)(w % nq);
  const int64_t row = w / nq;
  const int kvh = h / (nq / nkv);
  const float scale = 1.f / sqrtf((float)D);
  const float* qr = q + row * ld + (int64_t)h * D;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};  // D <= 128
  float m = -INFINITY, l = 0.f;
  const int64_t jmax = causal ? row : s - 1;
  for (int64_t j = 0; j <= jmax; ++j) {
    const float* kr = k + j * ld + (int64_t)kvh * D;
    float dot = 0.f;
    for (int d = lane; d < D; d += 32) dot += qr[d] * kr[d];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    const float x = dot * scale;
    const float mn = fmaxf(m, x);
    const float a = (m == -INFINITY) ? 0.f : expf(m - mn);
    const float p = expf(x - mn);
    l = l * a + p;
    const float* vr = v + j * ld + (int64_t)kvh * D;
    for (int d = lane, i = 0; d < D; d += 32, ++i) acc[i] = acc[i] * a + p * vr[d];
    m = mn;
  }
  float* orow = o + row * ldo + (int64_t)h * D;
  for (int d = lane, i = 0; d < D; d += 32, ++i) orow[d] = acc[i] / l;
  if (lane == 0) lse[(int64_t)h * s + row] = m + logf(l);
}

// dQ: one warp per (query row, head).
__global__ void attn_bwd_dq_f32(int s, int nq, int nkv, int D, int causal, const float* __restrict__ q,
                                const float* __restrict__ k, const float* __restrict__ v, int64_t ld,
                                const float* __restrict__ dout, int64_t ldo, const float* __restrict__ lse,
                                const float* __restrict__ Dl, float* dq, int64_t ldd) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)s * nq) return;
  const int h = (int)(w % nq);
  const int64_t row = w / nq;
  const int kvh = h / (nq / nkv);
  const float scale = 1.f / sqrtf((float)D);
  const float* qr = q + row * ld + (int64_t)h * D;
  const float* dor = dout + row * ldo + (int64_t)h * D;
  const float L = lse[(int64_t)h * s + row], Dv = Dl[(int64_t)h * s + row];
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const int64_t jmax = causal ? row : s - 1;
  for (int64_t j = 0; j <= jmax; ++j) {
    const float* kr = k + j * ld + (int64_t)kvh * D;
    const float* vr = v + j * ld + (int64_t)kvh * D;
    float dot = 0.f, dp = 0.f;
    for (int d = lane; d < D; d += 32) {
      dot += qr[d] * kr[d];
      dp += dor[d] * vr[d];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      dot += __shfl_xor_sync(0xffffffffu, dot, off);
      dp += __shfl_xor_sync(0xffffffffu, dp, off);
    }
    const float p = expf(dot * scale - L);
    const float ds = p * (dp - Dv);
    for (int d = lane, i = 0; d < D; d += 32, ++i) acc[i] += ds * kr[d];
  }
  float* r = dq + row * ldd + (int64_t)h * D;
  for (int d = lane, i = 0; d < D; d += 32, ++i) r[d] = acc[i] * scale;
}

// dK, dV: one warp per (key row, kv head), summing over the group's query heads.
__global__ void attn_bwd_dkdv_f32(int s, int nq, int nkv, int D, int causal, const float* __restrict__ q,
                                  const float* __restrict__ k, const float* __restrict__ v, int64_t ld,
                                  const float* __restrict__ dout, int64_t ldo, const float* __restrict__ lse,
                                  const float* __restrict__ Dl, float* dk, float* dv, int64_t ldd) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)s * nkv) return;
  const int kvh = (int)(w % nkv);
  const int64_t j = w / nkv;
  const int grp = nq / nkv;
  const float scale = 1.f / sqrtf((float)D);
  const float* kr = k + j * ld + (int64_t)kvh * D;
  const float* vr = v + j * ld + (int64_t)kvh * D;
  float ak[4] = {0.f, 0.f, 0.f, 0.f}, av[4] = {0.f, 0.f, 0.f, 0.f};
  for (int hh = 0; hh < grp; ++hh) {
    const int h = kvh * grp + hh;
    for (int64_t i = causal ? j : 0; i < s; ++i) {
      const float* qr = q + i * ld + (int64_t)h * D;
      const float* dor = dout + i * ldo + (int64_t)h * D;
      float dot = 0.f, dp = 0.f;
      for (int d = lane; d < D; d += 32) {
        dot += qr[d] * kr[d];
        dp += dor[d] * vr[d];
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        dot += __shfl_xor_sync(0xffffffffu, dot, off);
        dp += __shfl_xor_sync(0xffffffffu, dp, off);
      }
      const float p = expf(dot * scale - lse[(int64_t)h * s + i]);
      const float ds = p * (dp - Dl[(int64_t)h * s + i]);
      for (int d = lane, x = 0; d < D; d += 32, ++x) {
        av[x] += p * dor[d];
        ak[x] += ds * qr[d];
      }
    }
  }
  for (int d = lane, x = 0; d < D; d += 32, ++x) {
    dk[j * ldd + (int64_t)kvh * D + d] = ak[x] * scale;
    dv[j * ldd + (int64_t)kvh * D + d] = av[x];
  }
}

template <int D>
size_t fwd_smem() { return (size_t)(BR * (D + 8) + BC * (D + 8) + D * TL) * 2; }
template <int D>
size_t dkdv_smem() { return (size_t)(2 * BC * (D + 8) + 2 * BR * (D + 8) + 2 * D * TL) * 2 + 2 * BR * 4; }
template <int D>
size_t dq_smem() { return (size_t)(2 * BR * (D + 8) + 2 * BC * (D + 8) + D * TL) * 2; }

template <int D>
stp_status fwd_bf16(int s, int nq, int nkv, const void* q, const void* k, const void* v, int64_t ld, void* o,
                    int64_t ldo, float* lse, cudaStream_t st) {
  auto kern = attn_fwd_mma<D>;
  const size_t sm = fwd_smem<D>();
  STP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  dim3 grid((s + BR - 1) / BR, nq);
  kern<<<grid, 32 * NW, sm, st>>>(s, nq, nkv, (const bf16*)q, (const bf16*)k, (const bf16*)v, ld, (bf16*)o, ldo, lse);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

template <int D>
stp_status bwd_bf16(int s, int nq, int nkv, const void* q, const void* k, const void* v, int64_t ld,
                    const void* dout, int64_t ldo, const float* lse, const float* Dl, void* dq, void* dk, void* dv,
                    int64_t ldd, cudaStream_t st) {
  {
    auto kern = attn_bwd_dkdv_mma<D>;
    const size_t sm = dkdv_smem<D>();
    STP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dim3 grid((s + BC - 1) / BC, nkv);
    kern<<<grid, 32 * NW, sm, st>>>(s, nq, nkv, (const bf16*)q, (const bf16*)k, (const bf16*)v, ld,
                                    (const bf16*)dout, ldo, lse, Dl, (bf16*)dk, (bf16*)dv, ldd);
    count_launch();
    STP_LAUNCH_CHECK();
  }
  {
    auto kern = attn_bwd_dq_mma<D>;
    const size_t sm = dq_smem<D>();
    STP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dim3 grid((s + BR - 1) / BR, nq);
    kern<<<grid, 32 * NW, sm, st>>>(s, nq, nkv, (const bf16*)q, (const bf16*)k, (const bf16*)v, ld,
                                    (const bf16*)dout, ldo, lse, Dl, (bf16*)dq, ldd);
    count_launch();
    STP_LAUNCH_CHECK();
  }
  return STP_OK;
}

}  // namespace

stp_status attn_fwd_sm100_launch(int s, int nq, int nkv, int dh, int causal, const void* qkv_base, int64_t ld,
                                 void* o, int64_t ldo, float* lse, cudaStream_t st);


int64_t attn_bwd_fused_ws_bytes(int64_t s, int nq, int nkv);
stp_status attn_bwd_fused_launch(int s, int nq, int nkv, int dh, int causal, const void* qkv, int64_t ld,
                                 const void* o, const void* dout, int64_t ldo, const float* lse, void* dqkv,
                                 int64_t ldd, void* ws, cudaStream_t st);

// fp32 workspace: D = rowsum(dO*O) [nq, s] for the mma.sync / fp32 paths;
// the fused tcgen05 path (d = 128) needs attn_bwd_fused_ws_bytes.
int64_t attn_bwd_ws_bytes(int64_t s, int nq, int nkv, int d) {
  int64_t b = s * nq * (int64_t)sizeof(float);
  if (d == 128 || d == 80) b = std::max(b, attn_bwd_fused_ws_bytes(s, nq, nkv));
  return b;
}

stp_status attn_fwd(int dtype, int64_t s, int nq, int nkv, int d, int causal, const void* q, const void* k,
                    const void* v, int64_t ld, void* o, int64_t ldo, float* lse, cudaStream_t st) {
  STP_CHECK_ARG(nq > 0 && nkv > 0 && nq % nkv == 0, "nq % nkv == 0");
  STP_CHECK_ARG(d > 0 && d <= 128, "head_dim <= 128");
  if (s == 0) return STP_OK;
  // algorithmic FLOPs: QK^T and PV over the visible pairs (s(s+1)/2 causal, s^2 bidirectional)
  const double pairs = causal ? 0.5 * (double)s * (double)(s + 1) : (double)s * (double)s;
  ProfScope prof(PROF_ATTN_FWD, 4.0 * pairs * nq * d, (double)dtype_size(dtype) * s * (nq + 2 * nkv + nq) * d, st);
  if (dtype == STP_DTYPE_F32) {
    const int64_t warps = s * nq;
    attn_fwd_f32<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>((int)s, nq, nkv, d, causal, (const float*)q,
                                                             (const float*)k, (const float*)v, ld, (float*)o, ldo,
                                                             lse);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  }
  STP_CHECK_ARG(ld % 8 == 0 && ldo % 8 == 0, "bf16 attention strides % 8 == 0");
  // tcgen05 path: d = 128 or 80 with the fused [q | k | v] row layout
  static const bool force_mma = getenv("STP_ATTN_MMA_SYNC") != nullptr;
  const bool fused = (const uint8_t*)k == (const uint8_t*)q + (int64_t)nq * d * 2 &&
                     (const uint8_t*)v == (const uint8_t*)k + (int64_t)nkv * d * 2 && ld == (int64_t)(nq + 2 * nkv) * d;
  if ((d == 128 || d == 80) && fused && (!force_mma || d == 80))
    return attn_fwd_sm100_launch((int)s, nq, nkv, d, causal, q, ld, o, ldo, lse, st);
  if (!causal) return fail(STP_EUNSUPPORTED, "bidirectional bf16 attention needs d in {80, 128} and the [q|k|v] layout");
  switch (d) {
    case 16: return fwd_bf16<16>((int)s, nq, nkv, q, k, v, ld, o, ldo, lse, st);
    case 32: return fwd_bf16<32>((int)s, nq, nkv, q, k, v, ld, o, ldo, lse, st);
    case 64: return fwd_bf16<64>((int)s, nq, nkv, q, k, v, ld, o, ldo, lse, st);
    case 128: return fwd_bf16<128>((int)s, nq, nkv, q, k, v, ld, o, ldo, lse, st);
  }
  return fail(STP_EUNSUPPORTED, "bf16 attention head_dim must be 16, 32, 64 or 128");
}

stp_status attn_bwd(int dtype, int64_t s, int nq, int nkv, int d, int causal, const void* q, const void* k,
                    const void* v, int64_t ld, const void* o, int64_t ldo, const void* dout, const float* lse,
                    void* dq, void* dk, void* dv, int64_t ldd, void* ws, cudaStream_t st) {
  STP_CHECK_ARG(nq > 0 && nkv > 0 && nq % nkv == 0, "nq % nkv == 0");
  STP_CHECK_ARG(d > 0 && d <= 128, "head_dim <= 128");
  STP_CHECK_ARG(ws != nullptr, "workspace");
  if (s == 0) return STP_OK;
  const double pairs = causal ? 0.5 * (double)s * (double)(s + 1) : (double)s * (double)s;
  ProfScope prof(PROF_ATTN_BWD, 8.0 * pairs * nq * d,
                 (double)dtype_size(dtype) * s * (2 * (nq + 2 * nkv) + 2 * nq) * d, st);
  float* Dl = (float*)ws;
  const int64_t warps = s * nq;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    // fused tcgen05 backward (d = 128 or 80, [q | k | v] layouts): computes its own D
    if (dtype == STP_DTYPE_BF16 && (d == 128 || d == 80) && (d == 80 || getenv("STP_ATTN_MMA_SYNC") == nullptr) &&
        (const uint8_t*)k == (const uint8_t*)q + (int64_t)nq * d * 2 &&
        (const uint8_t*)v == (const uint8_t*)k + (int64_t)nkv * d * 2 && ld == (int64_t)(nq + 2 * nkv) * d &&
        (const uint8_t*)dk == (const uint8_t*)dq + (int64_t)nq * d * 2 &&
        (const uint8_t*)dv == (const uint8_t*)dk + (int64_t)nkv * d * 2 && ld % 8 == 0 && ldo % 8 == 0 && ldd % 8 == 0)
      return attn_bwd_fused_launch((int)s, nq, nkv, d, causal, q, ld, o, dout, ldo, lse, dq, ldd, ws, st);
    if (dtype == STP_DTYPE_BF16 && !causal)
      return fail(STP_EUNSUPPORTED, "bidirectional bf16 attention needs d in {80, 128} and the [q|k|v] layouts");
    attn_bwd_dot<T><<<(unsigned)((warps + 7) / 8), 256, 0, st>>>((int)s, nq, d, (const T*)o, ldo, (const T*)dout, Dl);
    count_launch();
    STP_LAUNCH_CHECK();
    if (dtype == STP_DTYPE_F32) {
      attn_bwd_dq_f32<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>((int)s, nq, nkv, d, causal, (const float*)q,
                                                                  (const float*)k, (const float*)v, ld,
                                                                  (const float*)dout, ldo, lse, Dl, (float*)dq, ldd);
      count_launch();
      STP_LAUNCH_CHECK();
      const int64_t kw = s * nkv;
      attn_bwd_dkdv_f32<<<(unsigned)((kw + 7) / 8), 256, 0, st>>>((int)s, nq, nkv, d, causal, (const float*)q,
                                                                 (const float*)k, (const float*)v, ld,
                                                                 (const float*)dout, ldo, lse, Dl, (float*)dk,
                                                                 (float*)dv, ldd);
      count_launch();
      STP_LAUNCH_CHECK();
      return STP_OK;
    }
    if (ld % 8 || ldo % 8 || ldd % 8) return fail(STP_EINVAL, "bf16 attention strides % 8 == 0");
    static const bool force_mma = getenv("STP_ATTN_MMA_SYNC") != nullptr;
    switch (d) {
      case 16: return bwd_bf16<16>((int)s, nq, nkv, q, k, v, ld, dout, ldo, lse, Dl, dq, dk, dv, ldd, st);
      case 32: return bwd_bf16<32>((int)s, nq, nkv, q, k, v, ld, dout, ldo, lse, Dl, dq, dk, dv, ldd, st);
      case 64: return bwd_bf16<64>((int)s, nq, nkv, q, k, v, ld, dout, ldo, lse, Dl, dq, dk, dv, ldd, st);
      case 128: return bwd_bf16<128>((int)s, nq, nkv, q, k, v, ld, dout, ldo, lse, Dl, dq, dk, dv, ldd, st);
    }
    return fail(STP_EUNSUPPORTED, "bf16 attention head_dim must be 16, 32, 64 or 128");
  });
}

}  // namespace stp

extern "C" {

int64_t stp_op_attn_bwd_ws_bytes(int64_t s, int32_t nq, int32_t nkv, int32_t d) {
  return stp::attn_bwd_ws_bytes(s, nq, nkv, d);
}
stp_status stp_op_attn_fwd(int32_t dtype, int64_t s, int32_t nq, int32_t nkv, int32_t d, const void* q, const void* k,
                           const void* v, int64_t ld_qkv, void* o, int64_t ld_o, float* lse, void* stream) {
  return stp::attn_fwd(dtype, s, nq, nkv, d, 1, q, k, v, ld_qkv, o, ld_o, lse, (cudaStream_t)stream);
}
stp_status stp_op_attn_full_fwd(int32_t dtype, int64_t s, int32_t nh, int32_t d, const void* qkv, int64_t ld_qkv,
                                void* o, int64_t ld_o, float* lse, void* stream) {
  const uint8_t* q = (const uint8_t*)qkv;
  const int64_t es = dtype == STP_DTYPE_BF16 ? 2 : 4;
  return stp::attn_fwd(dtype, s, nh, nh, d, 0, q, q + nh * d * es, q + 2 * nh * d * es, ld_qkv, o, ld_o, lse,
                       (cudaStream_t)stream);
}
stp_status stp_op_attn_full_bwd(int32_t dtype, int64_t s, int32_t nh, int32_t d, const void* qkv, int64_t ld_qkv,
                                const void* o, int64_t ld_o, const void* dout, const float* lse, void* dqkv,
                                int64_t ld_dqkv, void* ws, void* stream) {
  const uint8_t* q = (const uint8_t*)qkv;
  uint8_t* dq = (uint8_t*)dqkv;
  const int64_t es = dtype == STP_DTYPE_BF16 ? 2 : 4, hs = nh * d * es;
  return stp::attn_bwd(dtype, s, nh, nh, d, 0, q, q + hs, q + 2 * hs, ld_qkv, o, ld_o, dout, lse, dq, dq + hs,
                       dq + 2 * hs, ld_dqkv, ws, (cudaStream_t)stream);
}
stp_status stp_op_attn_bwd(int32_t dtype, int64_t s, int32_t nq, int32_t nkv, int32_t d, const void* q, const void* k,
                           const void* v, int64_t ld_qkv, const void* o, int64_t ld_o, const void* dout,
                           const float* lse, void* dq, void* dk, void* dv, int64_t ld_dqkv, void* ws, void* stream) {
  return stp::attn_bwd(dtype, s, nq, nkv, d, 1, q, k, v, ld_qkv, o, ld_o, dout, lse, dq, dk, dv, ld_dqkv, ws,
                       (cudaStream_t)stream);
}

}  // extern "C"
