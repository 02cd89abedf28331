// Fused memory-bound kernels of the STP units:
// RMSNorm fwd/bwd with the fused residual of Eq. 1-2 (SP
// reading Q10), rotate-half RoPE fwd/bwd, SwiGLU fwd/bwd, vocab-parallel
// embedding fwd/bwd, vocab-parallel cross-entropy (local stats, combine,
// gradient), bias column sums and dtype conversion.
//
// All are HBM-bound: 16-byte vectorised, coalesced row access (one warp per
// row for the [s, h] row kernels), warp-shuffle reductions, fp32 arithmetic,
// grids sized in multiples of the SM count.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>

#include "common.h"

namespace stp {
namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// 16-byte vector of T.
template <typename T>
struct Vec {
  static constexpr int N = 16 / sizeof(T);
  union {
    uint4 u;
    T v[N];
  };
  __device__ __forceinline__ void load(const T* p) { u = *reinterpret_cast<const uint4*>(p); }
  __device__ __forceinline__ void store(T* p) const { *reinterpret_cast<uint4*>(p) = u; }
  __device__ __forceinline__ float f(int i) const { return to_f<T>(v[i]); }
  __device__ __forceinline__ void set(int i, float x) { v[i] = from_f<T>(x); }
};

int grid_for(int64_t work_items, int items_per_block) {
  int64_t b = (work_items + items_per_block - 1) / items_per_block;
  int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// ---------------------------------------------------------------- RMSNorm
template <typename T>
__global__ void rmsnorm_fwd_kernel(int64_t rows, int h, const T* __restrict__ x, const T* __restrict__ resid,
                                   T* x_out, const T* __restrict__ g, float eps, T* y, float* rstd_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  constexpr int VN = Vec<T>::N;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    const T* xr = x + r * h;
    const T* rr = resid ? resid + r * h : nullptr;
    float ss = 0.f;
    for (int c = lane * VN; c < h; c += 32 * VN) {
      Vec<T> a;
      a.load(xr + c);
      if (rr) {
        Vec<T> b;
        b.load(rr + c);
#pragma unroll
        for (int i = 0; i < VN; ++i) a.set(i, a.f(i) + b.f(i));
        a.store(x_out + r * h + c);
      }
#pragma unroll
      for (int i = 0; i < VN; ++i) ss += a.f(i) * a.f(i);
    }
    ss = warp_sum(ss);
    const float rs = rsqrtf(ss / (float)h + eps);
    if (rstd_out && lane == 0) rstd_out[r] = rs;
    const T* src = rr ? x_out + r * h : xr;
    if (rr) __syncwarp();
    for (int c = lane * VN; c < h; c += 32 * VN) {
      Vec<T> a, gg, o;
      a.load(src + c);
      gg.load(g + c);
#pragma unroll
      for (int i = 0; i < VN; ++i) o.set(i, a.f(i) * rs * gg.f(i));
      o.store(y + r * h + c);
    }
  }
}

// Row-cached variant (h <= 32 * VN * NV): the row (x + resid) stays in
// registers for the normalisation pass instead of being re-read.
template <typename T, int NV>
__global__ void __launch_bounds__(256) rmsnorm_fwd_cached_kernel(int64_t rows, int h, const T* __restrict__ x,
                                                                  const T* __restrict__ resid, T* x_out,
                                                                  const T* __restrict__ g, float eps, T* y,
                                                                  float* rstd_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  constexpr int VN = Vec<T>::N;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    Vec<T> a[NV];
    float ss = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) a[v].load(x + r * h + c);
    }
    if (resid) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int c = (v * 32 + lane) * VN;
        if (c < h) {
          Vec<T> b;
          b.load(resid + r * h + c);
#pragma unroll
          for (int i = 0; i < VN; ++i) a[v].set(i, a[v].f(i) + b.f(i));
          a[v].store(x_out + r * h + c);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
#pragma unroll
        for (int i = 0; i < VN; ++i) ss += a[v].f(i) * a[v].f(i);
      }
    }
    ss = warp_sum(ss);
    const float rs = rsqrtf(ss / (float)h + eps);
    if (rstd_out && lane == 0) rstd_out[r] = rs;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
        Vec<T> gg, o;
        gg.load(g + c);
#pragma unroll
        for (int i = 0; i < VN; ++i) o.set(i, a[v].f(i) * rs * gg.f(i));
        o.store(y + r * h + c);
      }
    }
  }
}

// Row-per-CTA variants (round 2): 128 threads share a row, each holding
// RB_STEPS vectors of 4 elements in registers, a block-level reduction through
// shared memory.  The warp-per-row cached kernels above held a whole 3584-wide
// row per warp (175-200 registers per thread: one CTA of 8 warps per SM) and
// ran latency-bound at 2.1-2.2 TB/s (kbench, profiles/r02_kbench_elementwise.jsonl).
constexpr int RB_THREADS = 128;
constexpr int RB_STEPS = 8;  // h <= 128 * 4 * 8 = 4096

template <typename T>
struct V4 {  // 4 elements: 8 bytes (bf16) or 16 bytes (fp32)
  T v[4];
  __device__ __forceinline__ void load(const T* p) {
    if constexpr (sizeof(T) == 2) *reinterpret_cast<uint2*>(v) = *reinterpret_cast<const uint2*>(p);
    else *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(p);
  }
  __device__ __forceinline__ void store(T* p) const {
    if constexpr (sizeof(T) == 2) *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(v);
    else *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(v);
  }
  __device__ __forceinline__ float f(int i) const { return to_f<T>(v[i]); }
  __device__ __forceinline__ void set(int i, float x) { v[i] = from_f<T>(x); }
};

__device__ __forceinline__ float block_sum_128(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  const float t = red[0] + red[1] + red[2] + red[3];
  __syncthreads();  // red is reused by the next row
  return t;
}

template <typename T>
__global__ void __launch_bounds__(RB_THREADS) rmsnorm_fwd_rowblock_kernel(int64_t rows, int h, const T* __restrict__ x,
                                                                         const T* __restrict__ resid, T* x_out,
                                                                         const T* __restrict__ g, float eps, T* y,
                                                                         float* rstd_out) {
  __shared__ float red[4];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    V4<T> a[RB_STEPS];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < RB_STEPS; ++k) {
      const int c = (k * RB_THREADS + threadIdx.x) * 4;
      if (c < h) {
        a[k].load(x + r * h + c);
        if (resid) {
          V4<T> b;
          b.load(resid + r * h + c);
#pragma unroll
          for (int i = 0; i < 4; ++i) a[k].set(i, a[k].f(i) + b.f(i));
          a[k].store(x_out + r * h + c);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) ss += a[k].f(i) * a[k].f(i);
      }
    }
    const float rs = rsqrtf(block_sum_128(ss, red) / (float)h + eps);
    if (rstd_out && threadIdx.x == 0) rstd_out[r] = rs;
#pragma unroll
    for (int k = 0; k < RB_STEPS; ++k) {
      const int c = (k * RB_THREADS + threadIdx.x) * 4;
      if (c < h) {
        V4<T> gg, o;
        gg.load(g + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) o.set(i, a[k].f(i) * rs * gg.f(i));
        o.store(y + r * h + c);
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(RB_THREADS) rmsnorm_bwd_rowblock_kernel(int64_t rows, int h, const T* __restrict__ dy,
                                                                         const T* __restrict__ x,
                                                                         const T* __restrict__ g,
                                                                         const float* __restrict__ rstd,
                                                                         const T* dres, T* dx) {
  __shared__ float red[4];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float rs = rstd[r];
    V4<T> a[RB_STEPS], d[RB_STEPS];
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < RB_STEPS; ++k) {
      const int c = (k * RB_THREADS + threadIdx.x) * 4;
      if (c < h) {
        a[k].load(x + r * h + c);
        d[k].load(dy + r * h + c);
        V4<T> gg;
        gg.load(g + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) dot += gg.f(i) * d[k].f(i) * a[k].f(i);
      }
    }
    const float kk = rs * rs * rs * block_sum_128(dot, red) / (float)h;
#pragma unroll
    for (int k = 0; k < RB_STEPS; ++k) {
      const int c = (k * RB_THREADS + threadIdx.x) * 4;
      if (c < h) {
        V4<T> gg, o, q;
        gg.load(g + c);
        if (dres) q.load(dres + r * h + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float v = rs * gg.f(i) * d[k].f(i) - a[k].f(i) * kk;
          if (dres) v += q.f(i);
          o.set(i, v);
        }
        o.store(dx + r * h + c);
      }
    }
  }
}

// dgamma partials accumulate in shared memory, flushed once per block.
// dgamma[c] += sum_rows dy * x * rstd: one thread per column, a block of
// rows per blockIdx.y (coalesced across threads), one atomic per column.
template <typename T>
__global__ void rmsnorm_dgamma_kernel(int64_t rows, int h, const T* __restrict__ dy, const T* __restrict__ x,
                                      const float* __restrict__ rstd, float* dgamma, int64_t rows_per_block) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float acc = 0.f;
  for (int64_t r = r0; r < r1; ++r) acc += to_f<T>(dy[r * h + c]) * to_f<T>(x[r * h + c]) * rstd[r];
  atomicAdd(&dgamma[c], acc);
}

// Vectorised column reductions: one thread = VN consecutive columns (16-byte
// loads), a block of rows per blockIdx.y, one fp32 atomic per column.
template <typename T>
__global__ void rmsnorm_dgamma_vec_kernel(int64_t rows, int h, const T* __restrict__ dy, const T* __restrict__ x,
                                          const float* __restrict__ rstd, float* dgamma, int64_t rows_per_block) {
  constexpr int VN = Vec<T>::N;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * VN;
  if (c >= h) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float acc[VN];
#pragma unroll
  for (int i = 0; i < VN; ++i) acc[i] = 0.f;
#pragma unroll 4
  for (int64_t r = r0; r < r1; ++r) {
    Vec<T> a, b;
    a.load(dy + r * h + c);
    b.load(x + r * h + c);
    const float rs = rstd[r];
#pragma unroll
    for (int i = 0; i < VN; ++i) acc[i] = fmaf(a.f(i) * b.f(i), rs, acc[i]);
  }
#pragma unroll
  for (int i = 0; i < VN; ++i) atomicAdd(&dgamma[c + i], acc[i]);
}

template <typename T>
__global__ void colsum_vec_kernel(int64_t rows, int64_t n, const T* __restrict__ X, int64_t ld, float* acc,
                                  int64_t rows_per_block) {
  constexpr int VN = Vec<T>::N;
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VN;
  if (c >= n) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float sum[VN];
#pragma unroll
  for (int i = 0; i < VN; ++i) sum[i] = 0.f;
#pragma unroll 4
  for (int64_t r = r0; r < r1; ++r) {
    Vec<T> a;
    a.load(X + r * ld + c);
#pragma unroll
    for (int i = 0; i < VN; ++i) sum[i] += a.f(i);
  }
#pragma unroll
  for (int i = 0; i < VN; ++i) atomicAdd(&acc[c + i], sum[i]);
}

template <typename T>
__global__ void rmsnorm_bwd_kernel(int64_t rows, int h, const T* __restrict__ dy, const T* __restrict__ x,
                                   const T* __restrict__ g, const float* __restrict__ rstd,
                                   const T* dres, T* dx, float* dgamma) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  constexpr int VN = Vec<T>::N;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    const float rs = rstd[r];
    float dot = 0.f;
    for (int c = lane * VN; c < h; c += 32 * VN) {
      Vec<T> a, d, gg;
      a.load(x + r * h + c);
      d.load(dy + r * h + c);
      gg.load(g + c);
#pragma unroll
      for (int i = 0; i < VN; ++i) dot += gg.f(i) * d.f(i) * a.f(i);
    }
    dot = warp_sum(dot) / (float)h;
    const float k = rs * rs * rs * dot;
    for (int c = lane * VN; c < h; c += 32 * VN) {
      Vec<T> a, d, gg, o;
      a.load(x + r * h + c);
      d.load(dy + r * h + c);
      gg.load(g + c);
      Vec<T> rr;
      if (dres) rr.load(dres + r * h + c);
#pragma unroll
      for (int i = 0; i < VN; ++i) {
        float v = rs * gg.f(i) * d.f(i) - a.f(i) * k;
        if (dres) v += rr.f(i);
        o.set(i, v);
      }
      o.store(dx + r * h + c);
    }
  }
  (void)dgamma;
}

// Row-cached variant (h <= 32 * VN * NV): x and dy of the row stay in
// registers between the reduction and the output pass, so each is read from
// HBM once (the two-pass kernel above re-reads both).
template <typename T, int NV>
__global__ void __launch_bounds__(256) rmsnorm_bwd_cached_kernel(int64_t rows, int h, const T* __restrict__ dy,
                                                                  const T* __restrict__ x, const T* __restrict__ g,
                                                                  const float* __restrict__ rstd, const T* dres,
                                                                  T* dx) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  constexpr int VN = Vec<T>::N;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    const float rs = rstd[r];
    Vec<T> a[NV], d[NV];
    float dot = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
        a[v].load(x + r * h + c);
        d[v].load(dy + r * h + c);
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
        Vec<T> gg;
        gg.load(g + c);
#pragma unroll
        for (int i = 0; i < VN; ++i) dot += gg.f(i) * d[v].f(i) * a[v].f(i);
      }
    }
    dot = warp_sum(dot) / (float)h;
    const float k = rs * rs * rs * dot;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
        Vec<T> gg, o, rr;
        gg.load(g + c);
        if (dres) rr.load(dres + r * h + c);
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          float val = rs * gg.f(i) * d[v].f(i) - a[v].f(i) * k;
          if (dres) val += rr.f(i);
          o.set(i, val);
        }
        o.store(dx + r * h + c);
      }
    }
  }
}

// ------------------------------------------------------------------- RoPE
// cos/sin of pos * theta^(-2j/d), j < d/2, evaluated once in fp64 per
// (s, d, theta, pos0) and cached on the device as float2 [s][d/2].
__global__ void rope_table_kernel(int64_t s, int half, int d, double theta, int64_t pos0, float2* tab) {
  const int64_t total = s * half;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % half);
    const int64_t row = i / half;
    const double inv = pow(theta, -2.0 * (double)j / (double)d);
    double sn, cs;
    sincos((double)(pos0 + row) * inv, &sn, &cs);
    tab[i] = make_float2((float)cs, (float)sn);
  }
}

// one thread = 4 consecutive rotation pairs (j..j+3 with their partners j+d/2..)
template <typename T>
__global__ void rope_kernel(int64_t s, int64_t ld, int64_t col0, int nh, int d, const float2* __restrict__ tab,
                            int backward, T* x) {
  const int half = d / 2, q4 = half / 4;
  const int64_t total = s * nh * q4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % q4) * 4;
    const int64_t t = i / q4;
    const int hd = (int)(t % nh);
    const int64_t row = t / nh;
    T* p = x + row * ld + col0 + (int64_t)hd * d;
    const float2* cs = tab + row * half + j;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float c = cs[e].x, sv = cs[e].y;
      const float x1 = to_f<T>(p[j + e]), x2 = to_f<T>(p[j + e + half]);
      float y1, y2;
      if (!backward) {
        y1 = x1 * c - x2 * sv;
        y2 = x2 * c + x1 * sv;
      } else {
        y1 = x1 * c + x2 * sv;
        y2 = x2 * c - x1 * sv;
      }
      p[j + e] = from_f<T>(y1);
      p[j + e + half] = from_f<T>(y2);
    }
  }
}

// Vectorised variant: one thread = VN consecutive rotation pairs (16-byte
// loads / stores of both halves, float2 table rows through L2).  Needs
// 16-byte aligned rows (ld, col0 multiples of VN) and half % VN == 0.
template <typename T>
__global__ void rope_vec_kernel(int64_t s, int64_t ld, int64_t col0, int nh, int d, const float2* __restrict__ tab,
                                int backward, T* x) {
  constexpr int VN = Vec<T>::N;
  const int half = d / 2, qv = half / VN;
  const int64_t total = s * nh * qv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % qv) * VN;
    const int64_t t = i / qv;
    const int hd = (int)(t % nh);
    const int64_t row = t / nh;
    T* p = x + row * ld + col0 + (int64_t)hd * d + j;
    const float4* cs = reinterpret_cast<const float4*>(tab + row * half + j);  // VN float2 = VN/2 float4
    Vec<T> a, b;
    a.load(p);
    b.load(p + half);
    const float sg = backward ? -1.f : 1.f;
#pragma unroll
    for (int e = 0; e < VN; e += 2) {
      const float4 c2 = cs[e / 2];  // (cos_e, sin_e, cos_e+1, sin_e+1)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float c = k ? c2.z : c2.x, sv = sg * (k ? c2.w : c2.y);
        const float x1 = a.f(e + k), x2 = b.f(e + k);
        a.set(e + k, x1 * c - x2 * sv);
        b.set(e + k, x2 * c + x1 * sv);
      }
    }
    a.store(p);
    b.store(p + half);
  }
}

// ----------------------------------------------------------------- SwiGLU
__device__ __forceinline__ float sigm(float z) { return 1.f / (1.f + __expf(-z)); }

template <typename T>
__global__ void swiglu_fwd_kernel(int64_t s, int64_t I, const T* __restrict__ gu, T* H) {
  constexpr int VN = Vec<T>::N;
  const int64_t nv = I / VN;
  const int64_t total = s * nv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / nv, c = (i % nv) * VN;
    Vec<T> G, U, o;
    G.load(gu + r * 2 * I + c);
    U.load(gu + r * 2 * I + I + c);
#pragma unroll
    for (int k = 0; k < VN; ++k) {
      const float z = G.f(k);
      o.set(k, z * sigm(z) * U.f(k));
    }
    o.store(H + r * I + c);
  }
}

template <typename T>
__global__ void swiglu_bwd_kernel(int64_t s, int64_t I, const T* __restrict__ dH, const T* gu,
                                  T* dgu) {
  constexpr int VN = Vec<T>::N;
  const int64_t nv = I / VN;
  const int64_t total = s * nv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / nv, c = (i % nv) * VN;
    Vec<T> G, U, D, dG, dU;
    G.load(gu + r * 2 * I + c);
    U.load(gu + r * 2 * I + I + c);
    D.load(dH + r * I + c);
#pragma unroll
    for (int k = 0; k < VN; ++k) {
      const float z = G.f(k), sg = sigm(z), dh = D.f(k);
      dU.set(k, dh * z * sg);
      dG.set(k, dh * U.f(k) * sg * (1.f + z * (1.f - sg)));
    }
    dG.store(dgu + r * 2 * I + c);
    dU.store(dgu + r * 2 * I + I + c);
  }
}

// -------------------------------------------------------------- embedding
template <typename T>
__global__ void embed_fwd_kernel(int64_t s, int h, const int32_t* __restrict__ tok, int64_t v0, int64_t Vl,
                                 const T* __restrict__ E, T* out) {
  constexpr int VN = Vec<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t r = warp0; r < s; r += nwarps) {
    const int64_t t = (int64_t)tok[r] - v0;
    const bool own = t >= 0 && t < Vl;
    for (int c = lane * VN; c < h; c += 32 * VN) {
      Vec<T> a;
      if (own) a.load(E + t * h + c);
      else a.u = make_uint4(0, 0, 0, 0);
      a.store(out + r * h + c);
    }
  }
}

template <typename T>
__global__ void embed_bwd_kernel(int64_t s, int h, const int32_t* __restrict__ tok, int64_t v0, int64_t Vl,
                                 const T* __restrict__ dX, float* dE) {
  const int64_t total = s * h;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / h, c = i % h;
    const int64_t t = (int64_t)tok[r] - v0;
    if (t >= 0 && t < Vl) atomicAdd(&dE[t * h + c], to_f<T>(dX[i]));
  }
}

// ---------------------------------------------------------- cross-entropy
template <typename T>
__global__ void ce_stats_kernel(int64_t s, int64_t Vl, const T* __restrict__ logits, int64_t ld,
                                const int32_t* __restrict__ tgt, int64_t v0, float* stats) {
  __shared__ float sm[32], ssum[32];
  for (int64_t r = blockIdx.x; r < s; r += gridDim.x) {
    const T* z = logits + r * ld;
    float m = -INFINITY, sum = 0.f;
    constexpr int VN = Vec<T>::N;
    if (Vl % VN == 0 && ld % VN == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0) {
      // 16-byte vectors: one running-max update per vector
      for (int64_t j = (int64_t)threadIdx.x * VN; j < Vl; j += (int64_t)blockDim.x * VN) {
        Vec<T> x;
        x.load(z + j);
        float vm = x.f(0);
#pragma unroll
        for (int i = 1; i < VN; ++i) vm = fmaxf(vm, x.f(i));
        if (vm > m) {
          sum = (m == -INFINITY) ? 0.f : sum * __expf(m - vm);
          m = vm;
        }
#pragma unroll
        for (int i = 0; i < VN; ++i) sum += __expf(x.f(i) - m);
      }
    } else {
      for (int64_t j = threadIdx.x; j < Vl; j += blockDim.x) {
        const float v = to_f<T>(z[j]);
        if (v > m) {
          sum = sum * __expf(m - v) + 1.f;
          m = v;
        } else {
          sum += __expf(v - m);
        }
      }
    }
    // warp combine (m, sum)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, m, o), so = __shfl_xor_sync(0xffffffffu, sum, o);
      const float mn = fmaxf(m, mo);
      sum = (m == -INFINITY ? 0.f : sum * __expf(m - mn)) + (mo == -INFINITY ? 0.f : so * __expf(mo - mn));
      m = mn;
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0) {
      sm[w] = m;
      ssum[w] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float M = -INFINITY;
      for (int i = 0; i < nw; ++i) M = fmaxf(M, sm[i]);
      float S = 0.f;
      for (int i = 0; i < nw; ++i)
        if (sm[i] != -INFINITY) S += ssum[i] * __expf(sm[i] - M);
      const int64_t t = (int64_t)tgt[r] - v0;
      stats[r * 3 + 0] = M;
      stats[r * 3 + 1] = S;
      stats[r * 3 + 2] = (t >= 0 && t < Vl) ? to_f<T>(z[t]) : 0.f;
    }
    __syncthreads();
  }
}

__global__ void ce_combine_kernel(int64_t s, int t, const float* __restrict__ st, float* lse, float* loss_acc,
                                  float scale) {
  float local = 0.f;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < s; r += (int64_t)gridDim.x * blockDim.x) {
    float M = -INFINITY;
    for (int q = 0; q < t; ++q) M = fmaxf(M, st[((int64_t)q * s + r) * 3]);
    float Z = 0.f, tl = 0.f;
    for (int q = 0; q < t; ++q) {
      const float* p = st + ((int64_t)q * s + r) * 3;
      Z += p[1] * __expf(p[0] - M);
      tl += p[2];
    }
    const float l = M + logf(Z);
    lse[r] = l;
    local += l - tl;
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0) atomicAdd(loss_acc, local * scale);
}

template <typename T>
__global__ void ce_grad_kernel(int64_t s, int64_t Vl, T* logits, int64_t ld, const int32_t* __restrict__ tgt,
                               int64_t v0, const float* __restrict__ lse, float scale) {
  for (int64_t r = blockIdx.x; r < s; r += gridDim.x) {
    T* z = logits + r * ld;
    const float l = lse[r];
    const int64_t t = (int64_t)tgt[r] - v0;
    constexpr int VN = Vec<T>::N;
    if (Vl % VN == 0 && ld % VN == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0) {  // 16-byte vectors
      for (int64_t j = (int64_t)threadIdx.x * VN; j < Vl; j += (int64_t)blockDim.x * VN) {
        Vec<T> x;
        x.load(z + j);
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          float p = __expf(x.f(i) - l);
          if (j + i == t) p -= 1.f;
          x.set(i, p * scale);
        }
        x.store(z + j);
      }
    } else {
      for (int64_t j = threadIdx.x; j < Vl; j += blockDim.x) {
        float p = __expf(to_f<T>(z[j]) - l);
        if (j == t) p -= 1.f;
        z[j] = from_f<T>(p * scale);
      }
    }
  }
}

// ------------------------------------------------------------- misc
template <typename T>
__global__ void colsum_kernel(int64_t rows, int64_t n, const T* __restrict__ X, int64_t ld, float* acc,
                              int64_t rows_per_block) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += to_f<T>(X[r * ld + c]);
  atomicAdd(&acc[c], s);
}

template <typename S, typename D>
__global__ void convert_kernel(int64_t n, const S* __restrict__ src, D* dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = from_f<D>(to_f<S>(src[i]));
}

template <typename T>
__global__ void add_kernel(int64_t n, const T* __restrict__ a, const T* __restrict__ b, T* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = from_f<T>(to_f<T>(a[i]) + to_f<T>(b[i]));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename T>
stp_status launch_dgamma(int64_t rows, int64_t h, const T* dy, const T* x, const float* rstd, float* dgamma,
                         cudaStream_t st) {
  constexpr int VN = Vec<T>::N;
  // The vectorised variant measured slower in the step (launch list: 1.07% vs
  // 0.64% of the step for the column-per-thread kernel): kept opt-in.
  static const bool vec = getenv("STP_DGAMMA_VEC") != nullptr;
  if (vec && h % VN == 0 && aligned16(dy) && aligned16(x)) {
    const int64_t rpb = 64;
    dim3 grid((unsigned)((h / VN + 127) / 128), (unsigned)((rows + rpb - 1) / rpb));
    rmsnorm_dgamma_vec_kernel<T><<<grid, 128, 0, st>>>(rows, (int)h, dy, x, rstd, dgamma, rpb);
  } else {
    const int64_t rpb = 128;
    dim3 grid2((unsigned)((h + 255) / 256), (unsigned)((rows + rpb - 1) / rpb));
    rmsnorm_dgamma_kernel<T><<<grid2, 256, 0, st>>>(rows, (int)h, dy, x, rstd, dgamma, rpb);
  }
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

}  // namespace

// Shared launchers (also used by the executor).
stp_status rmsnorm_fwd(int dtype, int64_t rows, int64_t h, const void* x, const void* resid, void* x_out,
                       const void* g, float eps, void* y, float* rstd, cudaStream_t st) {
  STP_CHECK_ARG(h % 8 == 0, "hidden % 8 == 0");
  STP_CHECK_ARG(aligned16(x) && aligned16(y) && aligned16(g), "16-byte aligned rows");
  STP_CHECK_ARG(!resid || x_out, "resid needs x_out");
  if (rows == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    constexpr int VN = Vec<T>::N;
    if (h <= RB_THREADS * 4 * RB_STEPS && h % 4 == 0)
      rmsnorm_fwd_rowblock_kernel<T><<<(unsigned)std::min<int64_t>(rows, (int64_t)num_sms() * 16), RB_THREADS, 0, st>>>(
          rows, (int)h, (const T*)x, (const T*)resid, (T*)x_out, (const T*)g, eps, (T*)y, rstd);
    else if (h <= 32 * VN * 16)
      rmsnorm_fwd_cached_kernel<T, 16><<<grid_for(rows, kWarpsPerBlock), 32 * kWarpsPerBlock, 0, st>>>(
          rows, (int)h, (const T*)x, (const T*)resid, (T*)x_out, (const T*)g, eps, (T*)y, rstd);
    else
      rmsnorm_fwd_kernel<T><<<grid_for(rows, kWarpsPerBlock), 32 * kWarpsPerBlock, 0, st>>>(
          rows, (int)h, (const T*)x, (const T*)resid, (T*)x_out, (const T*)g, eps, (T*)y, rstd);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status rmsnorm_bwd(int dtype, int64_t rows, int64_t h, const void* dy, const void* x, const void* g,
                       const float* rstd, const void* dres, void* dx, float* dgamma, cudaStream_t st) {
  STP_CHECK_ARG(h % 8 == 0, "hidden % 8 == 0");
  if (rows == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    if (dgamma) {  // before dx: dx may alias dres, never dy / x
      STP_TRY(launch_dgamma<T>(rows, h, (const T*)dy, (const T*)x, rstd, dgamma, st));
    }
    constexpr int VN = Vec<T>::N;
    if (h <= RB_THREADS * 4 * RB_STEPS && h % 4 == 0)
      rmsnorm_bwd_rowblock_kernel<T><<<(unsigned)std::min<int64_t>(rows, (int64_t)num_sms() * 16), RB_THREADS, 0, st>>>(
          rows, (int)h, (const T*)dy, (const T*)x, (const T*)g, rstd, (const T*)dres, (T*)dx);
    else if (h <= 32 * VN * 16)
      rmsnorm_bwd_cached_kernel<T, 16><<<grid_for(rows, kWarpsPerBlock), 32 * kWarpsPerBlock, 0, st>>>(
          rows, (int)h, (const T*)dy, (const T*)x, (const T*)g, rstd, (const T*)dres, (T*)dx);
    else
      rmsnorm_bwd_kernel<T><<<grid_for(rows, kWarpsPerBlock), 32 * kWarpsPerBlock, 0, st>>>(
          rows, (int)h, (const T*)dy, (const T*)x, (const T*)g, rstd, (const T*)dres, (T*)dx, nullptr);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

// dgamma[c] += sum_rows dy * x * rstd (the W-type gamma partial of an
// RMSNorm backward whose dx was produced elsewhere, e.g. by the fused TP
// comm-phase kernel in tpcomm.cu).
stp_status rmsnorm_dgamma(int dtype, int64_t rows, int64_t h, const void* dy, const void* x, const float* rstd,
                          float* dgamma, cudaStream_t st) {
  if (rows == 0 || !dgamma) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    return launch_dgamma<T>(rows, h, (const T*)dy, (const T*)x, rstd, dgamma, st);
  });
}

struct RopeKey {
  int dev;
  int64_t s;
  int d;
  float theta;
  int64_t pos0;
  bool operator<(const RopeKey& o) const {
    return std::tie(dev, s, d, theta, pos0) < std::tie(o.dev, o.s, o.d, o.theta, o.pos0);
  }
};

stp_status rope_with_table(int dtype, int backward, int64_t s, int64_t ld, int64_t col0, int nh, int d,
                           const float2* tab, void* x, cudaStream_t st);

stp_status rope(int dtype, int backward, int64_t s, int64_t ld, int64_t col0, int nh, int d, float theta,
                int64_t pos0, void* x, cudaStream_t st) {
  STP_CHECK_ARG(d % 8 == 0, "head_dim % 8 == 0");
  if (s == 0 || nh == 0) return STP_OK;
  static std::mutex mu;
  static std::map<RopeKey, float2*> tables;  // device tables, kept for the process lifetime
  int dev = 0;
  STP_CUDA_TRY(cudaGetDevice(&dev));
  float2* tab = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    RopeKey key{dev, s, d, theta, pos0};
    auto it = tables.find(key);
    if (it == tables.end()) {
      STP_CUDA_TRY(cudaMalloc(&tab, (size_t)s * (d / 2) * sizeof(float2)));
      rope_table_kernel<<<grid_for(s * (d / 2), 256), 256, 0, st>>>(s, d / 2, d, (double)theta, pos0, tab);
      count_launch();
      STP_LAUNCH_CHECK();
      tables[key] = tab;
    } else {
      tab = it->second;
    }
  }
  return rope_with_table(dtype, backward, s, ld, col0, nh, d, tab, x, st);
}

// Rotate-half RoPE with a caller-built cos/sin table [s][d/2] (1-D positions
// above; the 2-D vision table of vit.cu).
stp_status rope_with_table(int dtype, int backward, int64_t s, int64_t ld, int64_t col0, int nh, int d,
                           const float2* tab, void* x, cudaStream_t st) {
  return STP_DISPATCH_DTYPE(dtype, [&] {
    constexpr int VN = Vec<T>::N;
    if ((d / 2) % VN == 0 && ld % VN == 0 && col0 % VN == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0)
      rope_vec_kernel<T><<<grid_for(s * nh * (d / 2 / VN), 256), 256, 0, st>>>(s, ld, col0, nh, d, tab, backward,
                                                                               (T*)x);
    else
      rope_kernel<T><<<grid_for(s * nh * (d / 8), 256), 256, 0, st>>>(s, ld, col0, nh, d, tab, backward, (T*)x);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status swiglu_fwd(int dtype, int64_t s, int64_t I, const void* gu, void* H, cudaStream_t st) {
  STP_CHECK_ARG(I % 8 == 0, "ffn shard % 8 == 0");
  if (s == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    swiglu_fwd_kernel<T><<<grid_for(s * I / Vec<T>::N, 256), 256, 0, st>>>(s, I, (const T*)gu, (T*)H);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status swiglu_bwd(int dtype, int64_t s, int64_t I, const void* dH, const void* gu, void* dgu, cudaStream_t st) {
  STP_CHECK_ARG(I % 8 == 0, "ffn shard % 8 == 0");
  if (s == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    swiglu_bwd_kernel<T><<<grid_for(s * I / Vec<T>::N, 256), 256, 0, st>>>(s, I, (const T*)dH, (const T*)gu,
                                                                            (T*)dgu);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status embed_fwd(int dtype, int64_t s, int64_t h, const int32_t* tok, int64_t v0, int64_t Vl, const void* E,
                     void* out, cudaStream_t st) {
  STP_CHECK_ARG(h % 8 == 0, "hidden % 8 == 0");
  if (s == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    embed_fwd_kernel<T><<<grid_for(s, kWarpsPerBlock), 32 * kWarpsPerBlock, 0, st>>>(s, (int)h, tok, v0, Vl,
                                                                                      (const T*)E, (T*)out);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status embed_bwd(int dtype, int64_t s, int64_t h, const int32_t* tok, int64_t v0, int64_t Vl, const void* dX,
                     float* dE, cudaStream_t st) {
  if (s == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    embed_bwd_kernel<T><<<grid_for(s * h, 256), 256, 0, st>>>(s, (int)h, tok, v0, Vl, (const T*)dX, dE);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status ce_stats(int dtype, int64_t s, int64_t Vl, const void* logits, int64_t ld, const int32_t* tgt, int64_t v0,
                    float* stats, cudaStream_t st) {
  if (s == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    ce_stats_kernel<T><<<(int)std::min<int64_t>(s, 16 * num_sms()), 512, 0, st>>>(s, Vl, (const T*)logits, ld, tgt,
                                                                                   v0, stats);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status ce_combine(int64_t s, int t, const float* stats_all, float* lse, float* loss_acc, float scale,
                      cudaStream_t st) {
  if (s == 0) return STP_OK;
  ce_combine_kernel<<<grid_for(s, 256), 256, 0, st>>>(s, t, stats_all, lse, loss_acc, scale);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

stp_status ce_grad(int dtype, int64_t s, int64_t Vl, void* logits, int64_t ld, const int32_t* tgt, int64_t v0,
                   const float* lse, float scale, cudaStream_t st) {
  if (s == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    ce_grad_kernel<T><<<(int)std::min<int64_t>(s, 16 * num_sms()), 512, 0, st>>>(s, Vl, (T*)logits, ld, tgt, v0, lse,
                                                                                  scale);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status colsum_acc(int dtype, int64_t rows, int64_t n, const void* X, int64_t ld, float* acc, cudaStream_t st) {
  if (rows == 0 || n == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    constexpr int VN = Vec<T>::N;
    if (n % VN == 0 && ld % VN == 0 && aligned16(X)) {
      const int64_t rpb = 64;
      dim3 grid((unsigned)((n / VN + 255) / 256), (unsigned)((rows + rpb - 1) / rpb));
      colsum_vec_kernel<T><<<grid, 256, 0, st>>>(rows, n, (const T*)X, ld, acc, rpb);
    } else {
      const int64_t rpb = 256;
      dim3 grid((unsigned)((n + 255) / 256), (unsigned)((rows + rpb - 1) / rpb));
      colsum_kernel<T><<<grid, 256, 0, st>>>(rows, n, (const T*)X, ld, acc, rpb);
    }
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status convert(int sd, int dd, int64_t n, const void* src, void* dst, cudaStream_t st) {
  if (n == 0) return STP_OK;
  const int grid = grid_for(n, 256);
  if (sd == STP_DTYPE_F32 && dd == STP_DTYPE_BF16)
    convert_kernel<float, bf16><<<grid, 256, 0, st>>>(n, (const float*)src, (bf16*)dst);
  else if (sd == STP_DTYPE_BF16 && dd == STP_DTYPE_F32)
    convert_kernel<bf16, float><<<grid, 256, 0, st>>>(n, (const bf16*)src, (float*)dst);
  else if (sd == STP_DTYPE_F32 && dd == STP_DTYPE_F32)
    convert_kernel<float, float><<<grid, 256, 0, st>>>(n, (const float*)src, (float*)dst);
  else if (sd == STP_DTYPE_BF16 && dd == STP_DTYPE_BF16)
    convert_kernel<bf16, bf16><<<grid, 256, 0, st>>>(n, (const bf16*)src, (bf16*)dst);
  else
    return fail(STP_EINVAL, "convert dtype");
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

// out = a + b (residual add without a norm, the chunk's last layer).
stp_status add(int dtype, int64_t n, const void* a, const void* b, void* out, cudaStream_t st) {
  if (n == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    add_kernel<T><<<grid_for(n, 256), 256, 0, st>>>(n, (const T*)a, (const T*)b, (T*)out);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

}  // namespace stp

extern "C" {

stp_status stp_op_rmsnorm_fwd(int32_t dtype, int64_t rows, int64_t h, const void* x, const void* resid, void* x_out,
                              const void* gamma, float eps, void* y, float* rstd_out, void* stream) {
  return stp::rmsnorm_fwd(dtype, rows, h, x, resid, x_out, gamma, eps, y, rstd_out, (cudaStream_t)stream);
}
stp_status stp_op_rmsnorm_bwd(int32_t dtype, int64_t rows, int64_t h, const void* dy, const void* x,
                              const void* gamma, const float* rstd, const void* dres, void* dx, float* dgamma_acc,
                              void* stream) {
  return stp::rmsnorm_bwd(dtype, rows, h, dy, x, gamma, rstd, dres, dx, dgamma_acc, (cudaStream_t)stream);
}
stp_status stp_op_rope(int32_t dtype, int32_t backward, int64_t s, int64_t ld, int64_t col0, int32_t n_heads,
                       int32_t d, float theta, int64_t pos0, void* x, void* stream) {
  return stp::rope(dtype, backward, s, ld, col0, n_heads, d, theta, pos0, x, (cudaStream_t)stream);
}
stp_status stp_op_swiglu_fwd(int32_t dtype, int64_t s, int64_t I, const void* gu, void* H, void* stream) {
  return stp::swiglu_fwd(dtype, s, I, gu, H, (cudaStream_t)stream);
}
stp_status stp_op_swiglu_bwd(int32_t dtype, int64_t s, int64_t I, const void* dH, const void* gu, void* dgu,
                             void* stream) {
  return stp::swiglu_bwd(dtype, s, I, dH, gu, dgu, (cudaStream_t)stream);
}
stp_status stp_op_embed_fwd(int32_t dtype, int64_t s, int64_t h, const int32_t* tok, int64_t v0, int64_t Vl,
                            const void* E, void* out, void* stream) {
  return stp::embed_fwd(dtype, s, h, tok, v0, Vl, E, out, (cudaStream_t)stream);
}
stp_status stp_op_embed_bwd(int32_t dtype, int64_t s, int64_t h, const int32_t* tok, int64_t v0, int64_t Vl,
                            const void* dX, float* dE_acc, void* stream) {
  return stp::embed_bwd(dtype, s, h, tok, v0, Vl, dX, dE_acc, (cudaStream_t)stream);
}
stp_status stp_op_ce_stats(int32_t dtype, int64_t s, int64_t Vl, const void* logits, int64_t ld, const int32_t* tgt,
                           int64_t v0, float* stats, void* stream) {
  return stp::ce_stats(dtype, s, Vl, logits, ld, tgt, v0, stats, (cudaStream_t)stream);
}
stp_status stp_op_ce_combine(int64_t s, int32_t t, const float* stats_all, float* lse, float* loss_acc,
                             float loss_scale, void* stream) {
  return stp::ce_combine(s, t, stats_all, lse, loss_acc, loss_scale, (cudaStream_t)stream);
}
stp_status stp_op_ce_grad(int32_t dtype, int64_t s, int64_t Vl, void* logits, int64_t ld, const int32_t* tgt,
                          int64_t v0, const float* lse, float grad_scale, void* stream) {
  return stp::ce_grad(dtype, s, Vl, logits, ld, tgt, v0, lse, grad_scale, (cudaStream_t)stream);
}
stp_status stp_op_colsum_acc(int32_t dtype, int64_t rows, int64_t n, const void* X, int64_t ld, float* acc,
                             void* stream) {
  return stp::colsum_acc(dtype, rows, n, X, ld, acc, (cudaStream_t)stream);
}
stp_status stp_op_convert(int32_t src_dtype, int32_t dst_dtype, int64_t n, const void* src, void* dst,
                          void* stream) {
  return stp::convert(src_dtype, dst_dtype, n, src, dst, (cudaStream_t)stream);
}

}  // extern "C"
