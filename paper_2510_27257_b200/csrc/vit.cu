// Memory-bound kernels of the MLLM's ViT first chunk (§5 P:L171 "the
// ViT encoder is assigned to the first virtual stage on device 0"; Table 3
// P:L231-263; math: oracle/vit.py):
//   LayerNorm fwd / bwd with the fused residual add of the SP comm phase
//     y = g (x - mu) r + b,  r = (var + eps)^(-1/2)
//     dx = r (g dy - mean(g dy) - xhat mean(g dy xhat)) (+ dres),  xhat = (x - mu) r
//   LayerNorm parameter gradients  dg += sum_rows dy xhat,  db += sum_rows dy
//   QuickGELU  h = a sigmoid(1.702 a)      (ViT MLP)
//   GELU (erf) h = z Phi(z)                (2x2 merger MLP)
//   2-D vision RoPE table (rotate-half; angles [h pos * inv | w pos * inv],
//     patches in 2x2 merge-window order), applied by the RoPE kernels of
//     elementwise.cu.
// Row kernels: one warp per row, the row cached in registers (h <= 32 * VN *
// 16), 16-byte vectors, warp-shuffle reductions, fp32 statistics.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.h"

namespace stp {
namespace {

constexpr int kWarps = 8;
constexpr int kNV = 16;

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
struct V16 {
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

int blocks_for(int64_t items, int per_block) {
  int64_t b = (items + per_block - 1) / per_block;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)std::max<int64_t>(1, std::min(b, cap));
}

// x (+ resid -> x_out) -> y = g (x - mu) r + b; mean / rstd fp32 per row (nullable).
template <typename T>
__global__ void __launch_bounds__(256) ln_fwd_kernel(int64_t rows, int h, const T* __restrict__ x,
                                                      const T* __restrict__ resid, T* x_out, const T* __restrict__ g,
                                                      const T* __restrict__ b, float eps, T* y, float* mean_out,
                                                      float* rstd_out) {
  const int lane = threadIdx.x & 31;
  constexpr int VN = V16<T>::N;
  for (int64_t r = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * kWarps) {
    V16<T> a[kNV];
    float s1 = 0.f;
#pragma unroll
    for (int v = 0; v < kNV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
        a[v].load(x + r * h + c);
        if (resid) {
          V16<T> q;
          q.load(resid + r * h + c);
#pragma unroll
          for (int i = 0; i < VN; ++i) a[v].set(i, a[v].f(i) + q.f(i));
          a[v].store(x_out + r * h + c);
        }
#pragma unroll
        for (int i = 0; i < VN; ++i) s1 += a[v].f(i);
      }
    }
    const float mu = wsum(s1) / (float)h;
    float s2 = 0.f;
#pragma unroll
    for (int v = 0; v < kNV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          const float d = a[v].f(i) - mu;
          s2 += d * d;
        }
      }
    }
    const float rs = rsqrtf(wsum(s2) / (float)h + eps);
    if (lane == 0) {
      if (mean_out) mean_out[r] = mu;
      if (rstd_out) rstd_out[r] = rs;
    }
#pragma unroll
    for (int v = 0; v < kNV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
        V16<T> gg, bb, o;
        gg.load(g + c);
        bb.load(b + c);
#pragma unroll
        for (int i = 0; i < VN; ++i) o.set(i, (a[v].f(i) - mu) * rs * gg.f(i) + bb.f(i));
        o.store(y + r * h + c);
      }
    }
  }
}

// dx = r (g dy - mean(g dy) - xhat mean(g dy xhat)) (+ dres)
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_kernel(int64_t rows, int h, const T* __restrict__ dy,
                                                      const T* __restrict__ x, const T* __restrict__ g,
                                                      const float* __restrict__ mean, const float* __restrict__ rstd,
                                                      const T* dres, T* dx) {
  const int lane = threadIdx.x & 31;
  constexpr int VN = V16<T>::N;
  for (int64_t r = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * kWarps) {
    const float mu = mean[r], rs = rstd[r];
    V16<T> a[kNV], d[kNV];
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int v = 0; v < kNV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
        a[v].load(x + r * h + c);
        d[v].load(dy + r * h + c);
        V16<T> gg;
        gg.load(g + c);
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          const float gd = gg.f(i) * d[v].f(i);
          sg += gd;
          sgx += gd * (a[v].f(i) - mu) * rs;
        }
      }
    }
    const float mg = wsum(sg) / (float)h, mgx = wsum(sgx) / (float)h;
#pragma unroll
    for (int v = 0; v < kNV; ++v) {
      const int c = (v * 32 + lane) * VN;
      if (c < h) {
        V16<T> gg, o, q;
        gg.load(g + c);
        if (dres) q.load(dres + r * h + c);
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          const float xh = (a[v].f(i) - mu) * rs;
          float val = rs * (gg.f(i) * d[v].f(i) - mg - xh * mgx);
          if (dres) val += q.f(i);
          o.set(i, val);
        }
        o.store(dx + r * h + c);
      }
    }
  }
}

// Row-per-CTA variants (128 threads per row, 4 elements per thread and step;
// the warp-per-row kernels above keep a whole row per warp in registers, which
// costs occupancy -- see elementwise.cu's RMSNorm row kernels, round 2).
constexpr int LB_THREADS = 128;
constexpr int LB_STEPS = 8;  // h <= 4096

// STP_LN_ROWBLOCK=0 keeps the warp-per-row kernels (A/B in tools/kbench.py).
bool ln_rowblock(int64_t h) {
  static const bool off = [] {
    const char* e = getenv("STP_LN_ROWBLOCK");
    return e && e[0] == '0';
  }();
  return !off && h % 4 == 0 && h <= LB_THREADS * 4 * LB_STEPS;
}

template <typename T>
struct W4 {
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

__device__ __forceinline__ float bsum128(float v, float* red) {
  v = wsum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  const float t = red[0] + red[1] + red[2] + red[3];
  __syncthreads();
  return t;
}

template <typename T>
__global__ void __launch_bounds__(LB_THREADS) ln_fwd_rowblock_kernel(int64_t rows, int h, const T* __restrict__ x,
                                                                     const T* __restrict__ resid, T* x_out,
                                                                     const T* __restrict__ g, const T* __restrict__ b,
                                                                     float eps, T* y, float* mean_out,
                                                                     float* rstd_out) {
  __shared__ float red[4];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    W4<T> a[LB_STEPS];
    float s1 = 0.f;
#pragma unroll
    for (int k = 0; k < LB_STEPS; ++k) {
      const int c = (k * LB_THREADS + threadIdx.x) * 4;
      if (c < h) {
        a[k].load(x + r * h + c);
        if (resid) {
          W4<T> q;
          q.load(resid + r * h + c);
#pragma unroll
          for (int i = 0; i < 4; ++i) a[k].set(i, a[k].f(i) + q.f(i));
          a[k].store(x_out + r * h + c);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) s1 += a[k].f(i);
      }
    }
    const float mu = bsum128(s1, red) / (float)h;
    float s2 = 0.f;
#pragma unroll
    for (int k = 0; k < LB_STEPS; ++k) {
      const int c = (k * LB_THREADS + threadIdx.x) * 4;
      if (c < h) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float d = a[k].f(i) - mu;
          s2 += d * d;
        }
      }
    }
    const float rs = rsqrtf(bsum128(s2, red) / (float)h + eps);
    if (threadIdx.x == 0) {
      if (mean_out) mean_out[r] = mu;
      if (rstd_out) rstd_out[r] = rs;
    }
#pragma unroll
    for (int k = 0; k < LB_STEPS; ++k) {
      const int c = (k * LB_THREADS + threadIdx.x) * 4;
      if (c < h) {
        W4<T> gg, bb, o;
        gg.load(g + c);
        bb.load(b + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) o.set(i, (a[k].f(i) - mu) * rs * gg.f(i) + bb.f(i));
        o.store(y + r * h + c);
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(LB_THREADS) ln_bwd_rowblock_kernel(int64_t rows, int h, const T* __restrict__ dy,
                                                                     const T* __restrict__ x, const T* __restrict__ g,
                                                                     const float* __restrict__ mean,
                                                                     const float* __restrict__ rstd, const T* dres,
                                                                     T* dx) {
  __shared__ float red[4];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float mu = mean[r], rs = rstd[r];
    W4<T> a[LB_STEPS], d[LB_STEPS];
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int k = 0; k < LB_STEPS; ++k) {
      const int c = (k * LB_THREADS + threadIdx.x) * 4;
      if (c < h) {
        a[k].load(x + r * h + c);
        d[k].load(dy + r * h + c);
        W4<T> gg;
        gg.load(g + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float gd = gg.f(i) * d[k].f(i);
          sg += gd;
          sgx += gd * (a[k].f(i) - mu) * rs;
        }
      }
    }
    const float mg = bsum128(sg, red) / (float)h, mgx = bsum128(sgx, red) / (float)h;
#pragma unroll
    for (int k = 0; k < LB_STEPS; ++k) {
      const int c = (k * LB_THREADS + threadIdx.x) * 4;
      if (c < h) {
        W4<T> gg, o, q;
        gg.load(g + c);
        if (dres) q.load(dres + r * h + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float xh = (a[k].f(i) - mu) * rs;
          float val = rs * (gg.f(i) * d[k].f(i) - mg - xh * mgx);
          if (dres) val += q.f(i);
          o.set(i, val);
        }
        o.store(dx + r * h + c);
      }
    }
  }
}

// dg[c] += sum_rows dy xhat, db[c] += sum_rows dy: one thread per column,
// a block of rows per blockIdx.y, one fp32 atomic per column and block.
template <typename T>
__global__ void ln_dparams_kernel(int64_t rows, int h, const T* __restrict__ dy, const T* __restrict__ x,
                                  const float* __restrict__ mean, const float* __restrict__ rstd, float* dg, float* db,
                                  int64_t rows_per_block) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float ag = 0.f, ab = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    const float d = to_f<T>(dy[r * h + c]);
    ag += d * (to_f<T>(x[r * h + c]) - mean[r]) * rstd[r];
    ab += d;
  }
  if (dg) atomicAdd(&dg[c], ag);
  if (db) atomicAdd(&db[c], ab);
}

__device__ __forceinline__ float sig(float z) { return 1.f / (1.f + __expf(-z)); }

// kind 0: QuickGELU a sigmoid(1.702 a); kind 1: GELU z Phi(z) (erf form).
template <typename T>
__global__ void act_fwd_kernel(int64_t n, int kind, const T* __restrict__ a, T* y) {
  constexpr int VN = V16<T>::N;
  const int64_t nv = n / VN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    V16<T> v, o;
    v.load(a + i * VN);
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      const float z = v.f(e);
      o.set(e, kind == 0 ? z * sig(1.702f * z) : 0.5f * z * (1.f + erff(z * 0.70710678118654752f)));
    }
    o.store(y + i * VN);
  }
}

// da = dy * act'(a); written over dy's buffer if da == dy.
template <typename T>
__global__ void act_bwd_kernel(int64_t n, int kind, const T* dy, const T* __restrict__ a, T* da) {
  constexpr int VN = V16<T>::N;
  const int64_t nv = n / VN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    V16<T> d, v, o;
    d.load(dy + i * VN);
    v.load(a + i * VN);
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      const float z = v.f(e);
      float gp;
      if (kind == 0) {
        const float s = sig(1.702f * z);
        gp = s + 1.702f * z * s * (1.f - s);
      } else {
        gp = 0.5f * (1.f + erff(z * 0.70710678118654752f)) + z * 0.39894228040143268f * __expf(-0.5f * z * z);
      }
      o.set(e, d.f(e) * gp);
    }
    o.store(da + i * VN);
  }
}

// cos / sin table [s][d/2] of the 2-D vision RoPE (oracle/vit.py
// vit_rope_tables): patch i in merge-window order of a (gh, gw) grid sits at
// window w = i / 4 (row-major over gw / 2 windows per row), k = i % 4:
// hp = 2 (w / (gw/2)) + k / 2, wp = 2 (w % (gw/2)) + k % 2; angle j < d/4:
// hp inv_j, d/4 <= j < d/2: wp inv_{j - d/4}, inv_j = theta^(-2j / (d/2)).
__global__ void vit_rope_table_kernel(int64_t s, int d, int gw, double theta, float2* tab) {
  const int half = d / 2, q = d / 4;
  const int64_t total = s * half;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % half);
    const int64_t row = i / half;
    const int64_t w = row / 4;
    const int k = (int)(row % 4);
    const int64_t wpr = gw / 2;
    const int64_t hp = 2 * (w / wpr) + k / 2, wp = 2 * (w % wpr) + k % 2;
    const int jj = j < q ? j : j - q;
    const double inv = pow(theta, -2.0 * (double)jj / (double)half);
    double sn, cs;
    sincos((double)(j < q ? hp : wp) * inv, &sn, &cs);
    tab[i] = make_float2((float)cs, (float)sn);
  }
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

stp_status rope_with_table(int dtype, int backward, int64_t s, int64_t ld, int64_t col0, int nh, int d,
                           const float2* tab, void* x, cudaStream_t st);

stp_status layernorm_fwd(int dtype, int64_t rows, int64_t h, const void* x, const void* resid, void* x_out,
                         const void* g, const void* b, float eps, void* y, float* mean, float* rstd, cudaStream_t st) {
  STP_CHECK_ARG(h % 8 == 0, "hidden % 8 == 0");
  STP_CHECK_ARG(al16(x) && al16(y) && al16(g) && al16(b), "16-byte aligned rows");
  STP_CHECK_ARG(!resid || (x_out && al16(resid) && al16(x_out)), "resid needs an aligned x_out");
  if (rows == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    if (h > 32 * V16<T>::N * kNV) return fail(STP_EUNSUPPORTED, "layernorm hidden too large for the row-cached kernel");
    if (ln_rowblock(h))
      ln_fwd_rowblock_kernel<T><<<(unsigned)std::min<int64_t>(rows, (int64_t)num_sms() * 16), LB_THREADS, 0, st>>>(
          rows, (int)h, (const T*)x, (const T*)resid, (T*)x_out, (const T*)g, (const T*)b, eps, (T*)y, mean, rstd);
    else
      ln_fwd_kernel<T><<<blocks_for(rows, kWarps), 32 * kWarps, 0, st>>>(rows, (int)h, (const T*)x, (const T*)resid,
                                                                         (T*)x_out, (const T*)g, (const T*)b, eps,
                                                                         (T*)y, mean, rstd);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status layernorm_bwd(int dtype, int64_t rows, int64_t h, const void* dy, const void* x, const void* g,
                         const float* mean, const float* rstd, const void* dres, void* dx, float* dg, float* db,
                         cudaStream_t st) {
  STP_CHECK_ARG(h % 8 == 0, "hidden % 8 == 0");
  STP_CHECK_ARG(al16(dy) && al16(x) && al16(g) && al16(dx) && (!dres || al16(dres)), "16-byte aligned rows");
  if (rows == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    if (h > 32 * V16<T>::N * kNV) return fail(STP_EUNSUPPORTED, "layernorm hidden too large for the row-cached kernel");
    if (dg || db) {  // before dx: dx may alias dres, never dy / x
      const int64_t rpb = 128;
      dim3 grid((unsigned)((h + 255) / 256), (unsigned)((rows + rpb - 1) / rpb));
      ln_dparams_kernel<T><<<grid, 256, 0, st>>>(rows, (int)h, (const T*)dy, (const T*)x, mean, rstd, dg, db, rpb);
      count_launch();
      STP_LAUNCH_CHECK();
    }
    if (ln_rowblock(h))
      ln_bwd_rowblock_kernel<T><<<(unsigned)std::min<int64_t>(rows, (int64_t)num_sms() * 16), LB_THREADS, 0, st>>>(
          rows, (int)h, (const T*)dy, (const T*)x, (const T*)g, mean, rstd, (const T*)dres, (T*)dx);
    else
      ln_bwd_kernel<T><<<blocks_for(rows, kWarps), 32 * kWarps, 0, st>>>(rows, (int)h, (const T*)dy, (const T*)x,
                                                                         (const T*)g, mean, rstd, (const T*)dres,
                                                                         (T*)dx);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status act_fwd(int dtype, int kind, int64_t n, const void* a, void* y, cudaStream_t st) {
  STP_CHECK_ARG(kind == 0 || kind == 1, "activation kind");
  STP_CHECK_ARG(n % 8 == 0 && al16(a) && al16(y), "n % 8 == 0, 16-byte aligned");
  if (n == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    act_fwd_kernel<T><<<blocks_for(n / V16<T>::N, 256), 256, 0, st>>>(n, kind, (const T*)a, (T*)y);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status act_bwd(int dtype, int kind, int64_t n, const void* dy, const void* a, void* da, cudaStream_t st) {
  STP_CHECK_ARG(kind == 0 || kind == 1, "activation kind");
  STP_CHECK_ARG(n % 8 == 0 && al16(a) && al16(dy) && al16(da), "n % 8 == 0, 16-byte aligned");
  if (n == 0) return STP_OK;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    act_bwd_kernel<T><<<blocks_for(n / V16<T>::N, 256), 256, 0, st>>>(n, kind, (const T*)dy, (const T*)a, (T*)da);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

struct VitRopeKey {
  int dev;
  int64_t s;
  int d, gw;
  float theta;
  bool operator<(const VitRopeKey& o) const {
    return std::tie(dev, s, d, gw, theta) < std::tie(o.dev, o.s, o.d, o.gw, o.theta);
  }
};

stp_status rope2d(int dtype, int backward, int64_t s, int64_t ld, int64_t col0, int nh, int d, int gw, float theta,
                  void* x, cudaStream_t st) {
  STP_CHECK_ARG(d % 8 == 0, "head_dim % 8 == 0");
  STP_CHECK_ARG(gw > 0 && gw % 2 == 0 && s % (2 * gw) == 0, "grid width even, s = gh * gw with gh even");
  if (s == 0 || nh == 0) return STP_OK;
  static std::mutex mu;
  static std::map<VitRopeKey, float2*> tables;  // device tables, kept for the process lifetime
  int dev = 0;
  STP_CUDA_TRY(cudaGetDevice(&dev));
  float2* tab = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    VitRopeKey key{dev, s, d, gw, theta};
    auto it = tables.find(key);
    if (it == tables.end()) {
      STP_CUDA_TRY(cudaMalloc(&tab, (size_t)s * (d / 2) * sizeof(float2)));
      vit_rope_table_kernel<<<blocks_for(s * (d / 2), 256), 256, 0, st>>>(s, d, gw, (double)theta, tab);
      count_launch();
      STP_LAUNCH_CHECK();
      tables[key] = tab;
    } else {
      tab = it->second;
    }
  }
  return rope_with_table(dtype, backward, s, ld, col0, nh, d, tab, x, st);
}

}  // namespace stp

extern "C" {

stp_status stp_op_layernorm_fwd(int32_t dtype, int64_t rows, int64_t h, const void* x, const void* resid, void* x_out,
                                const void* gamma, const void* beta, float eps, void* y, float* mean_out,
                                float* rstd_out, void* stream) {
  return stp::layernorm_fwd(dtype, rows, h, x, resid, x_out, gamma, beta, eps, y, mean_out, rstd_out,
                            (cudaStream_t)stream);
}
stp_status stp_op_layernorm_bwd(int32_t dtype, int64_t rows, int64_t h, const void* dy, const void* x,
                                const void* gamma, const float* mean, const float* rstd, const void* dres, void* dx,
                                float* dgamma_acc, float* dbeta_acc, void* stream) {
  return stp::layernorm_bwd(dtype, rows, h, dy, x, gamma, mean, rstd, dres, dx, dgamma_acc, dbeta_acc,
                            (cudaStream_t)stream);
}
stp_status stp_op_act_fwd(int32_t dtype, int32_t kind, int64_t n, const void* a, void* y, void* stream) {
  return stp::act_fwd(dtype, kind, n, a, y, (cudaStream_t)stream);
}
stp_status stp_op_act_bwd(int32_t dtype, int32_t kind, int64_t n, const void* dy, const void* a, void* da,
                          void* stream) {
  return stp::act_bwd(dtype, kind, n, dy, a, da, (cudaStream_t)stream);
}
stp_status stp_op_rope2d(int32_t dtype, int32_t backward, int64_t s, int64_t ld, int64_t col0, int32_t n_heads,
                         int32_t d, int32_t grid_w, float theta, void* x, void* stream) {
  return stp::rope2d(dtype, backward, s, ld, col0, n_heads, d, grid_w, theta, x, (cudaStream_t)stream);
}

}  // extern "C"
