// Copy-engine TP transport (STP_TP_TRANSPORT=ce): the device side.
//
// The TP reduce-scatter / all-gather of every comm phase (
// PAPER.md Eq. 1-2, SP reading Q10) without SM-resident collective
// kernels: the executor pulls peer rows with cudaMemcpyAsync over NVLink
// (copy engines, no SMs) from IPC-mapped symmetric buffers, and orders the
// pulls with flags in peer memory:
//   tp_signal    one tiny kernel: st.release.sys of the phase number into
//                every peer's flag word for this rank
//   tp_wait      cuStreamWaitValue32(flag >= phase): a stream memory op, no
//                SM, on the comm stream
//   tp_fused_fwd / tp_fused_bwd
//                the reduction of the pulled rows fused with the residual add
//                and RMSNorm of the comm phase: x = sum_q piece_q (+ resid)
//                -> x_out; y = x * rstd * gamma -> y (this rank's rows of the
//                all-gather destination)
// The contention calibration (tools/contention.py) shows why: NCCL's
// SM-resident kernels slow the overlapped GEMM by 3-11% (App. F's
// 7.5% on A800), copy-engine transfers by ~0%.
#include <cuda.h>

#include <algorithm>

#include "common.h"

namespace stp {
namespace {

constexpr int kWarps = 8;

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
};

struct SigArgs {
  uint32_t* dst[16];
  int n;
  uint32_t val;
};

__global__ void tp_signal_kernel(SigArgs a) {
  __threadfence_system();
  const int i = threadIdx.x;
  if (i < a.n) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.dst[i]), "r"(a.val) : "memory");
}

// Spin-wait fallback (STP_CE_WAIT=spin): one thread polls the flag with
// acquire loads; traps after 60 s so a broken handshake cannot hang the GPU.
__global__ void tp_wait_kernel(const uint32_t* flag, uint32_t val) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int32_t)(v - val) >= 0) return;
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 60ull * 1000000000ull) __trap();
    __nanosleep(200);
  }
}

struct Pieces {
  const void* p[16];
  int n;
};
struct Dsts {
  void* p[16];
  int n;
};

template <typename T>
__device__ __forceinline__ void store_all(const Dsts& d, int64_t off, const V16<T>& v) {
#pragma unroll 1
  for (int k = 0; k < d.n; ++k) v.store(reinterpret_cast<T*>(d.p[k]) + off);
}

// x = sum_k piece_k (+ resid), rounded to T -> x_out (if given);
// g: y = x * rstd * gamma, else y = x; y -> every destination.
// Pieces / destinations may live in peer memory (NVLink loads / stores).
// dsts.p[0] doubles as the row scratch when x_out is null.
template <typename T>
__global__ void tp_fused_fwd_kernel(int64_t rows, int h, Pieces pc, const T* __restrict__ resid, T* x_out,
                                    const T* __restrict__ g, float eps, float* rstd, Dsts ds) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  constexpr int VN = V16<T>::N;
  T* scratch = x_out ? x_out : reinterpret_cast<T*>(ds.p[0]);
  for (int64_t r = w0; r < rows; r += nw) {
    float ss = 0.f;
    for (int c = lane * VN; c < h; c += 32 * VN) {
      float acc[VN];
#pragma unroll
      for (int i = 0; i < VN; ++i) acc[i] = 0.f;
      V16<T> a[16];
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < pc.n) a[k].load(reinterpret_cast<const T*>(pc.p[k]) + r * h + c);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < pc.n) {
#pragma unroll
          for (int i = 0; i < VN; ++i) acc[i] += to_f<T>(a[k].v[i]);
        }
      if (resid) {
        V16<T> b;
        b.load(resid + r * h + c);
#pragma unroll
        for (int i = 0; i < VN; ++i) acc[i] += to_f<T>(b.v[i]);
      }
      V16<T> o;
#pragma unroll
      for (int i = 0; i < VN; ++i) {
        o.v[i] = from_f<T>(acc[i]);
        const float q = to_f<T>(o.v[i]);
        ss += q * q;
      }
      if (g) {
        o.store(scratch + r * h + c);
      } else {
        if (x_out) o.store(x_out + r * h + c);
        store_all(ds, r * h + c, o);
      }
    }
    if (!g) continue;
    ss = wsum(ss);
    const float rs = rsqrtf(ss / (float)h + eps);
    if (lane == 0 && rstd) rstd[r] = rs;
    __syncwarp();
    for (int c = lane * VN; c < h; c += 32 * VN) {
      V16<T> a, gg, o;
      a.load(scratch + r * h + c);
      gg.load(g + c);
#pragma unroll
      for (int i = 0; i < VN; ++i) o.v[i] = from_f<T>(to_f<T>(a.v[i]) * rs * to_f<T>(gg.v[i]));
      store_all(ds, r * h + c, o);
    }
  }
  __threadfence_system();
}

// RMSNorm backward of the summed gradient (Eq. 2 with the SP
// reading): dy = sum_k piece_k -> dy_out (rounded, for the dgamma partials);
// dx = rstd*gamma*dy - x*rstd^3*mean(gamma*dy*x) (+ dres) -> dx and every
// destination (the all-gather of dx).
template <typename T>
__global__ void tp_fused_bwd_kernel(int64_t rows, int h, Pieces pc, const T* __restrict__ x,
                                    const T* __restrict__ g, const float* __restrict__ rstd, const T* dres, T* dx,
                                    T* dy_out, Dsts ds) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  constexpr int VN = V16<T>::N;
  for (int64_t r = w0; r < rows; r += nw) {
    const float rs = rstd[r];
    float dot = 0.f;
    for (int c = lane * VN; c < h; c += 32 * VN) {
      float acc[VN];
#pragma unroll
      for (int i = 0; i < VN; ++i) acc[i] = 0.f;
      V16<T> a[16];
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < pc.n) a[k].load(reinterpret_cast<const T*>(pc.p[k]) + r * h + c);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < pc.n) {
#pragma unroll
          for (int i = 0; i < VN; ++i) acc[i] += to_f<T>(a[k].v[i]);
        }
      V16<T> o, xx, gg;
      xx.load(x + r * h + c);
      gg.load(g + c);
#pragma unroll
      for (int i = 0; i < VN; ++i) {
        o.v[i] = from_f<T>(acc[i]);
        dot += to_f<T>(gg.v[i]) * to_f<T>(o.v[i]) * to_f<T>(xx.v[i]);
      }
      o.store(dy_out + r * h + c);
    }
    dot = wsum(dot) / (float)h;
    const float kk = rs * rs * rs * dot;
    __syncwarp();
    for (int c = lane * VN; c < h; c += 32 * VN) {
      V16<T> d, xx, gg, rr, o;
      d.load(dy_out + r * h + c);
      xx.load(x + r * h + c);
      gg.load(g + c);
      if (dres) rr.load(dres + r * h + c);
#pragma unroll
      for (int i = 0; i < VN; ++i) {
        float v = rs * to_f<T>(gg.v[i]) * to_f<T>(d.v[i]) - to_f<T>(xx.v[i]) * kk;
        if (dres) v += to_f<T>(rr.v[i]);
        o.v[i] = from_f<T>(v);
      }
      o.store(dx + r * h + c);
      store_all(ds, r * h + c, o);
    }
  }
  __threadfence_system();
}

// CTAs of the fused comm-phase kernels: each warp owns one row at a time, so
// fewer CTAs mean a longer (still overlapped) phase but fewer SM slots taken
// from the other microbatch's GEMMs (STP_P2P_CTAS, default 2 x SMs).
int fused_grid(int64_t rows) {
  static const int64_t cap = [] {
    const char* e = getenv("STP_P2P_CTAS");
    return (int64_t)(e && atoi(e) > 0 ? atoi(e) : num_sms() * 2);
  }();
  int64_t blocks = (rows + kWarps - 1) / kWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, cap));
}

// Optional SM partitioning (STP_COMM_SMEM = bytes): the fused comm kernels
// request that much (unused) dynamic shared memory, so their CTAs cannot
// co-reside with a persistent GEMM CTA (~197 KB) and run only on the SMs the
// GEMM leaves free (STP_GEMM_MAX_CTAS < SMs): compute and communication on
// disjoint SMs instead of sharing issue slots (the overlap contention of
// PAPER.md App. F).  0 (default) = no partitioning.
int comm_smem() {
  static const int v = [] {
    const char* e = getenv("STP_COMM_SMEM");
    return e ? std::max(0, atoi(e)) : 0;
  }();
  return v;
}

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

PFN_waitValue32 get_wait() {
  static PFN_waitValue32 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_waitValue32>(p);
  }
  return fn;
}

}  // namespace

stp_status tp_signal(uint32_t* const* dst, int n, uint32_t val, cudaStream_t st) {
  STP_CHECK_ARG(n >= 0 && n <= 16, "1..16 peers");
  if (n == 0) return STP_OK;
  SigArgs a{};
  for (int i = 0; i < n; ++i) a.dst[i] = dst[i];
  a.n = n;
  a.val = val;
  tp_signal_kernel<<<1, 32, 0, st>>>(a);
  count_launch();
  STP_LAUNCH_CHECK();
  return STP_OK;
}

stp_status tp_wait(const uint32_t* flag, uint32_t val, bool spin, cudaStream_t st) {
  if (spin) {
    tp_wait_kernel<<<1, 1, 0, st>>>(flag, val);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  }
  PFN_waitValue32 w = get_wait();
  if (!w) return fail(STP_EUNSUPPORTED, "cuStreamWaitValue32 unavailable (use STP_CE_WAIT=spin)");
  CUresult r = w((CUstream)st, (CUdeviceptr)(uintptr_t)flag, val, 0 /* CU_STREAM_WAIT_VALUE_GEQ */);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue32 failed (%d)", (int)r);
    return STP_ECUDA;
  }
  return STP_OK;
}

stp_status tp_fused_fwd(int dtype, int64_t rows, int64_t h, const void* const* pieces, int np, const void* resid,
                        void* x_out, const void* g, float eps, float* rstd, void* const* dsts, int nd,
                        cudaStream_t st) {
  STP_CHECK_ARG(h % 8 == 0, "hidden % 8 == 0");
  STP_CHECK_ARG(np >= 1 && np <= 16 && nd >= 0 && nd <= 16, "1..16 pieces, 0..16 destinations");
  STP_CHECK_ARG(x_out || nd > 0, "x_out or a destination");
  if (rows == 0) return STP_OK;
  Pieces pc{};
  for (int i = 0; i < np; ++i) pc.p[i] = pieces[i];
  pc.n = np;
  Dsts ds{};
  for (int i = 0; i < nd; ++i) ds.p[i] = dsts[i];
  ds.n = nd;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    const int sm = comm_smem();
    if (sm > 48 * 1024)
      STP_CUDA_TRY(cudaFuncSetAttribute(tp_fused_fwd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    tp_fused_fwd_kernel<T><<<fused_grid(rows), 32 * kWarps, sm, st>>>(rows, (int)h, pc, (const T*)resid, (T*)x_out,
                                                                     (const T*)g, eps, rstd, ds);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

stp_status tp_fused_bwd(int dtype, int64_t rows, int64_t h, const void* const* pieces, int np, const void* x,
                        const void* g, const float* rstd, const void* dres, void* dx, void* dy_out,
                        void* const* dsts, int nd, cudaStream_t st) {
  STP_CHECK_ARG(h % 8 == 0, "hidden % 8 == 0");
  STP_CHECK_ARG(np >= 1 && np <= 16 && nd >= 0 && nd <= 16, "1..16 pieces, 0..16 destinations");
  if (rows == 0) return STP_OK;
  Pieces pc{};
  for (int i = 0; i < np; ++i) pc.p[i] = pieces[i];
  pc.n = np;
  Dsts ds{};
  for (int i = 0; i < nd; ++i) ds.p[i] = dsts[i];
  ds.n = nd;
  return STP_DISPATCH_DTYPE(dtype, [&] {
    const int sm = comm_smem();
    if (sm > 48 * 1024)
      STP_CUDA_TRY(cudaFuncSetAttribute(tp_fused_bwd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    tp_fused_bwd_kernel<T><<<fused_grid(rows), 32 * kWarps, sm, st>>>(rows, (int)h, pc, (const T*)x, (const T*)g,
                                                                     rstd, (const T*)dres, (T*)dx, (T*)dy_out, ds);
    count_launch();
    STP_LAUNCH_CHECK();
    return STP_OK;
  });
}

}  // namespace stp
