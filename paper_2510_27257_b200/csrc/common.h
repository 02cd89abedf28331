// Internal helpers shared by the libstp.so translation units (not part of
// the ABI).  Error model: every extern "C" entry point returns stp_status and
// records a thread-local message (stp_last_error).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "stp.h"
#include "stp_ops.h"

namespace stp {

void set_error(const char* fmt, ...);
inline stp_status fail(stp_status st, const std::string& msg) {
  set_error("%s", msg.c_str());
  return st;
}

#define STP_CUDA_TRY(expr)                                                     \
  do {                                                                         \
    cudaError_t e_ = (expr);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      ::stp::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,              \
                       cudaGetErrorString(e_));                                \
      cudaGetLastError(); /* clear a non-sticky error so a later launch check  \
                             does not report it again */                       \
      return STP_ECUDA;                                                        \
    }                                                                          \
  } while (0)

#define STP_CHECK_ARG(cond, msg)                                               \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::stp::set_error("invalid argument: %s (%s)", msg, #cond);              \
      return STP_EINVAL;                                                       \
    }                                                                          \
  } while (0)

#define STP_LAUNCH_CHECK()                                                     \
  do {                                                                         \
    cudaError_t e_ = cudaGetLastError();                                       \
    if (e_ != cudaSuccess) {                                                   \
      ::stp::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__,          \
                       cudaGetErrorString(e_));                                \
      return STP_ECUDA;                                                        \
    }                                                                          \
  } while (0)

int num_sms();
// Count of kernels launched by this library on this thread (for
// stp_step_stats.n_kernels / bench "gpu_launches").
extern thread_local int64_t g_kernel_launches;
inline void count_launch(int n = 1) { g_kernel_launches += n; }

typedef __nv_bfloat16 bf16;

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

inline size_t dtype_size(int dtype) { return dtype == STP_DTYPE_BF16 ? 2 : 4; }

}  // namespace stp

// Dispatch on stp_dtype: binds `T` to float or bf16 inside the body.
#define STP_DISPATCH_DTYPE(dtype, ...)                                         \
  [&]() -> stp_status {                                                        \
    if ((dtype) == STP_DTYPE_F32) {                                            \
      typedef float T;                                                         \
      return __VA_ARGS__();                                                    \
    } else if ((dtype) == STP_DTYPE_BF16) {                                    \
      typedef ::stp::bf16 T;                                                   \
      return __VA_ARGS__();                                                    \
    }                                                                          \
    ::stp::set_error("unknown dtype %d", (int)(dtype));                        \
    return STP_EINVAL;                                                         \
  }()

#ifndef STP_TRY
#define STP_TRY(expr)                     \
  do {                                    \
    stp_status s_ = (expr);               \
    if (s_ != STP_OK) return s_;          \
  } while (0)
#endif
#define STP_TRY_STATUS(expr) STP_TRY(expr)
