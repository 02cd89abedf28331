// Error reporting, device queries and version for libstp.so.
#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "common.h"

namespace stp {

namespace {
thread_local char g_err[2048] = "no error";
}

thread_local int64_t g_kernel_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int num_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
  int n = 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

}  // namespace stp

extern "C" {

const char* stp_last_error(void) { return stp::g_err; }

const char* stp_version(void) { return "stp-b200 0.1 (sm_100a)"; }

int32_t stp_num_sms(void) { return stp::num_sms(); }

int64_t stp_kernel_launches(void) { return stp::g_kernel_launches; }

}  // extern "C"
