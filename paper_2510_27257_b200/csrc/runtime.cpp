// Error reporting, device queries and version for libstp.so.
#include <cstdarg>
#include <cstdio>
#include <mutex>

#include <vector>

#include "common.h"
#include "prof.h"

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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device: keep
// one bit per device (a process driving several GPUs sets it on each).
stp_status set_max_smem_once(const void* func, int bytes, unsigned long long* mask) {
  int dev = 0;
  STP_CUDA_TRY(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_load_n(mask, __ATOMIC_ACQUIRE) & bit) return STP_OK;
  STP_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  __atomic_fetch_or(mask, bit, __ATOMIC_RELEASE);
  return STP_OK;
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

namespace {
struct ProfState {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  struct Rec {
    int cls;
    double flops, bytes;
    cudaEvent_t e0, e1;
  };
  std::vector<Rec> recs;
};
thread_local ProfState g_prof;
}  // namespace

bool prof_on() { return g_prof.on; }
cudaEvent_t prof_event() {
  if (g_prof.next >= g_prof.pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_prof.pool.push_back(e);
  }
  return g_prof.pool[g_prof.next++];
}
void prof_push(int cls, double flops, double bytes, cudaEvent_t e0, cudaEvent_t e1) {
  g_prof.recs.push_back({cls, flops, bytes, e0, e1});
}

int& gemm_mc_mode_ref();

}  // namespace stp

extern "C" {

// Runtime tuning knobs (stp_ops.h).
stp_status stp_set_option(const char* key, int64_t value) {
  if (!key) return stp::fail(STP_EINVAL, "key is NULL");
  const std::string k(key);
  if (k == "gemm_mc") {
    if (value < 0 || value > 3 || value == 2) return stp::fail(STP_EINVAL, "gemm_mc must be 0 (1-SM), 1 (auto) or 3 (2-SM)");
    stp::gemm_mc_mode_ref() = (int)value;
    return STP_OK;
  }
  return stp::fail(STP_EINVAL, "unknown option " + k);
}

// Kernel-class profiling (stp_ops.h): enable / reset / read per class.
stp_status stp_prof_enable(int32_t on) {
  stp::g_prof.on = on != 0;
  return STP_OK;
}
stp_status stp_prof_reset(void) {
  stp::g_prof.recs.clear();
  stp::g_prof.next = 0;
  return STP_OK;
}
stp_status stp_prof_read(int32_t cls, int64_t* count, double* flops, double* bytes, double* ms) {
  if (!count || !flops || !bytes || !ms) return stp::fail(STP_EINVAL, "NULL argument");
  *count = 0;
  *flops = *bytes = *ms = 0.0;
  for (auto& r : stp::g_prof.recs) {
    if (r.cls != cls) continue;
    cudaError_t e = cudaEventSynchronize(r.e1);
    if (e != cudaSuccess) return stp::fail(STP_ECUDA, cudaGetErrorString(e));
    float t = 0.f;
    e = cudaEventElapsedTime(&t, r.e0, r.e1);
    if (e != cudaSuccess) return stp::fail(STP_ECUDA, cudaGetErrorString(e));
    *count += 1;
    *flops += r.flops;
    *bytes += r.bytes;
    *ms += t;
  }
  return STP_OK;
}


const char* stp_last_error(void) { return stp::g_err; }

const char* stp_version(void) { return "stp-b200 0.1 (sm_100a)"; }

int32_t stp_num_sms(void) { return stp::num_sms(); }

int64_t stp_kernel_launches(void) { return stp::g_kernel_launches; }

}  // extern "C"
