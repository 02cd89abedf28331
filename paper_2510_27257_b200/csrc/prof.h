// Kernel-class profiler: when enabled (stp_prof_enable), every launch of a
// profiled class is bracketed by CUDA events on the stream it is launched on,
// with its algorithmic FLOPs / bytes; stp_prof_read sums them per class
// (bench.py's roofline "achieved" = sum FLOPs / sum event time).
#pragma once

#include <cuda_runtime.h>

namespace stp {

enum ProfClass { PROF_GEMM = 0, PROF_ATTN_FWD = 1, PROF_ATTN_BWD = 2, PROF_ELEMWISE = 3, PROF_NCLASS = 4 };

bool prof_on();
void prof_push(int cls, double flops, double bytes, cudaEvent_t e0, cudaEvent_t e1);
cudaEvent_t prof_event();

struct ProfScope {
  int cls;
  double flops, bytes;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  ProfScope(int c, double f, double b, cudaStream_t s) : cls(c), flops(f), bytes(b), st(s) {
    if (prof_on()) {
      e0 = prof_event();
      cudaEventRecord(e0, st);
    }
  }
  ~ProfScope() {
    if (e0) {
      cudaEvent_t e1 = prof_event();
      cudaEventRecord(e1, st);
      prof_push(cls, flops, bytes, e0, e1);
    }
  }
};

}  // namespace stp
