// Kernel launch accounting: every kernel launch of the library goes through a
// LaunchScope, which counts it (ttp_launch_count) and, when profiling is on,
// brackets it with CUDA events on the launching stream so bench.py can read
// per-kernel-class device time for the launches inside its timed region
// (ttp_profile_read).  Event records are asynchronous; elapsed times are
// resolved lazily at read time.
#pragma once

#include <cuda_runtime.h>

enum KernelClass {
  KC_FIBER = 0,
  KC_BOND,
  KC_CONV_SITE0,
  KC_CONV_SITE,
  KC_SAMPLE_DIFF,
  KC_ORACLE_POINTS,
  KC_TT_INNER,
  KC_TT_EVAL,
  KC_DENSE,
  KC_DENSE_FINAL,
  KC_MISC,
  KC_MC,
  KC_MC_FINAL,
  KC_CLUSTER_BOND,
  KC_COUNT
};

struct LaunchScope {
  LaunchScope(KernelClass k, cudaStream_t s);
  ~LaunchScope();
  KernelClass kind;
  cudaStream_t stream;
  cudaEvent_t start, stop;
  bool timed;
};
