// Internal (non-ABI) declarations shared by the kernel translation units and
// the host runtime in driver.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>

#include "../../include/ttpricer_b200.h"
#include "oracle_eval.cuh"

int ttp_record_cuda_error(cudaError_t e);
int ttp_fail(int status, const std::string& msg);

// Host-side queries (device attributes, occupancy, function opt-ins) are
// per-device facts: one process may drive several GPUs (torch.cuda.set_device
// between calls), so every memo is keyed by the current device.
template <class K, class T, class F>
T ttp_device_memo(std::map<std::pair<int, K>, T>& memo, std::mutex& mu, const K& key, F compute) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = memo.find({dev, key});
  if (it != memo.end()) return it->second;
  const T v = compute();
  memo[{dev, key}] = v;
  return v;
}

// Raise a kernel's dynamic shared-memory cap to the device's opt-in limit,
// once per function.  Setting it per launch to the launch's own size races
// when two host threads launch the same kernel with different sizes (the
// phi and vhat crosses run concurrently on two streams).
cudaError_t ensure_max_smem(const void* func);

// Index-set view used by fiber kernels: row t of set k of instance i is at
// base + i*set_stride + set_offsets[k] + t*d.
struct SetView {
  const int* base;
  long long set_stride;
  long long offset;  // set_offsets[k]
  int d;
};

// One sampled unfolding ("fiber block") per instance.
//   mode 0 (left-to-right, cross.py:412-423):  entry (a, s, b) is stored at
//          b*ld + a*na + s           (rows a*na+s, cols b; column-major)
//   mode 1 (right-to-left, cross.py:424-435):  entry (a, s, b) is stored at
//          a*ld + s*rr + b           (rows s*rr+b, cols a; column-major)
// The full multi-index is left[a] ++ (s) ++ right[b]; the axis sits at
// position kl = length of the left tuples.
struct FiberJob {
  int mode;
  int rl, na, rr;  // left count, axis size, right count
  int kl;          // left tuple length
  SetView left, right;
  cplx* out;
  long long out_stride;  // complex elements per instance
  long long ld;
};

bool fiber_fast_enabled();
void launch_fiber(const OracleDev& o, const FiberJob& job, const int* active, int n_inst,
                  cudaStream_t s);
void launch_oracle_points(const OracleDev& o, int n_inst, const int* idx, long long m,
                          cplx* out, cudaStream_t s);
