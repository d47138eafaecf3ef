// Launch counting and optional per-kernel-class device timing (see launch.h).
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "launch.h"
#include "ttp_internal.h"

namespace {

const char* kNames[KC_COUNT] = {"fiber_kernel",     "bond_kernel",      "conv_site0_kernel",
                                "conv_site_kernel", "sample_diff_kernel", "points_kernel",
                                "tt_inner_kernel",  "eval_warp_kernel", "dense_partial_kernel",
                                "dense_final_kernel", "misc_kernel", "mc_path_kernel",
                                "mc_final_kernel",  "cluster_bond_kernel"};

std::atomic<long long> g_launches{0};
std::atomic<int> g_profile{0};

struct Pending {
  int kind;
  cudaEvent_t a, b;
};

std::mutex g_mu;
std::vector<Pending> g_pending;
long long g_count[KC_COUNT];
long long g_timed[KC_COUNT];
double g_ms[KC_COUNT];

void drain_locked() {
  for (auto& p : g_pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      g_ms[p.kind] += ms;
      g_timed[p.kind] += 1;
    }
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  g_pending.clear();
}

}  // namespace

LaunchScope::LaunchScope(KernelClass k, cudaStream_t s) : kind(k), stream(s), timed(false) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_count[k] += 1;
  }
  if (g_profile.load(std::memory_order_relaxed)) {
    if (cudaEventCreate(&start) == cudaSuccess && cudaEventCreate(&stop) == cudaSuccess) {
      timed = (cudaEventRecord(start, s) == cudaSuccess);
    }
  }
}

LaunchScope::~LaunchScope() {
  if (!timed) return;
  cudaEventRecord(stop, stream);
  std::lock_guard<std::mutex> lk(g_mu);
  g_pending.push_back(Pending{kind, start, stop});
}

cudaError_t ensure_max_smem(const void* func) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> done;
  int dev = 0, lim = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, func})) return cudaSuccess;
  cudaFuncAttributes fa;
  e = cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, func);
  // the cap applies to dynamic shared memory on top of the static amount
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, lim - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done[{dev, func}] = true;
  return e;
}

extern "C" int64_t ttp_launch_count(void) { return g_launches.load(); }

extern "C" void ttp_profile_enable(int on) { g_profile.store(on ? 1 : 0); }

extern "C" void ttp_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  drain_locked();
  std::memset(g_count, 0, sizeof(g_count));
  std::memset(g_timed, 0, sizeof(g_timed));
  std::memset(g_ms, 0, sizeof(g_ms));
}

extern "C" int ttp_profile_read(ttp_kernel_stat* out, int32_t max_entries) {
  std::lock_guard<std::mutex> lk(g_mu);
  drain_locked();
  const int n = max_entries < KC_COUNT ? max_entries : KC_COUNT;
  for (int k = 0; k < n; ++k) {
    std::memset(out[k].name, 0, sizeof(out[k].name));
    std::strncpy(out[k].name, kNames[k], sizeof(out[k].name) - 1);
    out[k].launches = g_count[k];
    out[k].timed_launches = g_timed[k];
    out[k].total_ms = g_ms[k];
  }
  return n;
}
