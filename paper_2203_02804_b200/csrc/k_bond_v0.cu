// One-CTA bond kernel, wide shape (512 threads, 2 CTAs per SM), and the
// shape dispatch of launch_bond.
#define V0_NS v0_wide
#define V0_THREADS 512
#define V0_MIN_BLOCKS 2
#include "k_bond_v0_impl.cuh"

namespace v0_small {
size_t bond_smem_bytes(int r);
cudaError_t launch_bond(const BondJob& job, int n_inst, cudaStream_t s);
}  // namespace v0_small

// Row-parallel passes keep one row per thread, so a short block leaves most
// of a 512-thread CTA idle: blocks of at most V0_SMALL_BYTES (64 KB: configs
// 1-3's edge bonds and all of config 1) run 128-thread CTAs, eight per SM.
// Measured (profiles/r02/s4/ab_v0_shape.log): config 1 53.2k -> 74k
// options/s; the 129 x 32 edge bond of config 4 (66 KB) stays wide, where
// the step measured 5% faster (851 vs 806 options/s).
static bool v0_small_shape(int m, int r) {
  return (long long)m * r * (long long)sizeof(cplx) <= (long long)V0_SMALL_BYTES;
}

size_t bond_smem_bytes(int m, int r) {
  return v0_small_shape(m, r) ? v0_small::bond_smem_bytes(r) : v0_wide::bond_smem_bytes(r);
}

cudaError_t launch_bond(const BondJob& job, int n_inst, cudaStream_t s) {
  return v0_small_shape(job.m, job.r) ? v0_small::launch_bond(job, n_inst, s) : v0_wide::launch_bond(job, n_inst, s);
}
