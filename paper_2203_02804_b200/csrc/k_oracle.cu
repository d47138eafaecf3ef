// K1/K2: batched fiber evaluators.
//
// The reference samples each unfolding block with ONE oracle call on an
// index array built by _block (cross.py:310-332) and evaluates
// phi(-z) / conj(vhat(z)) entrywise (market.py:204-262).  Here the index
// tuples are assembled in registers from the nested pivot sets and the
// value is written straight into the column-major block the bond kernel
// factorizes: one thread per entry, consecutive threads on consecutive rows
// so the complex128 stores coalesce.
#include "ttp_internal.h"
#include "launch.h"

namespace {

__global__ void fiber_kernel(OracleDev o, FiberJob job, const int* __restrict__ active) {
  const int inst = blockIdx.y;
  if (active && !active[inst]) return;
  const long long total = (long long)job.rl * job.na * job.rr;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  int a, s, b;
  long long off;
  if (job.mode == 0) {
    // rows a*na + s (row fastest), columns b
    const long long rows = (long long)job.rl * job.na;
    b = (int)(e / rows);
    const long long row = e - (long long)b * rows;
    a = (int)(row / job.na);
    s = (int)(row - (long long)a * job.na);
    off = (long long)b * job.ld + row;
  } else {
    // rows s*rr + b (row fastest), columns a
    const long long rows = (long long)job.na * job.rr;
    a = (int)(e / rows);
    const long long row = e - (long long)a * rows;
    s = (int)(row / job.rr);
    b = (int)(row - (long long)s * job.rr);
    off = (long long)a * job.ld + row;
  }
  int idx[TTP_MAX_D];
  const int* L = job.left.base + inst * job.left.set_stride + job.left.offset + (long long)a * job.left.d;
  const int* R = job.right.base + inst * job.right.set_stride + job.right.offset + (long long)b * job.right.d;
  for (int j = 0; j < job.kl; ++j) idx[j] = L[j];
  idx[job.kl] = s;
  for (int j = job.kl + 1; j < o.d; ++j) idx[j] = R[j - job.kl - 1];
  job.out[inst * job.out_stride + off] = oracle_value(o, inst, idx);
}

__global__ void points_kernel(OracleDev o, const int* __restrict__ idx, long long m,
                              cplx* __restrict__ out) {
  const int inst = blockIdx.y;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  int loc[TTP_MAX_D];
  for (int k = 0; k < o.d; ++k) loc[k] = idx[j * o.d + k];
  out[inst * m + j] = oracle_value(o, inst, loc);
}

}  // namespace

void launch_fiber(const OracleDev& o, const FiberJob& job, const int* active, int n_inst,
                  cudaStream_t s) {
  const long long total = (long long)job.rl * job.na * job.rr;
  if (total == 0 || n_inst == 0) return;
  const int threads = 256;
  dim3 grid((unsigned)((total + threads - 1) / threads), (unsigned)n_inst);
  {
    LaunchScope _ls(KC_FIBER, s);
    fiber_kernel<<<grid, threads, 0, s>>>(o, job, active);
  }
}

void launch_oracle_points(const OracleDev& o, int n_inst, const int* idx, long long m,
                          cplx* out, cudaStream_t s) {
  if (m == 0 || n_inst == 0) return;
  const int threads = 256;
  dim3 grid((unsigned)((m + threads - 1) / threads), (unsigned)n_inst);
  {
    LaunchScope _ls(KC_ORACLE_POINTS, s);
    points_kernel<<<grid, threads, 0, s>>>(o, idx, m, out);
  }
}
