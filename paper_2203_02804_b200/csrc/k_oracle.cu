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
#include "dev_knobs.h"
#include "launch.h"
#include "fiber_fast.cuh"

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

// Separable variant (fiber_fast.cuh): the block's columns' parts are formed
// once per CTA in shared memory, each thread owns one ROW and sweeps the
// columns with one short inner product + exp (phi) or one divide (vhat).
__global__ void fiber_fast_kernel(OracleDev o, FiberJob job, const int* __restrict__ active) {
  extern __shared__ double2 ff_smem[];
  const int inst = blockIdx.y;
  if (active && !active[inst]) return;
  const int d = o.d;
  const double* p = o.params + inst * o.param_stride;
  const FiberSplit fs = fiber_split(job.mode, job.kl, d);
  const bool phi = o.kind == TTP_ORACLE_PHI_GBM;
  const int cstride = phi ? 1 + fs.ninner : 2;
  const int ncols = job.mode == 0 ? job.rr : job.rl;
  const long long nrows = job.mode == 0 ? (long long)job.rl * job.na : (long long)job.na * job.rr;
  int idx[TTP_MAX_D];
  for (int t = threadIdx.x; t < ncols; t += blockDim.x) {
    const int* T = (job.mode == 0)
                       ? job.right.base + inst * job.right.set_stride + job.right.offset + (long long)t * job.right.d
                       : job.left.base + inst * job.left.set_stride + job.left.offset + (long long)t * job.left.d;
    const int shift = (job.mode == 0) ? job.kl + 1 : 0;
    for (int j = fs.col_lo; j < fs.col_hi; ++j) idx[j] = T[j - shift];
    cplx* cb = ff_smem + t * cstride;
    if (phi) {
      PhiPart part;
      phi_part(p, d, idx, fs.col_lo, fs.col_hi, fs.inner_is_col, fs.row_lo, fs.row_hi, part);
      cb[0] = part.e;
      for (int q = 0; q < fs.ninner; ++q) cb[1 + q] = part.vec[q];
    } else {
      vhat_part(p, idx, fs.col_lo, fs.col_hi, cb[0], cb[1]);
    }
  }
  __syncthreads();
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  if (job.mode == 0) {
    const int a = (int)(row / job.na), s = (int)(row - (long long)a * job.na);
    const int* L = job.left.base + inst * job.left.set_stride + job.left.offset + (long long)a * job.left.d;
    for (int j = 0; j < job.kl; ++j) idx[j] = L[j];
    idx[job.kl] = s;
  } else {
    const int s = (int)(row / job.rr), b = (int)(row - (long long)s * job.rr);
    const int* R = job.right.base + inst * job.right.set_stride + job.right.offset + (long long)b * job.right.d;
    idx[job.kl] = s;
    for (int j = job.kl + 1; j < d; ++j) idx[j] = R[j - job.kl - 1];
  }
  cplx* out = job.out + inst * job.out_stride + row;
  if (phi) {
    PhiPart rp;
    phi_part(p, d, idx, fs.row_lo, fs.row_hi, !fs.inner_is_col, fs.col_lo, fs.col_hi, rp);
    for (int t = 0; t < ncols; ++t) out[(long long)t * job.ld] = phi_combine_packed(rp, ff_smem + t * cstride, fs.ninner);
  } else {
    cplx prow, wrow;
    vhat_part(p, idx, fs.row_lo, fs.row_hi, prow, wrow);
    for (int t = 0; t < ncols; ++t) {
      const cplx* cb = ff_smem + t * cstride;
      out[(long long)t * job.ld] = vhat_combine(p, d, prow, wrow, cb[0], cb[1]);
    }
  }
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

// TTP_FIBER_FAST=0 forces the direct per-entry evaluation (A/B checks).
bool fiber_fast_enabled() {
  static const bool on = [] {
    const char* e = ttp_dev_env("TTP_FIBER_FAST");
    return !(e && e[0] == '0');
  }();
  return on;
}

void launch_fiber(const OracleDev& o, const FiberJob& job, const int* active, int n_inst,
                  cudaStream_t s) {
  const long long total = (long long)job.rl * job.na * job.rr;
  if (total == 0 || n_inst == 0) return;
  const int threads = 256;
  if ((o.kind == TTP_ORACLE_PHI_GBM || o.kind == TTP_ORACLE_VHAT_MIN) && o.d <= 2 * FF_MAXI &&
      fiber_fast_enabled()) {
    const int ncols = job.mode == 0 ? job.rr : job.rl;
    const long long nrows = job.mode == 0 ? (long long)job.rl * job.na : (long long)job.na * job.rr;
    const size_t smem = sizeof(cplx) * (size_t)ncols * (1 + FF_MAXI);
    if (ncols >= 4 && smem <= 48 * 1024) {
      dim3 grid((unsigned)((nrows + threads - 1) / threads), (unsigned)n_inst);
      LaunchScope _ls(KC_FIBER, s);
      fiber_fast_kernel<<<grid, threads, smem, s>>>(o, job, active);
      return;
    }
  }
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
