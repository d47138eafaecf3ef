// K8: dense full-grid contour sum  sum_grid phi(-z) vhat(z)
// (_dense_contour_sum, pricers.py:185-196).
//
// The reference walks flat C-order indices in chunks of 2^20 and sums
// phi(-z) * vhat(z) chunk by chunk.  Here the flat range is split into a
// fixed number of contiguous slabs per instance (one CTA each); every term is
// evaluated in registers (nothing is materialised, so the kernel is FP64 /
// transcendental bound, not HBM bound) and the per-slab sums are combined in
// slab order by a second kernel, so the result is independent of scheduling.
#include "ttp_internal.h"
#include "launch.h"

namespace {

constexpr int DENSE_THREADS = 256;
constexpr int DENSE_SLABS = 1184;  // 8 CTAs per SM on 148 SMs

// The flat range is walked by grid LINES (all points of the last axis for
// fixed outer indices): per line the outer parts of both oracles are formed
// once -- phi's linear and quadratic forms over the first d-1 coordinates
// and their coupling to the last one, vhat's partial sum w and product of
// i z_j -- and each of the line's terms then costs O(1) plus the two complex
// exponentials and one division (market.py:216-218, 256-261).  Same values
// as oracle_value() up to the association of the d-term sums.
__global__ void __launch_bounds__(DENSE_THREADS)
dense_partial_kernel(OracleDev phi, OracleDev vhat, long long first, long long count,
                     cplx* __restrict__ part) {
  const int inst = blockIdx.y;
  const int slab = blockIdx.x;
  const long long per = (count + gridDim.x - 1) / gridDim.x;
  const long long lo = first + slab * per;
  const long long hi = min(first + count, lo + per);
  const int d = phi.d;
  const int nl = phi.shape[d - 1];
  const double* pp = phi.params + inst * phi.param_stride;
  const double* pv = vhat.params + inst * vhat.param_stride;
  const double* mu = pp + 3;
  const double* C = pp + 3 + d;
  const double mul = mu[d - 1], cll = C[(d - 1) * d + d - 1];
  const double lnK = log(pv[3]);
  const bool vconj = pv[4] != 0.0, vneg = ((d - 1) & 1) != 0;
  cplx acc = mk(0.0, 0.0);
  if (lo < hi) {
    const long long L0 = lo / nl, L1 = (hi - 1) / nl;
    for (long long L = L0 + threadIdx.x; L <= L1; L += DENSE_THREADS) {
      int idx[TTP_MAX_D];
      long long rem = L;
      for (int k = d - 2; k >= 0; --k) {
        const int n = phi.shape[k];
        const long long q = rem / n;
        idx[k] = (int)(rem - q * n);
        rem = q;
      }
      // phi outer parts: lin_o = sum y_j mu_j, quad_o = y^T C y, cpl = the
      // last coordinate's coefficient (C[j][l] + C[l][j]) y_j  (y = -z)
      cplx lin_o = mk(0.0, 0.0), quad_o = mk(0.0, 0.0), cpl = mk(0.0, 0.0);
      // vhat outer parts: w_o = sum z_j, prod_o = prod i z_j
      cplx w_o = mk(0.0, 0.0), prod_o = mk(1.0, 0.0);
      for (int j = 0; j < d - 1; ++j) {
        const cplx yj = cneg(contour_point(pp, idx[j]));
        lin_o = cadd(lin_o, cscale(yj, mu[j]));
        cplx row = mk(0.0, 0.0);
        for (int k = 0; k < d - 1; ++k) row = cadd(row, cscale(cneg(contour_point(pp, idx[k])), C[j * d + k]));
        quad_o = cfma(yj, row, quad_o);
        cpl = cadd(cpl, cscale(yj, C[j * d + d - 1] + C[(d - 1) * d + j]));
        const cplx zj = contour_point(pv, idx[j]);
        w_o = cadd(w_o, zj);
        prod_o = cmul(prod_o, mk(-zj.y, zj.x));
      }
      const long long base = L * nl;
      const int t0 = (int)(max(lo, base) - base), t1 = (int)(min(hi, base + nl) - base);
      for (int t = t0; t < t1; ++t) {
        const cplx y = cneg(contour_point(pp, t));
        const cplx lin = cadd(lin_o, cscale(y, mul));
        const cplx quad = cadd(quad_o, cmul(y, cadd(cpl, cscale(y, cll))));
        const cplx a = cexp_d(mk(-lin.y - 0.5 * quad.x, lin.x - 0.5 * quad.y));
        const cplx z = contour_point(pv, t);
        const cplx w = cadd(w_o, z);
        const cplx prod = cmul(prod_o, mk(-z.y, z.x));
        const cplx onepiw = mk(1.0 - w.y, w.x);
        cplx v = cdiv(cexp_d(cscale(onepiw, lnK)), cmul(onepiw, prod));
        if (vneg) v = cneg(v);
        if (vconj) v = cconj(v);
        acc = cfma(a, v, acc);
      }
    }
  }
  __shared__ cplx red[DENSE_THREADS / 32];
  acc = warp_sum(acc);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = acc;
  __syncthreads();
  if (w == 0) {
    acc = lane < DENSE_THREADS / 32 ? red[lane] : mk(0.0, 0.0);
    acc = warp_sum(acc);
    if (lane == 0) part[(long long)inst * gridDim.x + slab] = acc;
  }
}

__global__ void dense_final_kernel(const cplx* __restrict__ part, int slabs, cplx* __restrict__ out) {
  const int inst = blockIdx.x;
  __shared__ cplx red[32];
  cplx acc = mk(0.0, 0.0);
  // contiguous block of slabs per thread keeps the summation order fixed
  const int per = (slabs + blockDim.x - 1) / blockDim.x;
  for (int q = 0; q < per; ++q) {
    const int s = threadIdx.x * per + q;
    if (s < slabs) acc = cadd(acc, part[(long long)inst * slabs + s]);
  }
  acc = warp_sum(acc);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = acc;
  __syncthreads();
  if (w == 0) {
    acc = lane < (int)(blockDim.x >> 5) ? red[lane] : mk(0.0, 0.0);
    acc = warp_sum(acc);
    if (lane == 0) out[inst] = acc;
  }
}

}  // namespace

extern "C" size_t ttp_dense_workspace(int32_t n_inst, int64_t) {
  return sizeof(cplx) * ((size_t)n_inst * DENSE_SLABS + (size_t)n_inst);
}

extern "C" int ttp_dense_sum_range(const ttp_oracle* phi, const ttp_oracle* vhat, const int32_t* h_shape,
                                   const int32_t* d_shape, int32_t n_inst, int64_t first, int64_t count,
                                   double* h_out, void* d_ws, size_t ws_bytes, void* stream);

extern "C" int ttp_dense_sum(const ttp_oracle* phi, const ttp_oracle* vhat, const int32_t* h_shape,
                             const int32_t* d_shape, int32_t n_inst, double* h_out, void* d_ws,
                             size_t ws_bytes, void* stream) {
  return ttp_dense_sum_range(phi, vhat, h_shape, d_shape, n_inst, 0, -1, h_out, d_ws, ws_bytes, stream);
}

extern "C" int ttp_dense_sum_range(const ttp_oracle* phi, const ttp_oracle* vhat, const int32_t* h_shape,
                                   const int32_t* d_shape, int32_t n_inst, int64_t first, int64_t count,
                                   double* h_out, void* d_ws, size_t ws_bytes, void* stream) {
  if (!phi || !vhat || phi->kind != TTP_ORACLE_PHI_GBM || vhat->kind != TTP_ORACLE_VHAT_MIN ||
      phi->d != vhat->d || phi->d < 1 || phi->d > TTP_MAX_D || n_inst < 0)
    return ttp_fail(TTP_ERR_INVALID, "dense_sum: expects a PHI_GBM and a VHAT_MIN oracle");
  long long n_terms = 1;
  for (int k = 0; k < phi->d; ++k) {
    if (h_shape[k] < 1) return ttp_fail(TTP_ERR_INVALID, "dense_sum: empty axis");
    if (n_terms > (1LL << 62) / h_shape[k]) return ttp_fail(TTP_ERR_CAPACITY, "dense_sum: grid too large");
    n_terms *= h_shape[k];
  }
  if (count < 0) count = n_terms - first;
  if (first < 0 || first > n_terms || count > n_terms - first)
    return ttp_fail(TTP_ERR_INVALID, "dense_sum: term range outside the grid");
  if (ws_bytes < ttp_dense_workspace(n_inst, n_terms))
    return ttp_fail(TTP_ERR_WORKSPACE, "dense_sum: workspace too small");
  if (n_inst == 0) return TTP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  OracleDev a = oracle_dev_from(*phi, d_shape);
  OracleDev b = oracle_dev_from(*vhat, d_shape);
  cplx* part = reinterpret_cast<cplx*>(d_ws);
  cplx* out = part + (size_t)n_inst * DENSE_SLABS;
  dim3 grid(DENSE_SLABS, (unsigned)n_inst);
  {
    LaunchScope _ls(KC_DENSE, s);
    dense_partial_kernel<<<grid, DENSE_THREADS, 0, s>>>(a, b, first, count, part);
  }
  TTP_CUDA_CHECK(cudaGetLastError());
  {
    LaunchScope _ls(KC_DENSE_FINAL, s);
    dense_final_kernel<<<n_inst, 256, 0, s>>>(part, DENSE_SLABS, out);
  }
  TTP_CUDA_CHECK(cudaGetLastError());
  TTP_CUDA_CHECK(cudaMemcpyAsync(h_out, out, sizeof(cplx) * n_inst, cudaMemcpyDeviceToHost, s));
  TTP_CUDA_CHECK(cudaStreamSynchronize(s));
  return TTP_OK;
}
