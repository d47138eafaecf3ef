// K8: dense full-grid contour sum  sum_grid phi(-z) vhat(z)
// (_dense_contour_sum, pricers.py:185-196).
//
// The reference walks flat C-order indices in chunks of 2^20 and sums
// phi(-z) * vhat(z) chunk by chunk.  Here the flat range is split into a
// fixed number of contiguous slabs per instance (one CTA each); every term is
// evaluated in registers (nothing is materialised, so the kernel is FP64
// bound, not HBM bound) and the per-slab sums are combined in slab order by
// a second kernel, so the result is independent of scheduling.
#include "ttp_internal.h"
#include "launch.h"

namespace {

constexpr int DENSE_THREADS = 256;
constexpr int DENSE_SLABS = 1184;  // 8 CTAs per SM on 148 SMs

__global__ void __launch_bounds__(DENSE_THREADS)
dense_partial_kernel(OracleDev phi, OracleDev vhat, long long first, long long count,
                     cplx* __restrict__ part) {
  const int inst = blockIdx.y;
  const int slab = blockIdx.x;
  const long long per = (count + gridDim.x - 1) / gridDim.x;
  const long long lo = first + slab * per;
  const long long hi = min(first + count, lo + per);
  const int d = phi.d;
  cplx acc = mk(0.0, 0.0);
  int idx[TTP_MAX_D];
  for (long long f = lo + threadIdx.x; f < hi; f += DENSE_THREADS) {
    long long rem = f;
    for (int k = d - 1; k >= 0; --k) {
      const int n = phi.shape[k];
      const long long q = rem / n;
      idx[k] = (int)(rem - q * n);
      rem = q;
    }
    const cplx a = oracle_value(phi, inst, idx);
    const cplx b = oracle_value(vhat, inst, idx);
    acc = cfma(a, b, acc);
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
