// K9: Monte Carlo pricer for the min-option (price_monte_carlo,
// pricers.py:297-350), the first "next" row of SURVEY.md 8(f).
//
// The reference draws numpy PCG64 streams per chunk (SeedSequence.spawn,
// pricers.py:316-323); those streams are not reproduced (parity is
// statistical).  Here every path is a pure function of
// (seed, path index): Philox4x32-10 (Salmon et al., SC'11 / Random123) with
// key = seed and counter = (path lo, path hi, draw, 0x4D43) gives four 32-bit
// words -> two 53-bit uniforms -> one Box-Muller pair.  Correlation enters
// through the Cholesky factor (pricers.py:325, 329), exactly as the
// reference: terminal_exact S = s0 exp(drift + vol L z), euler_path
// S <- S (1 + r dt + sigma sqrt(dt) L z) for n_steps, S = max(S, 0).
// One thread per path (grid-stride); per-thread (sum, sum of squares) of
// the discounted payoff reduce through a fixed tree in each CTA and the CTA
// partials in CTA order, so the result is bitwise reproducible.
#include "ttp_internal.h"
#include "launch.h"

namespace {

constexpr int MC_THREADS = 256;
constexpr int MC_MAX_BLOCKS = 148 * 8;
constexpr int MC_MAXD = 64;
constexpr uint32_t MC_TAG = 0x4D43u;

struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ inline U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// 53-bit uniform in (0, 1) from two 32-bit words
__device__ __forceinline__ double u53(uint32_t lo, uint32_t hi) {
  const uint64_t v = ((uint64_t)hi << 32) | lo;
  return ((double)(v >> 11) + 0.5) * 0x1.0p-53;
}

// normals 2p, 2p+1 of draw group g for path s
__device__ __forceinline__ void normal_pair(uint64_t s, uint32_t g, uint32_t k0, uint32_t k1, double& z0,
                                            double& z1) {
  const U4 o = philox4x32_10(U4{(uint32_t)s, (uint32_t)(s >> 32), g, MC_TAG}, k0, k1);
  const double u1 = u53(o.x, o.y), u2 = u53(o.z, o.w);
  const double rad = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  z0 = rad * cs;
  z1 = rad * sn;
}

// d normals of draw step t into z
__device__ __forceinline__ void normals(uint64_t s, int t, int d, uint32_t k0, uint32_t k1, double* z) {
  const int np = (d + 1) / 2;
  for (int p = 0; p < np; ++p) {
    double a, b;
    normal_pair(s, (uint32_t)(t * np + p), k0, k1, a, b);
    z[2 * p] = a;
    if (2 * p + 1 < d) z[2 * p + 1] = b;
  }
}

__global__ void __launch_bounds__(MC_THREADS)
mc_path_kernel(const double* __restrict__ params, long long pstride, int d, long long n,
               const unsigned long long* __restrict__ seeds, int scheme, int n_steps,
               double2* __restrict__ partial) {
  extern __shared__ double prm[];
  const int inst = blockIdx.y;
  const double* P = params + inst * pstride;
  const int np = 5 * d + d * d + 3;
  for (int e = threadIdx.x; e < np; e += blockDim.x) prm[e] = P[e];
  __syncthreads();
  const double* s0 = prm;
  const double* drift = prm + d;
  const double* vol = prm + 2 * d;
  const double* rates = prm + 3 * d;
  const double* sigma = prm + 4 * d;
  const double* L = prm + 5 * d;
  const double strike = prm[5 * d + d * d];
  const double disc = prm[5 * d + d * d + 1];
  const double dt = prm[5 * d + d * d + 2];
  const double sdt = sqrt(dt);
  const unsigned long long seed = seeds[inst];
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  double z[MC_MAXD], st[MC_MAXD];
  double sum = 0.0, sq = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += stride) {
    double mn;
    if (scheme == 0) {
      normals((uint64_t)s, 0, d, k0, k1, z);
      mn = INFINITY;
      for (int j = 0; j < d; ++j) {
        double w = 0.0;
        for (int k = 0; k <= j; ++k) w = fma(L[j * d + k], z[k], w);
        mn = fmin(mn, s0[j] * exp(drift[j] + vol[j] * w));
      }
    } else {
      for (int j = 0; j < d; ++j) st[j] = s0[j];
      for (int t = 0; t < n_steps; ++t) {
        normals((uint64_t)s, t, d, k0, k1, z);
        for (int j = 0; j < d; ++j) {
          double w = 0.0;
          for (int k = 0; k <= j; ++k) w = fma(L[j * d + k], z[k], w);
          st[j] *= 1.0 + rates[j] * dt + sigma[j] * (w * sdt);
        }
      }
      mn = INFINITY;
      for (int j = 0; j < d; ++j) mn = fmin(mn, fmax(st[j], 0.0));
    }
    const double pay = disc * fmax(mn - strike, 0.0);
    sum += pay;
    sq = fma(pay, pay, sq);
  }
  // fixed-order block reduction
  __shared__ double rs[MC_THREADS], rq[MC_THREADS];
  rs[threadIdx.x] = sum;
  rq[threadIdx.x] = sq;
  __syncthreads();
  for (int h = MC_THREADS / 2; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) {
      rs[threadIdx.x] += rs[threadIdx.x + h];
      rq[threadIdx.x] += rq[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(long long)inst * gridDim.x + blockIdx.x] = make_double2(rs[0], rq[0]);
}

__global__ void mc_final_kernel(const double2* __restrict__ partial, int nblk, double2* __restrict__ out) {
  const int inst = blockIdx.x;
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < nblk; ++k) {
      const double2 v = partial[(long long)inst * nblk + k];
      a += v.x;
      b += v.y;
    }
    out[inst] = make_double2(a, b);
  }
}

int mc_blocks(long long n) {
  const long long want = (n + MC_THREADS * 8 - 1) / (MC_THREADS * 8);
  return (int)(want < 1 ? 1 : (want > MC_MAX_BLOCKS ? MC_MAX_BLOCKS : want));
}

}  // namespace

extern "C" int32_t ttp_mc_param_count(int32_t d) { return 5 * d + d * d + 3; }

extern "C" size_t ttp_mc_workspace(int32_t n_inst, int64_t n_samples) {
  if (n_inst < 0 || n_samples < 0) return 0;
  return sizeof(double2) * ((size_t)n_inst * mc_blocks(n_samples) + (size_t)n_inst) +
         sizeof(unsigned long long) * (size_t)n_inst + 256;
}

extern "C" int ttp_mc_price(const double* d_params, int64_t param_stride, int32_t d, int32_t n_inst,
                            int64_t n_samples, const uint64_t* h_seeds, int32_t scheme, int32_t n_steps,
                            double* h_out, void* d_ws, size_t ws_bytes, void* stream) {
  if (d < 1 || d > MC_MAXD || n_inst < 0 || n_samples < 2 || (scheme != 0 && scheme != 1) ||
      (scheme == 1 && n_steps < 1) || param_stride < ttp_mc_param_count(d) || !h_seeds || !h_out)
    return ttp_fail(TTP_ERR_INVALID, "mc_price: invalid argument");
  if (ws_bytes < ttp_mc_workspace(n_inst, n_samples))
    return ttp_fail(TTP_ERR_WORKSPACE, "mc_price: workspace too small");
  if (n_inst == 0) return TTP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int nblk = mc_blocks(n_samples);
  double2* part = reinterpret_cast<double2*>(d_ws);
  double2* out = part + (size_t)n_inst * nblk;
  unsigned long long* seeds = reinterpret_cast<unsigned long long*>(out + n_inst);
  TTP_CUDA_CHECK(cudaMemcpyAsync(seeds, h_seeds, sizeof(unsigned long long) * n_inst, cudaMemcpyHostToDevice, s));
  const size_t smem = sizeof(double) * ttp_mc_param_count(d);
  dim3 grid((unsigned)nblk, (unsigned)n_inst);
  {
    LaunchScope _ls(KC_MC, s);
    mc_path_kernel<<<grid, MC_THREADS, smem, s>>>(d_params, param_stride, d, n_samples, seeds, scheme,
                                                  scheme == 1 ? n_steps : 0, part);
  }
  TTP_CUDA_CHECK(cudaGetLastError());
  {
    LaunchScope _ls(KC_MC_FINAL, s);
    mc_final_kernel<<<n_inst, 32, 0, s>>>(part, nblk, out);
  }
  TTP_CUDA_CHECK(cudaGetLastError());
  TTP_CUDA_CHECK(cudaMemcpyAsync(h_out, out, sizeof(double2) * n_inst, cudaMemcpyDeviceToHost, s));
  TTP_CUDA_CHECK(cudaStreamSynchronize(s));
  return TTP_OK;
}

extern "C" int ttp_philox4x32(const uint32_t* h_ctr, const uint32_t* h_key, uint32_t* h_out) {
  if (!h_ctr || !h_key || !h_out) return ttp_fail(TTP_ERR_INVALID, "philox4x32: null argument");
  // same routine the kernel inlines (host instantiation of the __host__ __device__ body)
  const U4 o = philox4x32_10(U4{h_ctr[0], h_ctr[1], h_ctr[2], h_ctr[3]}, h_key[0], h_key[1]);
  h_out[0] = o.x;
  h_out[1] = o.y;
  h_out[2] = o.z;
  h_out[3] = o.w;
  return TTP_OK;
}
