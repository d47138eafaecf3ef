#include <cstdio>
// Host runtime of the B200 TT-Fourier pricer: the C ABI entry points and the
// batched TT-cross sweep driver.
//
// tt_cross (cross.py:358-453) is a short, strictly sequential host loop in
// the reference.  Here the loop runs natively: per bond it launches the
// fiber evaluator (K1/K2, all instances x all entries) and the bond kernel
// (K3-K5, one CTA per instance), then after each directional pass the
// convergence check (K6).  Only the per-instance convergence scalars and
// status codes come back to the host between sweeps; pivot sets, cores and
// fibers stay resident in HBM.  Instances that converged or failed are
// masked out of later sweeps (ragged batches).
#include <cstring>
#include <string>
#include <vector>

#include "ttp_internal.h"
#include "dev_knobs.h"
#include "launch.h"
#include "k_bond.h"

// conv-check kernels from k_tt.cu
__global__ void conv_site0_kernel(const cplx* cores, long long stride, long long off0, int r1,
                                  const int* idx, int d, long long m, cplx* V, long long vstride,
                                  const int* active);
__global__ void conv_site_kernel(const cplx* cores, long long stride, long long offk, int ra, int n,
                                 int rb, const int* perm, const int* goff, const cplx* Vin,
                                 cplx* Vout, long long vstride, const int* active);
__global__ void sample_diff_kernel(const cplx* exact, const cplx* approx, long long m,
                                   long long estride, long long astride, double* out,
                                   const int* active);
size_t conv_site_smem(int ra, int rb, int threads);
int conv_site_dmma_nt(int rb);
cudaError_t launch_conv_site_dmma(const cplx* cores, long long stride, long long offk, int ra, int n,
                                  int rb, const int* perm, const int* goff, const cplx* vin, cplx* vout,
                                  long long vstride, const int* active, int n_inst, cudaStream_t s,
                                  long long off0 = 0, const int* idx0 = nullptr, int idx_d = 0,
                                  int mode = 0, int n0 = 0);

// TTP_CONV_DMMA=0 selects the scalar-FMA site kernel (dev build A/B checks).
bool conv_dmma_enabled() {
  static const bool on = [] {
    const char* e = ttp_dev_env("TTP_CONV_DMMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

namespace {
thread_local std::string g_last_error;

__global__ void replicate_kernel(const int* __restrict__ src, long long n, int* __restrict__ dst,
                                 long long stride) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[blockIdx.y * stride + e] = src[e];
}

// row-major (rows x cols) numpy matrices -> column-major blocks
__global__ void to_colmajor_kernel(const cplx* __restrict__ src, long long rows, int cols,
                                   cplx* __restrict__ dst, long long dstride) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const long long i = e / cols;
  const int j = (int)(e - i * cols);
  dst[blockIdx.y * dstride + (long long)j * rows + i] = src[blockIdx.y * rows * cols + e];
}

long long sat_mul(long long a, long long b, long long cap) {
  if (a == 0 || b == 0) return 0;
  if (a > cap / b) return cap;
  return std::min(cap, a * b);
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct CrossWs {
  cplx *A, *W, *B, *V0, *V1, *exact, *cores_unused;
  int *iwork, *active, *status, *err_bond;
  double* dwork;
  double* diff;
  long long mat_stride, v_stride, iw_stride, dw_stride;
  size_t bytes;
};

CrossWs carve_cross(const ttp_cross_layout& L, int n_inst, long long M, unsigned char* base) {
  CrossWs w{};
  // padded so row slices of up to 16 cluster CTAs (ceil(m / C) rows each) fit
  const long long mr = (L.max_rows + 16) * (long long)L.max_rank;
  w.mat_stride = mr;
  w.v_stride = M * (long long)L.max_rank;
  w.iw_stride = 2 * (L.max_rows + 16);  // also the per-CTA row arrays of big cluster jobs
  w.dw_stride = 2 * (L.max_rows + 16);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  w.A = (cplx*)take(sizeof(cplx) * mr * n_inst);
  w.W = (cplx*)take(sizeof(cplx) * mr * n_inst);
  w.B = (cplx*)take(sizeof(cplx) * mr * n_inst);
  w.V0 = (cplx*)take(sizeof(cplx) * w.v_stride * n_inst);
  w.V1 = (cplx*)take(sizeof(cplx) * w.v_stride * n_inst);
  w.exact = (cplx*)take(sizeof(cplx) * M * n_inst);
  w.iwork = (int*)take(sizeof(int) * w.iw_stride * n_inst);
  w.dwork = (double*)take(sizeof(double) * w.dw_stride * n_inst);
  w.active = (int*)take(sizeof(int) * n_inst);
  w.status = (int*)take(sizeof(int) * n_inst);
  w.err_bond = (int*)take(sizeof(int) * n_inst);
  w.diff = (double*)take(sizeof(double) * 2 * n_inst);
  w.bytes = off;
  return w;
}

}  // namespace

int ttp_record_cuda_error(cudaError_t e) {
  g_last_error = std::string("CUDA error: ") + cudaGetErrorName(e) + ": " + cudaGetErrorString(e);
  return TTP_ERR_CUDA;
}

int ttp_fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

extern "C" int ttp_abi_version(void) { return TTP_ABI_VERSION; }

extern "C" const char* ttp_last_error(void) { return g_last_error.c_str(); }

extern "C" int ttp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

extern "C" int ttp_oracle_eval(const ttp_oracle* oracle, const int32_t* d_shape, int32_t n_inst,
                               const int32_t* d_idx, int64_t m, double* d_out, void* stream) {
  if (!oracle || oracle->d < 1 || oracle->d > TTP_MAX_D || n_inst < 0 || m < 0)
    return ttp_fail(TTP_ERR_INVALID, "oracle_eval: invalid arguments");
  if (oracle->kind < TTP_ORACLE_PHI_GBM || oracle->kind > TTP_ORACLE_TABLE)
    return ttp_fail(TTP_ERR_INVALID, "oracle_eval: unknown oracle kind");
  OracleDev o = oracle_dev_from(*oracle, d_shape);
  launch_oracle_points(o, n_inst, d_idx, m, reinterpret_cast<cplx*>(d_out), (cudaStream_t)stream);
  TTP_CUDA_CHECK(cudaGetLastError());
  return TTP_OK;
}

extern "C" int ttp_eval_fibers(const ttp_oracle* oracle, const int32_t* d_shape, int32_t n_inst,
                               int32_t layout, int32_t axis, int32_t axis_size, const int32_t* d_left,
                               int32_t n_left, const int32_t* d_right, int32_t n_right, double* d_out,
                               int64_t out_stride, void* stream) {
  if (!oracle || oracle->d < 1 || oracle->d > TTP_MAX_D || n_inst < 0 || n_left < 1 || n_right < 1 ||
      axis_size < 1 || axis < 0 || axis >= oracle->d || (layout != 0 && layout != 1) || !d_out)
    return ttp_fail(TTP_ERR_INVALID, "eval_fibers: invalid arguments");
  if (oracle->kind < TTP_ORACLE_PHI_GBM || oracle->kind > TTP_ORACLE_TABLE)
    return ttp_fail(TTP_ERR_INVALID, "eval_fibers: unknown oracle kind");
  const long long rows = layout == 0 ? (long long)n_left * axis_size : (long long)axis_size * n_right;
  const long long cols = layout == 0 ? n_right : n_left;
  if (out_stride < rows * cols) return ttp_fail(TTP_ERR_INVALID, "eval_fibers: out_stride too small");
  if (n_inst == 0) return TTP_OK;
  OracleDev o = oracle_dev_from(*oracle, d_shape);
  FiberJob f{};
  f.mode = layout;
  f.rl = n_left;
  f.na = axis_size;
  f.rr = n_right;
  f.kl = axis;
  // the index sets are shared by all instances (set_stride 0), rows packed
  // at their tuple length
  f.left = SetView{d_left, 0, 0, axis};
  f.right = SetView{d_right, 0, 0, oracle->d - axis - 1};
  f.out = reinterpret_cast<cplx*>(d_out);
  f.out_stride = out_stride;
  f.ld = rows;
  launch_fiber(o, f, nullptr, n_inst, (cudaStream_t)stream);
  TTP_CUDA_CHECK(cudaGetLastError());
  return TTP_OK;
}

extern "C" int ttp_cross_layout_of(int32_t d, const int32_t* h_shape, int32_t bond_dim,
                                   ttp_cross_layout* out) {
  if (d < 1 || d > TTP_MAX_D || bond_dim < 1 || bond_dim > 64 || !h_shape || !out)
    return ttp_fail(TTP_ERR_INVALID, "cross layout: need 1 <= d <= 64 and 1 <= bond_dim <= 64");
  std::memset(out, 0, sizeof(*out));
  const long long cap = 1LL << 40;
  for (int k = 0; k <= d; ++k) {
    long long pre = 1, suf = 1;
    for (int j = 0; j < k; ++j) pre = sat_mul(pre, h_shape[j], cap);
    for (int j = k; j < d; ++j) suf = sat_mul(suf, h_shape[j], cap);
    long long r = std::min<long long>(bond_dim, std::min(pre, suf));
    if (d == 1) r = 1;
    out->ranks[k] = (int)r;
  }
  out->ranks[0] = 1;
  out->ranks[d] = 1;
  long long off = 0, soff = 0, maxrows = 1;
  int maxr = 1;
  for (int k = 0; k < d; ++k) {
    out->core_offsets[k] = off;
    off += (long long)out->ranks[k] * h_shape[k] * out->ranks[k + 1];
  }
  out->core_offsets[d] = off;
  out->core_stride = off;
  for (int k = 0; k <= d; ++k) {
    out->set_offsets[k] = soff;
    soff += (long long)out->ranks[k] * d;
    maxr = std::max(maxr, out->ranks[k]);
  }
  out->set_stride = soff;
  for (int k = 1; k < d; ++k) {
    maxrows = std::max(maxrows, (long long)out->ranks[k - 1] * h_shape[k - 1]);  // L2R
    maxrows = std::max(maxrows, (long long)h_shape[k] * out->ranks[k + 1]);      // R2L
  }
  out->max_rows = maxrows;
  out->max_rank = maxr;
  return TTP_OK;
}

extern "C" size_t ttp_cross_workspace(const ttp_cross_problem* prob) {
  ttp_cross_layout L;
  if (!prob || ttp_cross_layout_of(prob->d, prob->h_shape, prob->cfg.bond_dim, &L) != TTP_OK) return 0;
  return carve_cross(L, prob->n_inst, prob->cfg.n_conv_samples, nullptr).bytes;
}

namespace {

SetView set_view(const int* base, const ttp_cross_layout& L, int k, int d) {
  SetView v;
  v.base = base;
  v.set_stride = L.set_stride;
  v.offset = L.set_offsets[k];
  v.d = d;
  return v;
}

// Bond path selection.  The release library picks the path from the block
// shape alone, never from the batch size, so an option's cores and price do
// not depend on how many other options share its launch (the reference's
// determinism contracts, test_cross.py:180-190 and test_bench_cli.py:151-158):
//   * blocks of >= 1 MB (cfg4, cfg5): global-slice clusters of 2 CTAs, the
//     256-thread two-CTAs-per-SM instantiation (ck_tp) when its carve fits
//     twice per SM (r <= 32), else the 512-thread one (ck_lat, r = 64);
//   * smaller blocks (cfg1-3, the reference test suite): the one-CTA-per-
//     instance kernel (k_bond_v0.cu) after the fiber kernel.
// Measured on B200 (profiles/r01/path_sweep*.log): at throughput batch sizes
// these are the fastest paths for their block sizes.  Dev builds keep the
// other paths reachable for A/B runs: TTP_BOND_PATH=v0 | cluster (shared-
// memory clusters) | l2:C (global-slice clusters of C CTAs), TTP_CK=lat|tp.
int bond_path_mode() {
  static const int v = [] {
    const char* e = ttp_dev_env("TTP_BOND_PATH");
    if (e && std::strcmp(e, "v0") == 0) return 1;
    if (e && std::strcmp(e, "cluster") == 0) return 2;
    if (e && std::strncmp(e, "l2", 2) == 0) return 3;
    return 0;
  }();
  return v;
}

// Cluster size of the global-slice mode (dev: TTP_BOND_PATH=l2:C); powers of
// two only, since the row split assumes it (3-CTA clusters fault).
int l2_cluster_size() {
  static const int v = [] {
    const char* e = ttp_dev_env("TTP_BOND_PATH");
    int c = (e && std::strncmp(e, "l2:", 3) == 0) ? std::max(1, atoi(e + 3)) : 2;
    int p = 1;
    while (p * 2 <= std::min(c, 16)) p *= 2;
    return p;
  }();
  return v;
}

// dev: TTP_CK=lat|tp forces a global-slice instantiation
static int tp_knob() {
  static const int forced = [] {
    const char* e = ttp_dev_env("TTP_CK");
    if (e && std::strcmp(e, "lat") == 0) return 0;
    if (e && std::strcmp(e, "tp") == 0) return 1;
    return -1;
  }();
  return forced;
}

size_t smem_optin_limit() {
  static std::mutex mu;
  static std::map<std::pair<int, int>, size_t> memo;
  return ttp_device_memo(memo, mu, 0, [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) v = 0;
    return (size_t)v;
  });
}

// Largest power of two <= min(want, m / r): every CTA of a cluster must own
// at least r rows, and the row split assumes a power of two.
int pow2_cluster(int want, int m, int r) {
  const int cap = std::max(1, std::min(want, m / std::max(1, r)));
  int p = 1;
  while (p * 2 <= cap) p *= 2;
  return p;
}

// One bond for every active instance: fibers + column basis + maxvol +
// factor (path chosen from the block shape, see above).
int run_bond(const OracleDev& o, const FiberJob& f, const BondJob& bj, const CrossWs& w, int n,
             cudaStream_t s) {
  const long long block_bytes = (long long)bj.m * bj.r * (long long)sizeof(cplx);
  const int mode = bond_path_mode();
  if (mode == 3 || (mode == 0 && block_bytes >= (1LL << 20))) {
    ClusterJob cj{};
    cj.b = bj;
    cj.cl = pow2_cluster(l2_cluster_size(), bj.m, bj.r);
    cj.src_mode = 0;
    cj.fiber_fast = fiber_fast_enabled() ? 1 : 0;
    cj.oracle = o;
    cj.fiber = f;
    cj.Qg = w.A;
    cj.q_stride = w.mat_stride;
    cj.Wg = w.W;
    cj.Sg = w.B;
    cj.wg_stride = w.mat_stride;
    const int act_tp = ck_tp::max_active_clusters(cj), act_lat = ck_lat::max_active_clusters(cj);
    const bool tp = tp_knob() >= 0 ? tp_knob() == 1 : act_tp > act_lat;
#ifdef TTP_DEV
    if (std::getenv("TTP_DEBUG_ACT")) std::fprintf(stderr, "run_bond m=%d r=%d act_tp=%d act_lat=%d\n", bj.m, bj.r, act_tp, act_lat);
#endif
    if (tp && act_tp > 0) {
      TTP_CUDA_CHECK(ck_tp::launch_cluster_bond(cj, n, s));
      return TTP_OK;
    }
    if (!tp && act_lat > 0) {
      TTP_CUDA_CHECK(ck_lat::launch_cluster_bond(cj, n, s));
      return TTP_OK;
    }
  }
  if (mode == 2) {
    const int C = ck_lat::pick_cluster_size(bj.m, bj.r, smem_optin_limit());
    ClusterJob cj{};
    cj.b = bj;
    cj.cl = C;
    cj.src_mode = 0;
    cj.fiber_fast = fiber_fast_enabled() ? 1 : 0;
    cj.oracle = o;
    cj.fiber = f;
    cj.Qg = w.A;
    cj.q_stride = w.mat_stride;
    if (C > 0 && ck_lat::max_active_clusters(cj) > 0) {
      TTP_CUDA_CHECK(ck_lat::launch_cluster_bond(cj, n, s));
      return TTP_OK;
    }
  }
  launch_fiber(o, f, w.active, n, s);
  TTP_CUDA_CHECK(launch_bond(bj, n, s));
  return TTP_OK;
}

int run_conv_check(const ttp_cross_problem& P, const ttp_cross_layout& L, const CrossWs& w,
                   const ttp_cross_out& out, const int* d_active, cudaStream_t s) {
  const int d = P.d, n = P.n_inst;
  const long long M = P.cfg.n_conv_samples;
  const cplx* cores = reinterpret_cast<const cplx*>(out.d_cores);
  const int r1 = L.ranks[1];
  // site 1 on the DMMA path gathers its input rows straight from the first
  // core (row i_0 of each sample), so the site-0 rows are not materialised
  const bool gather0 = d >= 2 && conv_dmma_enabled() && conv_site_dmma_nt(L.ranks[2]) > 0;
  if (!gather0) {
    const long long tot = M * r1;
    dim3 grid((unsigned)((tot + 255) / 256), (unsigned)n);
    {
      LaunchScope _ls(KC_CONV_SITE0, s);
      conv_site0_kernel<<<grid, 256, 0, s>>>(cores, L.core_stride, L.core_offsets[0], r1, P.d_conv_idx,
                                             d, M, w.V0, w.v_stride, d_active);
    }
  }
  cplx* vin = w.V0;
  cplx* vout = w.V1;
  // site 1 as a dense (i_1, i_0) table when that has fewer rows than the
  // sample set (cfg1-4): one product per pair, written over V0 (free, since
  // site 0 is not materialised); site 2 gathers from it
  const long long tab_rows = d >= 3 ? (long long)P.h_shape[0] * P.h_shape[1] : 0;
  const bool table = gather0 && d >= 3 && tab_rows <= M && conv_site_dmma_nt(L.ranks[3]) > 0;
  if (table) std::swap(vin, vout);  // site 1 writes V0, site 2 reads it
  long long goff = 0;
  for (int k = 0; k < d; ++k) {
    if (k >= 1) {
      const int ra = L.ranks[k], rb = L.ranks[k + 1], nk = P.h_shape[k];
      if (conv_dmma_enabled() && conv_site_dmma_nt(rb) > 0) {
        LaunchScope _ls(KC_CONV_SITE, s);
        const int mode = (gather0 && k == 1) ? (table ? 2 : 1) : (table && k == 2) ? 3 : 0;
        TTP_CUDA_CHECK(launch_conv_site_dmma(cores, L.core_stride, L.core_offsets[k], ra, nk, rb,
                                             P.d_conv_perm + (long long)k * M, P.d_conv_off + goff, vin,
                                             vout, w.v_stride, d_active, n, s, L.core_offsets[0],
                                             P.d_conv_idx, d, mode, P.h_shape[0]));
        std::swap(vin, vout);
        goff += P.h_shape[k] + 1;
        continue;
      }
      const size_t smem = conv_site_smem(ra, rb, 256);
      TTP_CUDA_CHECK(ensure_max_smem((const void*)conv_site_kernel));
      dim3 grid((unsigned)nk, (unsigned)n);
      {
        LaunchScope _ls(KC_CONV_SITE, s);
        conv_site_kernel<<<grid, 256, smem, s>>>(cores, L.core_stride, L.core_offsets[k], ra, nk, rb,
                                                 P.d_conv_perm + (long long)k * M, P.d_conv_off + goff,
                                                 vin, vout, w.v_stride, d_active);
      }
      std::swap(vin, vout);
    }
    goff += P.h_shape[k] + 1;
  }
  {
    LaunchScope _ls(KC_SAMPLE_DIFF, s);
    sample_diff_kernel<<<n, 1024, 0, s>>>(w.exact, vin, M, M, w.v_stride, w.diff, d_active);
  }
  TTP_CUDA_CHECK(cudaGetLastError());
  return TTP_OK;
}

}  // namespace

extern "C" int ttp_cross_run(const ttp_cross_problem* prob, ttp_cross_out* out, void* d_ws,
                             size_t ws_bytes, void* stream) {
  if (!prob || !out) return ttp_fail(TTP_ERR_INVALID, "cross_run: null argument");
  const ttp_cross_problem& P = *prob;
  const int d = P.d, n = P.n_inst;
  const ttp_cross_cfg& cfg = P.cfg;
  if (n < 0 || cfg.max_sweeps < 1 || cfg.n_conv_samples < 1 || cfg.eps_tol <= 0 || cfg.maxvol_slack < 0)
    return ttp_fail(TTP_ERR_INVALID, "cross_run: invalid configuration");
  ttp_cross_layout L;
  int st = ttp_cross_layout_of(d, P.h_shape, cfg.bond_dim, &L);
  if (st != TTP_OK) return st;
  for (int k = 0; k < d; ++k)
    if (P.h_shape[k] < 1) return ttp_fail(TTP_ERR_INVALID, "cross_run: invalid shape");
  const long long M = cfg.n_conv_samples;
  CrossWs w = carve_cross(L, n, M, reinterpret_cast<unsigned char*>(d_ws));
  if (ws_bytes < w.bytes) return ttp_fail(TTP_ERR_WORKSPACE, "cross_run: workspace too small");
  for (int i = 0; i < n; ++i) {
    out->h_status[i] = TTP_OK;
    out->h_error_bond[i] = -1;
    out->h_converged[i] = 0;
    out->h_sweeps[i] = 0;
    out->h_oracle_calls[i] = 0;
    out->h_conv_calls[i] = 0;
    out->h_final_diff[i] = INFINITY;
    for (int k = 0; k <= d; ++k) out->h_left_valid[i * (d + 1) + k] = (k == 0);
  }
  if (n == 0) return TTP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  OracleDev o = oracle_dev_from(P.oracle, P.d_shape);
  cplx* cores = reinterpret_cast<cplx*>(out->d_cores);

  TTP_CUDA_CHECK(cudaMemsetAsync(w.status, 0, sizeof(int) * n, s));
  // initial right sets (same draw for every instance: cross.py:402-403)
  {
    dim3 grid((unsigned)((L.set_stride + 255) / 256), (unsigned)n);
    {
      LaunchScope _ls(KC_MISC, s);
      replicate_kernel<<<grid, 256, 0, s>>>(P.d_right_init, L.set_stride, out->d_right, L.set_stride);
    }
    TTP_CUDA_CHECK(cudaMemsetAsync(out->d_left, 0, sizeof(int) * L.set_stride * n, s));
  }
  // exact oracle values at the convergence samples: identical every sweep
  // (tensor_train.py:191-196 with seed = cfg.seed), so evaluated once.
  launch_oracle_points(o, n, P.d_conv_idx, M, w.exact, s);
  TTP_CUDA_CHECK(cudaGetLastError());

  std::vector<int> active(n, 1), dev_status(n, 0), dev_bond(n, -1);
  std::vector<double> diffs(2 * n);
  const long long budget = cfg.oracle_call_budget;

  // oracle calls per directional pass (identical for every instance)
  long long calls_l2r = 0, calls_r2l = 0;
  if (d == 1) {
    calls_l2r = calls_r2l = P.h_shape[0];
  } else {
    for (int k = 1; k < d; ++k) calls_l2r += (long long)L.ranks[k - 1] * P.h_shape[k - 1] * L.ranks[k];
    calls_l2r += (long long)L.ranks[d - 1] * P.h_shape[d - 1];
    for (int k = d - 1; k >= 1; --k) calls_r2l += (long long)L.ranks[k] * P.h_shape[k] * L.ranks[k + 1];
    calls_r2l += (long long)P.h_shape[0] * L.ranks[1];
  }
  const int max_sweeps = (d == 1) ? 1 : cfg.max_sweeps;

  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    const long long calls = (sweep % 2 == 0) ? calls_l2r : calls_r2l;
    int n_active = 0;
    for (int i = 0; i < n; ++i) {
      active[i] = (out->h_status[i] == TTP_OK && !out->h_converged[i]) ? 1 : 0;
      if (active[i] && budget >= 0) {
        // _CallCounter raises before evaluating (cross.py:282-288); counts are
        // monotone, so the pass raises iff its final total exceeds the budget.
        const long long total = out->h_oracle_calls[i] + out->h_conv_calls[i] + calls + M;
        if (total > budget) {
          out->h_status[i] = TTP_ERR_BUDGET;
          active[i] = 0;
        }
      }
      n_active += active[i];
    }
    if (n_active == 0) break;
    TTP_CUDA_CHECK(cudaMemcpyAsync(w.active, active.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));

    BondJob bj{};
    bj.mat_stride = w.mat_stride;
    bj.A = w.A;
    bj.W = w.W;
    bj.B = w.B;
    bj.iwork = w.iwork;
    bj.iw_stride = w.iw_stride;
    bj.dwork = w.dwork;
    bj.dw_stride = w.dw_stride;
    bj.active = w.active;
    bj.status = w.status;
    bj.err_bond = w.err_bond;
    bj.rank_tol = 0.0;
    bj.max_iters = -1;
    bj.slack = cfg.maxvol_slack;
    bj.pairwise = 1;
    bj.sel_out = nullptr;
    bj.core_stride = L.core_stride;
    bj.set_stride = L.set_stride;
    bj.set_d = d;

    if (d == 1) {
      FiberJob f{};
      f.mode = 0;
      f.rl = 1;
      f.na = P.h_shape[0];
      f.rr = 1;
      f.kl = 0;
      f.left = set_view(out->d_left, L, 0, d);
      f.right = set_view(out->d_right, L, 1, d);
      f.out = cores + L.core_offsets[0];
      f.out_stride = L.core_stride;
      f.ld = P.h_shape[0];
      launch_fiber(o, f, w.active, n, s);
    } else if (sweep % 2 == 0) {
      for (int k = 1; k < d; ++k) {
        FiberJob f{};
        f.mode = 0;
        f.rl = L.ranks[k - 1];
        f.na = P.h_shape[k - 1];
        f.rr = L.ranks[k];
        f.kl = k - 1;
        f.left = set_view(out->d_left, L, k - 1, d);
        f.right = set_view(out->d_right, L, k, d);
        f.out = w.A;
        f.out_stride = w.mat_stride;
        f.ld = (long long)f.rl * f.na;
        bj.m = f.rl * f.na;
        bj.r = L.ranks[k];
        bj.write_mode = 1;
        bj.core_out = cores + L.core_offsets[k - 1];
        bj.set_out = out->d_left;
        bj.set_in = out->d_left;
        bj.set_out_off = L.set_offsets[k];
        bj.set_in_off = L.set_offsets[k - 1];
        bj.klen = k;
        bj.bond = k;
        bj.na = P.h_shape[k - 1];
        bj.rr = 1;
        st = run_bond(o, f, bj, w, n, s);
        if (st != TTP_OK) return st;
      }
      FiberJob f{};
      f.mode = 0;
      f.rl = L.ranks[d - 1];
      f.na = P.h_shape[d - 1];
      f.rr = 1;
      f.kl = d - 1;
      f.left = set_view(out->d_left, L, d - 1, d);
      f.right = set_view(out->d_right, L, d, d);
      f.out = cores + L.core_offsets[d - 1];
      f.out_stride = L.core_stride;
      f.ld = (long long)f.rl * f.na;
      launch_fiber(o, f, w.active, n, s);
    } else {
      for (int k = d - 1; k >= 1; --k) {
        FiberJob f{};
        f.mode = 1;
        f.rl = L.ranks[k];
        f.na = P.h_shape[k];
        f.rr = L.ranks[k + 1];
        f.kl = k;
        f.left = set_view(out->d_left, L, k, d);
        f.right = set_view(out->d_right, L, k + 1, d);
        f.out = w.A;
        f.out_stride = w.mat_stride;
        f.ld = (long long)f.na * f.rr;
        bj.m = f.na * f.rr;
        bj.r = L.ranks[k];
        bj.write_mode = 2;
        bj.core_out = cores + L.core_offsets[k];
        bj.set_out = out->d_right;
        bj.set_in = out->d_right;
        bj.set_out_off = L.set_offsets[k];
        bj.set_in_off = L.set_offsets[k + 1];
        bj.klen = d - k;
        bj.bond = k;
        bj.na = P.h_shape[k];
        bj.rr = L.ranks[k + 1];
        st = run_bond(o, f, bj, w, n, s);
        if (st != TTP_OK) return st;
      }
      FiberJob f{};
      f.mode = 1;
      f.rl = 1;
      f.na = P.h_shape[0];
      f.rr = L.ranks[1];
      f.kl = 0;
      f.left = set_view(out->d_left, L, 0, d);
      f.right = set_view(out->d_right, L, 1, d);
      f.out = cores + L.core_offsets[0];
      f.out_stride = L.core_stride;
      f.ld = (long long)f.na * f.rr;
      launch_fiber(o, f, w.active, n, s);
    }
    TTP_CUDA_CHECK(cudaGetLastError());
    st = run_conv_check(P, L, w, *out, w.active, s);
    if (st != TTP_OK) return st;
    TTP_CUDA_CHECK(cudaMemcpyAsync(diffs.data(), w.diff, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, s));
    TTP_CUDA_CHECK(cudaMemcpyAsync(dev_status.data(), w.status, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    TTP_CUDA_CHECK(cudaMemcpyAsync(dev_bond.data(), w.err_bond, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    TTP_CUDA_CHECK(cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i) {
      if (!active[i]) continue;
      if (dev_status[i] != TTP_OK) {
        out->h_status[i] = dev_status[i];
        out->h_error_bond[i] = dev_bond[i];
        continue;
      }
      out->h_sweeps[i] += 1;
      out->h_oracle_calls[i] += calls;
      out->h_conv_calls[i] += M;
      const double num = diffs[2 * i], den = diffs[2 * i + 1];
      const double diff = (den == 0.0) ? (num == 0.0 ? 0.0 : INFINITY) : num / den;
      out->h_final_diff[i] = diff;
      out->h_converged[i] = (diff <= cfg.eps_tol) ? 1 : 0;
      if (sweep % 2 == 0 && d > 1)
        for (int k = 1; k < d; ++k) out->h_left_valid[i * (d + 1) + k] = 1;
    }
  }
  return TTP_OK;
}

extern "C" size_t ttp_maxvol_workspace(int32_t n_mat, int64_t rows, int32_t cols) {
  if (n_mat < 0 || rows < 1 || cols < 1) return 0;
  const long long mr = rows * (long long)cols;
  size_t off = 0;
  off += 3 * align_up(sizeof(cplx) * mr * n_mat);
  off += align_up(sizeof(int) * 2 * rows * n_mat);
  off += align_up(sizeof(double) * 2 * rows * n_mat);
  off += align_up(sizeof(int) * cols * n_mat);
  off += align_up(sizeof(int) * n_mat);
  return off;
}

extern "C" int ttp_maxvol(int32_t n_mat, int64_t rows, int32_t cols, const double* d_mats, double slack,
                          int64_t max_iters, double rank_tol, int64_t* h_sel, int32_t* h_status,
                          void* d_ws, size_t ws_bytes, void* stream) {
  if (n_mat < 0 || rows < 1 || cols < 1 || cols > 64 || rows < cols)
    return ttp_fail(TTP_ERR_INVALID, "maxvol: need rows >= cols and 1 <= cols <= 64");
  if (ws_bytes < ttp_maxvol_workspace(n_mat, rows, cols))
    return ttp_fail(TTP_ERR_WORKSPACE, "maxvol: workspace too small");
  if (n_mat == 0) return TTP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const long long mr = rows * (long long)cols;
  unsigned char* base = reinterpret_cast<unsigned char*>(d_ws);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* p = base + off;
    off += align_up(bytes);
    return p;
  };
  BondJob bj{};
  bj.A = (cplx*)take(sizeof(cplx) * mr * n_mat);
  bj.W = (cplx*)take(sizeof(cplx) * mr * n_mat);
  bj.B = (cplx*)take(sizeof(cplx) * mr * n_mat);
  bj.iwork = (int*)take(sizeof(int) * 2 * rows * n_mat);
  bj.dwork = (double*)take(sizeof(double) * 2 * rows * n_mat);
  bj.sel_out = (int*)take(sizeof(int) * cols * n_mat);
  bj.status = (int*)take(sizeof(int) * n_mat);
  bj.err_bond = nullptr;
  bj.m = (int)rows;
  bj.r = cols;
  bj.mat_stride = mr;
  bj.iw_stride = 2 * rows;
  bj.dw_stride = 2 * rows;
  bj.active = nullptr;
  bj.rank_tol = rank_tol;
  bj.max_iters = max_iters;
  bj.slack = slack;
  bj.pairwise = 1;
  bj.sel_stride = cols;
  bj.write_mode = 0;
  TTP_CUDA_CHECK(cudaMemsetAsync(bj.status, 0, sizeof(int) * n_mat, s));
  const int C = bond_path_mode() == 1 ? 0 : ck_lat::pick_cluster_size((int)rows, cols, smem_optin_limit());
  ClusterJob cj{};
  cj.b = bj;
  cj.cl = C;
  cj.src_mode = 1;
  cj.src = reinterpret_cast<const cplx*>(d_mats);
  cj.src_stride = mr;
  cj.Qg = bj.A;
  cj.q_stride = mr;
  if (C > 0 && ck_lat::max_active_clusters(cj) > 0) {
    TTP_CUDA_CHECK(ck_lat::launch_cluster_bond(cj, n_mat, s));
  } else {
    dim3 grid((unsigned)((mr + 255) / 256), (unsigned)n_mat);
    {
      LaunchScope _ls(KC_MISC, s);
      to_colmajor_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const cplx*>(d_mats), rows, cols, bj.A, mr);
    }
    TTP_CUDA_CHECK(launch_bond(bj, n_mat, s));
  }
  std::vector<int> sel((size_t)cols * n_mat), stat(n_mat);
  TTP_CUDA_CHECK(cudaMemcpyAsync(sel.data(), bj.sel_out, sizeof(int) * cols * n_mat, cudaMemcpyDeviceToHost, s));
  TTP_CUDA_CHECK(cudaMemcpyAsync(stat.data(), bj.status, sizeof(int) * n_mat, cudaMemcpyDeviceToHost, s));
  TTP_CUDA_CHECK(cudaStreamSynchronize(s));
  for (long long e = 0; e < (long long)cols * n_mat; ++e) h_sel[e] = sel[e];
  for (int i = 0; i < n_mat; ++i) h_status[i] = stat[i];
  return TTP_OK;
}

extern "C" size_t ttp_column_basis_workspace(int32_t n_mat, int64_t rows, int32_t cols) {
  return ttp_maxvol_workspace(n_mat, rows, cols);
}

// _column_basis (cross.py:103-119) on n_mat (rows x cols) matrices, exactly as
// the bond kernel's global-slice path computes it for blocks of >= 1 MB
// (2-CTA clusters; TSQR + zlaqp2 on the triangle for 17 <= cols <= 32, the
// restated zlaqp2 otherwise).  d_q: n_mat column-major (rows x cols) Q
// factors, columns in pivot order.  h_status: TTP_OK or TTP_ERR_SINGULAR.
extern "C" int ttp_column_basis(int32_t n_mat, int64_t rows, int32_t cols, const double* d_mats,
                                double rank_tol, double* d_q, int32_t* h_status, void* d_ws,
                                size_t ws_bytes, void* stream) {
  if (n_mat < 0 || rows < 1 || cols < 1 || cols > 64 || rows < 2 * (int64_t)cols ||
      rows * (int64_t)cols * (int64_t)sizeof(cplx) < (1LL << 20))
    return ttp_fail(TTP_ERR_INVALID,
                    "column_basis: the global-slice path serves blocks of >= 1 MiB with rows >= 2 cols, cols <= 64");
  if (ws_bytes < ttp_column_basis_workspace(n_mat, rows, cols))
    return ttp_fail(TTP_ERR_WORKSPACE, "column_basis: workspace too small");
  if (n_mat == 0) return TTP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const long long mr = rows * (long long)cols;
  unsigned char* base = reinterpret_cast<unsigned char*>(d_ws);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* p = base + off;
    off += align_up(bytes);
    return p;
  };
  BondJob bj{};
  bj.A = (cplx*)take(sizeof(cplx) * mr * n_mat);
  bj.W = (cplx*)take(sizeof(cplx) * mr * n_mat);
  bj.B = (cplx*)take(sizeof(cplx) * mr * n_mat);
  bj.iwork = (int*)take(sizeof(int) * 2 * rows * n_mat);
  bj.dwork = (double*)take(sizeof(double) * 2 * rows * n_mat);
  bj.sel_out = (int*)take(sizeof(int) * cols * n_mat);
  bj.status = (int*)take(sizeof(int) * n_mat);
  bj.m = (int)rows;
  bj.r = cols;
  bj.mat_stride = mr;
  bj.iw_stride = 2 * rows;
  bj.dw_stride = 2 * rows;
  bj.rank_tol = rank_tol;
  bj.max_iters = -1;
  bj.slack = 0.01;
  bj.sel_stride = cols;
  bj.write_mode = 0;
  TTP_CUDA_CHECK(cudaMemsetAsync(bj.status, 0, sizeof(int) * n_mat, s));
  ClusterJob cj{};
  cj.b = bj;
  cj.cl = pow2_cluster(l2_cluster_size(), bj.m, bj.r);
  cj.src_mode = 1;
  cj.src = reinterpret_cast<const cplx*>(d_mats);
  cj.src_stride = mr;
  cj.Qg = reinterpret_cast<cplx*>(d_q);
  cj.q_stride = mr;
  cj.Wg = bj.W;
  cj.Sg = bj.B;
  cj.wg_stride = mr;
  cj.basis_only = 1;
  const int act_tp = ck_tp::max_active_clusters(cj), act_lat = ck_lat::max_active_clusters(cj);
  if (act_tp > act_lat && act_tp > 0) TTP_CUDA_CHECK(ck_tp::launch_cluster_bond(cj, n_mat, s));
  else if (act_lat > 0) TTP_CUDA_CHECK(ck_lat::launch_cluster_bond(cj, n_mat, s));
  else return ttp_fail(TTP_ERR_INVALID, "column_basis: no cluster configuration fits");
  std::vector<int> stat(n_mat);
  TTP_CUDA_CHECK(cudaMemcpyAsync(stat.data(), bj.status, sizeof(int) * n_mat, cudaMemcpyDeviceToHost, s));
  TTP_CUDA_CHECK(cudaStreamSynchronize(s));
  for (int i = 0; i < n_mat; ++i) h_status[i] = stat[i];
  return TTP_OK;
}

// ---------------------------------------------------------------------------
// One-call batch pricing: phi cross, vhat cross, inner product, prefactor.
extern "C" size_t ttp_price_tt_workspace(const ttp_price_problem* prob) {
  if (!prob) return 0;
  const size_t a = ttp_cross_workspace(&prob->phi), b = ttp_cross_workspace(&prob->vhat);
  return (a > b ? a : b) + 256 + 16 * (size_t)(prob->phi.n_inst > 0 ? prob->phi.n_inst : 1);
}

extern "C" int ttp_price_tt_batch(const ttp_price_problem* prob, ttp_cross_out* out_phi, ttp_cross_out* out_v,
                                  double* h_price, double* h_imag, void* d_ws, size_t ws_bytes,
                                  void* stream) {
  if (!prob || !out_phi || !out_v || !h_price || !h_imag || !prob->h_prefactor)
    return ttp_fail(TTP_ERR_INVALID, "price_tt_batch: null argument");
  const ttp_cross_problem& P = prob->phi;
  const ttp_cross_problem& V = prob->vhat;
  if (P.d != V.d || P.n_inst != V.n_inst || P.oracle.kind != TTP_ORACLE_PHI_GBM ||
      V.oracle.kind != TTP_ORACLE_VHAT_MIN)
    return ttp_fail(TTP_ERR_INVALID, "price_tt_batch: expects a PHI_GBM and a VHAT_MIN problem of one batch");
  for (int k = 0; k < P.d; ++k)
    if (P.h_shape[k] != V.h_shape[k]) return ttp_fail(TTP_ERR_INVALID, "price_tt_batch: shape mismatch");
  if (ws_bytes < ttp_price_tt_workspace(prob))
    return ttp_fail(TTP_ERR_WORKSPACE, "price_tt_batch: workspace too small");
  const int n = P.n_inst, d = P.d;
  if (n == 0) return TTP_OK;
  const size_t cross_ws = ws_bytes - 256 - 16 * (size_t)n;
  int st = ttp_cross_run(&P, out_phi, d_ws, cross_ws, stream);
  if (st != TTP_OK) return st;
  st = ttp_cross_run(&V, out_v, d_ws, cross_ws, stream);
  if (st != TTP_OK) return st;
  ttp_cross_layout Lp, Lv;
  if (ttp_cross_layout_of(d, P.h_shape, P.cfg.bond_dim, &Lp) != TTP_OK ||
      ttp_cross_layout_of(d, V.h_shape, V.cfg.bond_dim, &Lv) != TTP_OK)
    return ttp_fail(TTP_ERR_INVALID, "price_tt_batch: bad layout");
  ttp_tt_batch bra{}, ket{};
  bra.d = ket.d = d;
  bra.n_inst = ket.n_inst = n;
  bra.h_shape = V.h_shape;
  ket.h_shape = P.h_shape;
  bra.h_bonds = Lv.ranks;
  ket.h_bonds = Lp.ranks;
  bra.h_offsets = Lv.core_offsets;
  ket.h_offsets = Lp.core_offsets;
  bra.stride = Lv.core_stride;
  ket.stride = Lp.core_stride;
  bra.d_cores = out_v->d_cores;
  ket.d_cores = out_phi->d_cores;
  double* d_raw = reinterpret_cast<double*>(static_cast<unsigned char*>(d_ws) + cross_ws + 128);
  st = ttp_tt_inner(&bra, &ket, d_raw, stream);
  if (st != TTP_OK) return st;
  std::vector<double> raw(2 * (size_t)n);
  TTP_CUDA_CHECK(cudaMemcpyAsync(raw.data(), d_raw, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost,
                                 (cudaStream_t)stream));
  TTP_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  for (int i = 0; i < n; ++i) {
    const bool ok = out_phi->h_status[i] == TTP_OK && out_v->h_status[i] == TTP_OK;
    h_price[i] = ok ? prob->h_prefactor[i] * raw[2 * i] : NAN;
    h_imag[i] = ok ? prob->h_prefactor[i] * raw[2 * i + 1] : NAN;
  }
  return TTP_OK;
}

#ifdef TTP_DEV
// Phase clocks of whichever cluster instantiation ran since the last enable
// (dev build only; tools/phase_timing.py).
extern "C" int ttp_dev_phase_clocks(int enable, int64_t* out, int32_t n) {
  int64_t a[32] = {}, b[32] = {};
  int st = ck_tp::debug_phase_clocks(0, a, 32);
  if (st == TTP_OK) st = ck_lat::debug_phase_clocks(0, b, 32);
  if (st != TTP_OK) return st;
  if (out && n > 0) {
    const int64_t* src = (a[8] != 0 || a[1] != 0) ? a : b;
    for (int i = 0; i < n && i < 32; ++i) out[i] = src[i];
  }
  st = ck_tp::debug_phase_clocks(enable, nullptr, 0);
  if (st == TTP_OK) st = ck_lat::debug_phase_clocks(enable, nullptr, 0);
  return st;
}

// dev: per-instance [start ns][end ns][sm] of the throughput instantiation
extern "C" int ttp_dev_inst_times(int64_t* out, int32_t n) {
  std::vector<int64_t> a((size_t)3 * n), b((size_t)3 * n);
  int st = ck_tp::debug_inst_times(a.data(), n);
  if (st == TTP_OK) st = ck_lat::debug_inst_times(b.data(), n);
  const bool use_a = a[n] != 0;  // an end mark of instance 0
  for (size_t i = 0; i < a.size(); ++i) out[i] = use_a ? a[i] : b[i];
  std::fprintf(stderr, "inst times from %s\n", use_a ? "ck_tp" : "ck_lat");
  return st;
}
#endif
