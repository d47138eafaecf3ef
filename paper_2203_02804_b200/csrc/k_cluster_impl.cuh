// K3-K5 on thread-block clusters: the per-bond TT-cross linear algebra with
// the whole unfolding block resident in distributed shared memory.
//
// One cluster of C CTAs (C in {1,2,4,8,16}; 16 = non-portable size) owns one
// instance's m x r block.  CTA c holds rows [c*ms, c*ms + ms) of the block
// in its shared memory, column-major (ld = ms): a thread owns a row for the
// row-parallel phases, a warp owns a column for the column reductions, and
// every access is bank-conflict free.  Each sequential step of the
// reference algorithm is ONE cluster round: every CTA writes a small record
// (partial reductions, or its best candidate row plus that row's data) into
// its own shared memory, the cluster barrier (release/acquire) publishes it,
// and every CTA reads all C records over DSMEM and reduces them in rank
// order -- so all CTAs take bitwise-identical decisions with no second
// round and no global-memory traffic on the critical path.
//
// Global-slice mode (ClusterJob.Wg set; every throughput batch of blocks
// >= 1 MB): the row slices live in global memory instead (L2/HBM), only the
// small state stays in shared memory, and clusters of 2 CTAs keep 74
// (512-thread instantiation) or 148 (256-thread, two per SM) instances in
// flight.  Peers then read a swap winner's row straight from its owner's
// slice, ordered against the owner's rewrites by a split cluster barrier.
//
// Phases per bond (reference decision order, as in k_bond_v0.cu):
//   0  fibers: the oracle is evaluated straight into shared memory (no HBM
//      round trip for the sampled block; pricers.py:234-253 via cross.py:310-332)
//   A  zgeqp3 (zlaqp2: pivot, zlarfg, zlarf, partial-norm downdate/recompute)
//      distributed: 1 round per step (+1 when a norm recompute fires); each
//      step's update pass also forms the next step's partials (fused QR);
//      Q in compact-WY form -> orthonormal Q (global, L2-resident)  cross.py:103-119
//   B+C both starts fused in one read-only pass per round over Q: zlaqp2 on
//      Q^H and zgetrf partial pivoting (|Re|+|Im|)                 cross.py:184-187
//   D  _swap_to_dominance from each start; every CTA keeps a replicated
//      copy of B[sel, :] so the rank-1 update needs only the winning row;
//      in global-slice mode up to 4 rank-1 updates are deferred into
//      read-only row passes (bitwise the eager values)             cross.py:122-139
//   E  slogdet choice, cond screen, factor Q Q[sel]^-1 -> TT core     cross.py:191-205,349-355
//
// This file is compiled twice (k_cluster.cu, k_cluster_tp.cu) with different
// CTA shapes; CK_NS names the host API of each instantiation.
#ifndef CK_NS
#error "define CK_NS (and optionally CLUSTER_THREADS, CLUSTER_MIN_BLOCKS, QX_ROWS_DEF) before including"
#endif
#include <cooperative_groups.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "ttp_internal.h"
#include "bond_common.cuh"
#include "fiber_fast.cuh"
#include "dev_knobs.h"
#include "k_bond.h"
#include "launch.h"

namespace cg = cooperative_groups;

#ifdef TTP_DEV
namespace {
// Phase clocks of instance 0 / cluster rank 0 (dev build only;
// ttp_dev_phase_clocks, tools/phase_timing.py).
__device__ long long g_phase_clock[16];
__device__ int g_phase_enable;
#define PHASE_MARK(k)                                                           \
  do {                                                                          \
    if (g_phase_enable && inst == 0 && c.crank == 0 && threadIdx.x == 0)        \
      g_phase_clock[k] = clock64();                                             \
  } while (0)

// Sub-phase cycle accumulators (cluster rank 0, thread 0 of instance 0).
__device__ unsigned long long g_sub_clock[16];
// Per-instance start / end (globaltimer ns) and SM of cluster rank 0.
constexpr int INST_T_MAX = 8192;
__device__ long long g_inst_t[3][INST_T_MAX];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define INST_MARK(k)                                                                         \
  do {                                                                                       \
    if (g_phase_enable && c.crank == 0 && threadIdx.x == 0 && inst < INST_T_MAX) {           \
      g_inst_t[k][inst] = gtimer();                                                          \
      if (k == 0) {                                                                          \
        unsigned sm;                                                                         \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));                                      \
        g_inst_t[2][inst] = sm;                                                              \
      }                                                                                      \
    }                                                                                        \
  } while (0)
}  // namespace
#define SP_BEGIN(t)                                                             \
  long long t = (g_phase_enable && c.crank == 0 && threadIdx.x == 0 && blockIdx.x < (unsigned)c.C) \
                    ? clock64() : 0
#define SP(t, k)                                                                \
  do {                                                                          \
    if (t) {                                                                    \
      const long long _n = clock64();                                           \
      atomicAdd(&g_sub_clock[k], (unsigned long long)(_n - t));                 \
      t = _n;                                                                   \
    }                                                                           \
  } while (0)
#else
#define PHASE_MARK(k) do { } while (0)
#define INST_MARK(k) do { } while (0)
#define SP_BEGIN(t) do { } while (0)
#define SP(t, k) do { } while (0)
#endif

namespace {

constexpr int CT = CLUSTER_THREADS;
constexpr int CW = CT / 32;
constexpr int RMAX = 64;
#ifndef QX_ROWS_DEF
#define QX_ROWS_DEF 64
#endif
constexpr int QX_ROWS = QX_ROWS_DEF;  // rows per staged tile of the DMMA Q*X products
constexpr int LAZY_MAX = 4;  // most deferred swap updates (global-slice mode)
#ifdef TTP_DEV
__constant__ int g_lazy_f = LAZY_MAX;  // flush cadence of the deferred updates (1 = eager)
__constant__ int g_serpentine = 1;  // A/B of the serpentine row order
__constant__ int g_swap_filter = 1;  // bound-filtered swap passes (global-slice mode)
__constant__ int g_gram_dmma = 1;   // WY Gram on DMMA (else the 4x4 scalar tiles)
#else
constexpr int g_lazy_f = LAZY_MAX;
constexpr int g_serpentine = 1;
constexpr int g_swap_filter = 1;
constexpr int g_gram_dmma = 1;
#endif

struct __align__(16) Rec {
  double v;
  long long key;
  int row;
  int pad[3];
  cplx data[2 * RMAX + 4];
};

struct Cand {
  double v;
  long long key;
  int row;
};

struct __align__(16) WCand {
  double v;
  long long key;
  int row;  // global row, -1 = none
  int pad;
};

__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {
  return argmax_better(a.v, a.key, b.v, b.key);
}

__device__ __forceinline__ Cand warp_cand(Cand a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.key = __shfl_xor_sync(0xffffffffu, a.key, o);
    b.row = __shfl_xor_sync(0xffffffffu, a.row, o);
    if (cand_better(b, a)) a = b;
  }
  return a;
}

struct CC {
  int m, r, C, crank, row0, nrows, ldw;
  int ns_global;   // the row slices live in global memory (readable by every CTA)
  cplx* Ws;        // local slice, column-major, ld ldw
  cplx* Qg;        // global Q of this instance, column-major, ld m, logical columns
  cplx* aug;       // r x 2r
  cplx* selb;      // r x r replicated B[sel, :]
  cplx* vec;       // r
  cplx* vec2;      // 2r
  cplx* tau;       // r
  double* betas;   // r
  double* cn1;     // r
  double* cn2;     // r
  int* colmap;     // r
  int* flags;      // r
  int* first;      // r: row at LAPACK position t < r
  int* sel;        // r
  int* best;       // r
  int* starts;     // 2r
  double* vn1;     // ldw
  double* vn2;     // ldw
  int* rpos;       // ldw
  Rec* rec;        // 2 (parity double buffer)
  WCand* wrec;     // [2][CW] per-warp candidates (warp-granular rounds)
  WCand* wrec2;    // [2][CW] second candidate stream (fused starts)
  int* rpos2;      // ldw: LU positions (fused starts)
  cplx* sp;        // 8r scratch vectors (fused starts)
  double* qtile;   // QX_ROWS x (2r padded + 4) interleaved Q rows (DMMA Q*X), or nullptr
  cplx* wrow;      // [2][CW][r] per-warp candidate row data
  Cand* wcand;     // CW
  Ssq* wss;        // CW
  int* ibc;        // 8
  double* dbc;     // 8
  cplx* cbc;       // 8
  cplx* pend;      // [LAZY_MAX][r] deferred swap updates w_s (global-slice mode), or nullptr
  int* pendj;      // [LAZY_MAX] their pivot columns j_s
};

__device__ __forceinline__ cplx& Wl(const CC& c, int l, int t) { return c.Ws[(long long)t * c.ldw + l]; }
__device__ __forceinline__ const cplx* Qrow(const CC& c, int g) { return c.Qg + g; }  // stride m

// ---- row kernels with batched loads -------------------------------------
// In global-slice mode the row slice is L2-resident; issuing a batch of
// independent loads before the dependent FMAs keeps KB loads in flight per
// warp instead of one.  Accumulation order is unchanged (t ascending).
constexpr int KB = 8;

// Serpentine row passes: this thread's rows (l = tid + k CT) in ascending
// (rev = false) or descending order.  Consecutive passes over a slice run in
// opposite directions, so each pass starts on the lines the previous one
// touched last -- still in L2 when the working set (74 instances' slices)
// exceeds the L2 -- instead of on the ones evicted first.  Only used for
// passes whose per-row work is order independent.
#define FOR_MY_ROWS(l, nl, rev)                                                \
  for (int _k = 0, _nk = ((nl) + CT - 1) / CT; _k < _nk; ++_k)                 \
    if (const int l = threadIdx.x + ((rev) ? (_nk - 1 - _k) : _k) * CT; l < (nl))

// sum_t conj(S[t]) * W(l, t), t in [t0, r)
__device__ __forceinline__ cplx row_dotc(const CC& c, const cplx* S, int l, int t0, int r) {
  const cplx* p = c.Ws + l;
  const long long ld = c.ldw;
  cplx acc = mk(0.0, 0.0);
  int t = t0;
  for (; t + KB <= r; t += KB) {
    cplx x[KB];
#pragma unroll
    for (int q = 0; q < KB; ++q) x[q] = p[(t + q) * ld];
#pragma unroll
    for (int q = 0; q < KB; ++q) acc = cfmac(S[t + q], x[q], acc);
  }
  for (; t < r; ++t) acc = cfmac(S[t], p[t * ld], acc);
  return acc;
}

// W(l, t) -= S[t] * f, t in [t0, r)
__device__ __forceinline__ void row_sub_scaled(const CC& c, const cplx* S, cplx f, int l, int t0, int r) {
  cplx* p = c.Ws + l;
  const long long ld = c.ldw;
  int t = t0;
  for (; t + KB <= r; t += KB) {
    cplx x[KB];
#pragma unroll
    for (int q = 0; q < KB; ++q) x[q] = p[(t + q) * ld];
#pragma unroll
    for (int q = 0; q < KB; ++q) p[(t + q) * ld] = csub(x[q], cmul(S[t + q], f));
  }
  for (; t < r; ++t) p[t * ld] = csub(p[t * ld], cmul(S[t], f));
}

// W(l, colmap[j0 + q]) -= v * T[q], q in [0, n)   (column-basis updates)
__device__ __forceinline__ void row_sub_cols(const CC& c, const int* cols, const cplx* T, cplx v, int l,
                                             int n) {
  cplx* p = c.Ws + l;
  const long long ld = c.ldw;
  int q = 0;
  for (; q + KB <= n; q += KB) {
    cplx x[KB];
    long long off[KB];
#pragma unroll
    for (int u = 0; u < KB; ++u) {
      off[u] = cols[q + u] * ld;
      x[u] = p[off[u]];
    }
#pragma unroll
    for (int u = 0; u < KB; ++u) p[off[u]] = csub(x[u], cmul(v, T[q + u]));
  }
  for (; q < n; ++q) {
    cplx& a = p[cols[q] * ld];
    a = csub(a, cmul(v, T[q]));
  }
}

// sum over local rows l = l0, l0+32, ... < nl of conj(W(l, ci)) * W(l, cj)
__device__ __forceinline__ cplx col_dotc(const CC& c, int ci, int cj, int l0, int nl) {
  const cplx* a = c.Ws + (long long)ci * c.ldw;
  const cplx* b = c.Ws + (long long)cj * c.ldw;
  cplx acc = mk(0.0, 0.0);
  int l = l0;
  constexpr int RB = 8;
  for (; l + 32 * (RB - 1) < nl; l += 32 * RB) {
    cplx x[RB], y[RB];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      x[u] = a[l + 32 * u];
      y[u] = b[l + 32 * u];
    }
#pragma unroll
    for (int u = 0; u < RB; ++u) acc = cfmac(x[u], y[u], acc);
  }
  for (; l < nl; l += 32) acc = cfmac(a[l], b[l], acc);
  return acc;
}

// col_dotc for n <= G columns cols[0..n) against column ci, reading column
// ci once for all of them (same per-lane accumulation order as col_dotc)
template <int G>
__device__ __forceinline__ void col_dotc_group(const CC& c, int ci, const int* cols, int n, int l0, int nl,
                                               cplx* acc) {
  const cplx* a = c.Ws + (long long)ci * c.ldw;
  const cplx* b[G];
#pragma unroll
  for (int k = 0; k < G; ++k) {
    b[k] = c.Ws + (long long)cols[min(k, n - 1)] * c.ldw;
    acc[k] = mk(0.0, 0.0);
  }
  int l = l0;
#ifndef PART_LOADS
#define PART_LOADS 18
#endif
  constexpr int RB = (PART_LOADS / (G + 1)) > 1 ? PART_LOADS / (G + 1) : 1;  // ~PART_LOADS loads in flight
  for (; l + 32 * (RB - 1) < nl; l += 32 * RB) {
    cplx x[RB], y[RB][G];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      x[u] = a[l + 32 * u];
#pragma unroll
      for (int k = 0; k < G; ++k) y[u][k] = b[k][l + 32 * u];
    }
#pragma unroll
    for (int u = 0; u < RB; ++u)
#pragma unroll
      for (int k = 0; k < G; ++k) acc[k] = cfmac(x[u], y[u][k], acc[k]);
  }
  for (; l < nl; l += 32) {
    const cplx x = a[l];
#pragma unroll
    for (int k = 0; k < G; ++k) acc[k] = cfmac(x, b[k][l], acc[k]);
  }
}

// big: (global-slice mode, blocks whose normal carve exceeds shared memory,
// e.g. r = 64) the per-row arrays vn1/vn2/rpos/rpos2 and B[sel,:] live in
// global memory (the instance's dwork/iwork and B buffers) instead.
__host__ __device__ size_t carve(unsigned char* base, int ldw, int r, CC* c, bool global_slice = false,
                                 int big = 0) {
  const bool grows = (big & 1) != 0, gselb = (big & 2) != 0;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* p = base ? base + off : nullptr;
    off += (bytes + 15) & ~(size_t)15;
    return p;
  };
  CC t;
  t.Ws = global_slice ? nullptr : (cplx*)take(sizeof(cplx) * (size_t)ldw * r);
  t.aug = (cplx*)take(sizeof(cplx) * 2 * r * r);
  t.selb = gselb ? nullptr : (cplx*)take(sizeof(cplx) * r * r);
  t.vec = (cplx*)take(sizeof(cplx) * r);
  t.vec2 = (cplx*)take(sizeof(cplx) * 5 * r);  // also Gauss-Jordan scratch
  t.tau = (cplx*)take(sizeof(cplx) * r);
  t.betas = (double*)take(sizeof(double) * r);
  t.cn1 = (double*)take(sizeof(double) * r);
  t.cn2 = (double*)take(sizeof(double) * r);
  t.colmap = (int*)take(sizeof(int) * r);
  t.flags = (int*)take(sizeof(int) * r);
  t.first = (int*)take(sizeof(int) * r);
  t.sel = (int*)take(sizeof(int) * r);
  t.best = (int*)take(sizeof(int) * r);
  t.starts = (int*)take(sizeof(int) * 2 * r);
  // The starts' per-row state (vn1, vn2, rpos, rpos2) and the staged Q row
  // tile of the DMMA Q*X products (form_B / the factor, global-slice mode,
  // r <= 32) are never live together: they share one region, which keeps
  // the carve (and so the L1 the row passes lose to shared memory) small.
  {
    const size_t a8 = (sizeof(double) * (size_t)ldw + 15) & ~(size_t)15;
    const size_t a4 = (sizeof(int) * (size_t)ldw + 15) & ~(size_t)15;
    const size_t rows_bytes = grows ? 0 : 2 * a8 + 2 * a4;
    const size_t qt_bytes = (global_slice && r <= 32)
                                ? 2 * sizeof(double) * QX_ROWS * (size_t)(((2 * r + 3) & ~3) + 4) : 0;
    unsigned char* u = (unsigned char*)take(rows_bytes > qt_bytes ? rows_bytes : qt_bytes);
    t.vn1 = grows ? nullptr : (double*)u;
    t.vn2 = grows ? nullptr : (double*)(u ? u + a8 : nullptr);
    t.rpos = grows ? nullptr : (int*)(u ? u + 2 * a8 : nullptr);
    t.rpos2 = grows ? nullptr : (int*)(u ? u + 2 * a8 + a4 : nullptr);
    t.qtile = qt_bytes ? (double*)u : nullptr;
  }
  t.rec = (Rec*)take(sizeof(Rec) * 2);
  t.wrec = (WCand*)take(sizeof(WCand) * 2 * CW);
  t.wrec2 = (WCand*)take(sizeof(WCand) * 2 * CW);
  t.sp = (cplx*)take(sizeof(cplx) * 8 * r);
  t.wrow = (cplx*)take(sizeof(cplx) * 2 * CW * r);
  t.wcand = (Cand*)take(sizeof(Cand) * CW);
  t.wss = (Ssq*)take(sizeof(Ssq) * CW);
  t.ibc = (int*)take(sizeof(int) * 16);
  t.dbc = (double*)take(sizeof(double) * 8);
  t.cbc = (cplx*)take(sizeof(cplx) * 8);
  t.pend = global_slice ? (cplx*)take(sizeof(cplx) * LAZY_MAX * r) : nullptr;
  t.pendj = global_slice ? (int*)take(sizeof(int) * LAZY_MAX) : nullptr;
  if (c) {
    c->Ws = t.Ws; c->aug = t.aug; c->selb = t.selb; c->vec = t.vec; c->vec2 = t.vec2;
    c->tau = t.tau; c->betas = t.betas; c->cn1 = t.cn1; c->cn2 = t.cn2; c->colmap = t.colmap;
    c->flags = t.flags; c->first = t.first; c->sel = t.sel; c->best = t.best; c->starts = t.starts;
    c->vn1 = t.vn1; c->vn2 = t.vn2; c->rpos = t.rpos; c->rec = t.rec; c->wcand = t.wcand;
    c->wrec = t.wrec; c->wrow = t.wrow;
    c->wrec2 = t.wrec2; c->rpos2 = t.rpos2; c->sp = t.sp; c->qtile = t.qtile;
    c->wss = t.wss; c->ibc = t.ibc; c->dbc = t.dbc; c->cbc = t.cbc;
    c->pend = t.pend; c->pendj = t.pendj;
  }
  return off;
}

// Block-wide best candidate; every thread returns the same value.
__device__ Cand block_cand(Cand a, Cand* red) {
  a = warp_cand(a);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  Cand b = red[0];
  for (int w = 1; w < CW; ++w)
    if (cand_better(red[w], b)) b = red[w];
  return b;
}

// Winning candidate across the cluster from the records of this parity;
// returns it in every thread (rank in .pad via ibc[3]).
__device__ Cand cluster_winner(cg::cluster_group& cl, const CC& c, int par, int* wrank) {
  if (threadIdx.x < 32) {
    Cand a{-1.0, LLONG_MAX, -1};
    int rk = 0;
    if ((int)threadIdx.x < c.C) {
      const Rec* rr = cl.map_shared_rank(&c.rec[par], (int)threadIdx.x);
      a.v = rr->v;
      a.key = rr->key;
      a.row = rr->row;
      rk = threadIdx.x;
    }
    // carry the rank in the low bits of a lane-local variable via shuffle of (v,key,row,rank)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Cand b;
      b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
      b.key = __shfl_xor_sync(0xffffffffu, a.key, o);
      b.row = __shfl_xor_sync(0xffffffffu, a.row, o);
      const int brk = __shfl_xor_sync(0xffffffffu, rk, o);
      if (cand_better(b, a)) {
        a = b;
        rk = brk;
      }
    }
    if (threadIdx.x == 0) {
      c.wcand[0] = a;
      c.ibc[3] = rk;
    }
  }
  __syncthreads();
  *wrank = c.ibc[3];
  return c.wcand[0];
}

// Cross-rank reductions of one record slot, done by a whole warp: lane k
// reads rank k's value over DSMEM (all C loads in flight at once) and a
// fixed xor tree combines them, so every CTA obtains the same bits.
__device__ __forceinline__ cplx rank_sum(cg::cluster_group& cl, const CC& c, int par, int idx) {
  const int lane = threadIdx.x & 31;
  cplx v = mk(0.0, 0.0);
  if (lane < c.C) v = cl.map_shared_rank(&c.rec[par], lane)->data[idx];
  return warp_sum(v);
}

__device__ __forceinline__ Ssq rank_ssq(cg::cluster_group& cl, const CC& c, int par, int idx) {
  const int lane = threadIdx.x & 31;
  Ssq s = ssq_init();
  if (lane < c.C) {
    const cplx v = cl.map_shared_rank(&c.rec[par], lane)->data[idx];
    s = Ssq{v.x, v.y};
  }
  return warp_ssq(s);
}

__device__ void set_error(const BondJob& job, int inst, int code) {
  job.status[inst] = code;
  if (job.err_bond) job.err_bond[inst] = job.bond;
}

__device__ void insertion_sort(int* v, int r) {
  for (int p = 1; p < r; ++p) {
    const int x = v[p];
    int q = p - 1;
    while (q >= 0 && v[q] > x) {
      v[q + 1] = v[q];
      --q;
    }
    v[q + 1] = x;
  }
}

// ------------------------------------------------------------ phase 0
__device__ void load_block(const CC& c, const ClusterJob& J, int inst) {
  const int r = c.r;
  const long long tot = (long long)c.nrows * r;
  if (J.src_mode == 0 && J.fiber_fast && fiber_fast_ok(J.oracle) && r >= 9) {
    // separable evaluation (fiber_fast.cuh): column parts once per column in
    // shared memory (aug is free here), row parts once per row in registers
    const FiberJob& f = J.fiber;
    const OracleDev& o = J.oracle;
    const int d = o.d;
    const double* p = o.params + inst * o.param_stride;
    const FiberSplit fs = fiber_split(f.mode, f.kl, d);
    const bool phi = o.kind == TTP_ORACLE_PHI_GBM;
    cplx* colbuf = c.aug;  // per column: PHI 1 + FF_MAXI values, VHAT 2 values
    const int cstride = phi ? 1 + FF_MAXI : 2;
    int idx[TTP_MAX_D];
    for (int t = threadIdx.x; t < r; t += CT) {
      const int* T = (f.mode == 0)
                         ? f.right.base + inst * f.right.set_stride + f.right.offset + (long long)t * f.right.d
                         : f.left.base + inst * f.left.set_stride + f.left.offset + (long long)t * f.left.d;
      const int shift = (f.mode == 0) ? f.kl + 1 : 0;
      for (int j = fs.col_lo; j < fs.col_hi; ++j) idx[j] = T[j - shift];
      cplx* cb = colbuf + t * cstride;
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
    for (int l = threadIdx.x; l < c.nrows; l += CT) {
      const int g = c.row0 + l;
      if (f.mode == 0) {
        const int a = g / f.na, s = g - a * f.na;
        const int* L = f.left.base + inst * f.left.set_stride + f.left.offset + (long long)a * f.left.d;
        for (int j = 0; j < f.kl; ++j) idx[j] = L[j];
        idx[f.kl] = s;
      } else {
        const int s = g / f.rr, b = g - s * f.rr;
        const int* R = f.right.base + inst * f.right.set_stride + f.right.offset + (long long)b * f.right.d;
        idx[f.kl] = s;
        for (int j = f.kl + 1; j < d; ++j) idx[j] = R[j - f.kl - 1];
      }
      if (phi) {
        PhiPart rp;
        phi_part(p, d, idx, fs.row_lo, fs.row_hi, !fs.inner_is_col, fs.col_lo, fs.col_hi, rp);
        for (int t = 0; t < r; ++t) Wl(c, l, t) = phi_combine_packed(rp, colbuf + t * cstride, fs.ninner);
      } else {
        cplx prow, wrow;
        vhat_part(p, idx, fs.row_lo, fs.row_hi, prow, wrow);
        for (int t = 0; t < r; ++t) {
          const cplx* cb = colbuf + t * cstride;
          Wl(c, l, t) = vhat_combine(p, d, prow, wrow, cb[0], cb[1]);
        }
      }
    }
  } else if (J.src_mode == 0) {
    const FiberJob& f = J.fiber;
    int idx[TTP_MAX_D];
    for (long long e = threadIdx.x; e < tot; e += CT) {
      const int t = (int)(e / c.nrows), l = (int)(e - (long long)t * c.nrows);
      const int g = c.row0 + l;
      int a, s, b;
      if (f.mode == 0) {
        a = g / f.na;
        s = g - a * f.na;
        b = t;
      } else {
        s = g / f.rr;
        b = g - s * f.rr;
        a = t;
      }
      const int* L = f.left.base + inst * f.left.set_stride + f.left.offset + (long long)a * f.left.d;
      const int* R = f.right.base + inst * f.right.set_stride + f.right.offset + (long long)b * f.right.d;
      for (int j = 0; j < f.kl; ++j) idx[j] = L[j];
      idx[f.kl] = s;
      for (int j = f.kl + 1; j < J.oracle.d; ++j) idx[j] = R[j - f.kl - 1];
      Wl(c, l, t) = oracle_value(J.oracle, inst, idx);
    }
  } else {
    const cplx* src = J.src + inst * J.src_stride;
    for (long long e = threadIdx.x; e < tot; e += CT) {
      const int t = (int)(e / c.nrows), l = (int)(e - (long long)t * c.nrows);
      Wl(c, l, t) = src[(long long)(c.row0 + l) * r + t];  // numpy row-major
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ phase A'
// Q = H(0)...H(r-1) [I; 0] in compact-WY form (the representation zungqr's
// blocked path uses, LAPACK zlarft + zlarfb):  Q = E - V (T V1^H) with
// V the unit lower-trapezoidal reflector block, V1 its top r x r block and
// T upper triangular from the Gram matrix V^H V.  Two cluster barriers
// instead of zung2r's r rounds, and each row slice is read ~r/4 times
// instead of ~2r.  Same Q up to rounding (both are backward stable).
//
// V(g, a) = 1 (g == a), W(g, colmap[a]) (g > a), 0 (g < a).
__device__ __forceinline__ cplx vref(const CC& c, int l, int g, int a) {
  return g > a ? Wl(c, l, c.colmap[a]) : mk(g == a ? 1.0 : 0.0, 0.0);
}

// Gram partials X[a r + b] = sum_{local rows g >= r} conj(V(g,a)) V(g,b),
// a < b, on the FP64 tensor cores (r <= 32, qtile present): the rows stream
// through the Q*X staging tiles by cp.async (double-buffered, V columns in
// logical order, real interleaved) and the real Gram of the interleaved
// rows accumulates in DMMA fragments (each warp owns upper-triangle 8x8
// tiles); the complex entries follow from its 2x2 blocks.  Every V element
// is read from global memory once.
__device__ void gram_dmma(const CC& c, cplx* X) {
  const int r = c.r, nl = c.nrows, lo = c.row0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int Kp = (2 * r + 3) & ~3, ldA = Kp + 4;
  const int nt8 = (2 * r + 7) / 8;              // real 8-wide tiles per side
  const int ntiles = nt8 * (nt8 + 1) / 2;       // upper triangle incl. diagonal
  constexpr int MAXT = 8;                       // tiles per warp (36 / CW)
  double acc[MAXT][2];
#pragma unroll
  for (int q = 0; q < MAXT; ++q) acc[q][0] = acc[q][1] = 0.0;
  double* tiles[2] = {c.qtile, c.qtile + QX_ROWS * ldA};
  __syncthreads();  // the region is shared with the starts' per-row state
  for (int e = threadIdx.x; e < 2 * QX_ROWS * (Kp - 2 * r); e += CT) {
    const int bb = e / (QX_ROWS * (Kp - 2 * r)), e2 = e - bb * QX_ROWS * (Kp - 2 * r);
    const int row = e2 / (Kp - 2 * r), k = 2 * r + (e2 - row * (Kp - 2 * r));
    tiles[bb][row * ldA + k] = 0.0;
  }
  const int lfast = max(0, r - lo);  // rows below hold the unit-diagonal part of V
  // rows past nl are zero-filled by cp.async with a 0-byte source
  auto issue = [&](int l0, double* dst) {
    for (int e = threadIdx.x; e < QX_ROWS * r; e += CT) {
      const int t = e / QX_ROWS, row = e - t * QX_ROWS;
      const int l = l0 + row;
      const cplx* src = c.Ws + (long long)c.colmap[t] * c.ldw + min(l, nl - 1);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + row * ldA + 2 * t);
      const int bytes = (l < nl) ? 16 : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(bytes));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  if (lfast < nl) issue(lfast, tiles[0]);
  int buf = 0;
  for (int l0 = lfast; l0 < nl; l0 += QX_ROWS, buf ^= 1) {
    if (l0 + QX_ROWS < nl) {
      issue(l0 + QX_ROWS, tiles[buf ^ 1]);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* tile = tiles[buf];
#pragma unroll
    for (int q = 0; q < MAXT; ++q) {
      const int tt = warp + q * CW;
      if (tt < ntiles) {
        int ti = 0, rem = tt;
        while (rem >= nt8 - ti) {
          rem -= nt8 - ti;
          ++ti;
        }
        const int tj = ti + rem;
        // A(m, k) = tile[k][ti*8 + m], B(k, n) = tile[k][tj*8 + n]
#pragma unroll
        for (int k0 = 0; k0 < QX_ROWS; k0 += 4) {
          const double av = tile[(k0 + tig) * ldA + ti * 8 + gid];
          const double bv = tile[(k0 + tig) * ldA + tj * 8 + gid];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[q][0]), "+d"(acc[q][1]) : "d"(av), "d"(bv));
        }
      }
    }
    __syncthreads();  // tile buf is refilled by the issue two steps later
  }
  // complex entries from the real 2x2 blocks: lane (gid = 2p, tig) holds
  // R(2a, 2b), R(2a, 2b+1); its partner gid = 2p + 1 (lane ^ 4) holds
  // R(2a+1, 2b), R(2a+1, 2b+1), with a = 4 ti + p, b = 4 tj + tig
#pragma unroll
  for (int q = 0; q < MAXT; ++q) {
    const int tt = warp + q * CW;
    if (tt < ntiles) {
      int ti = 0, rem = tt;
      while (rem >= nt8 - ti) {
        rem -= nt8 - ti;
        ++ti;
      }
      const int tj = ti + rem;
      const double o0 = __shfl_xor_sync(0xffffffffu, acc[q][0], 4);
      const double o1 = __shfl_xor_sync(0xffffffffu, acc[q][1], 4);
      if ((gid & 1) == 0) {
        const int a = 4 * ti + (gid >> 1), b = 4 * tj + tig;
        if (a < b && b < r) X[a * r + b] = mk(acc[q][0] + o1, acc[q][1] - o0);
      }
    }
  }
  // the unit-diagonal rows (g < r, CTA 0 only): V(g,a) = 1 (g == a), W (g > a), 0
  if (lfast > 0) {
    __syncthreads();
    for (int e = threadIdx.x; e < r * r; e += CT) {
      const int a = e / r, b = e - a * r;
      if (a < b) {
        cplx s = X[e];
        for (int l = 0; l < min(lfast, nl); ++l) s = cfmac(vref(c, l, lo + l, a), vref(c, l, lo + l, b), s);
        X[e] = s;
      }
    }
  }
}

// norms: also leave each Q row's squared norm and the starts' initial row
// positions in vn1/vn2/rpos/rpos2 (the fused starts then skip their norm pass)
__device__ void form_q_wy(cg::cluster_group& cl, CC& c, bool norms) {
  const int r = c.r, m = c.m, lo = c.row0, nl = c.nrows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  cplx* X = c.aug;          // this CTA's packed partials (read remotely)
  cplx* P = c.aug + r * r;  // reduced: strict upper = V^H V, strict lower = V1
  cplx* T = c.selb;         // r x r row-major, upper triangular
  SP_BEGIN(spw);
  // (1) Gram partials over local rows: on DMMA when the staging tile exists
  //     (r <= 32), else 4 x 4 tiles (upper tile triangle), lanes stride rows
  //     (coalesced column reads), one warp per tile.
  if (c.qtile && g_gram_dmma) {
    gram_dmma(c, X);
  } else {
  constexpr int TB = 4;
  const int nt = (r + TB - 1) / TB;
  const int ntiles = nt * (nt + 1) / 2;
  for (int tile = warp; tile < ntiles; tile += CW) {
    int ta = 0, rem = tile;
    while (rem >= nt - ta) {
      rem -= nt - ta;
      ++ta;
    }
    const int tb = ta + rem;
    const int a0 = ta * TB, b0 = tb * TB;
    int ca[TB], cb[TB];
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      ca[u] = c.colmap[min(a0 + u, r - 1)];
      cb[u] = c.colmap[min(b0 + u, r - 1)];
    }
    cplx acc[TB][TB];
#pragma unroll
    for (int u = 0; u < TB; ++u)
#pragma unroll
      for (int v = 0; v < TB; ++v) acc[u][v] = mk(0.0, 0.0);
    // rows with g >= r hold plain W values in every column
    const int lfast = max(0, r - lo);
    for (int l = lfast + lane; l < nl; l += 32) {
      cplx xa[TB], xb[TB];
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        xa[u] = Wl(c, l, ca[u]);
        xb[u] = Wl(c, l, cb[u]);
      }
#pragma unroll
      for (int u = 0; u < TB; ++u)
#pragma unroll
        for (int v = 0; v < TB; ++v) acc[u][v] = cfmac(xa[u], xb[v], acc[u][v]);
    }
    for (int l = lane; l < min(lfast, nl); l += 32) {
      const int g = lo + l;
#pragma unroll
      for (int u = 0; u < TB; ++u)
#pragma unroll
        for (int v = 0; v < TB; ++v)
          if (a0 + u < r && b0 + v < r)
            acc[u][v] = cfmac(vref(c, l, g, a0 + u), vref(c, l, g, b0 + v), acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < TB; ++u)
#pragma unroll
      for (int v = 0; v < TB; ++v) {
        const cplx s = warp_sum(acc[u][v]);
        const int a = a0 + u, b = b0 + v;
        if (lane == 0 && a < b && b < r) X[a * r + b] = s;
      }
  }
  }
  // strict lower: V1(a, b), a > b, from the CTA owning row a (0 elsewhere)
  for (int e = threadIdx.x; e < r * r; e += CT) {
    const int a = e / r, b = e - a * r;
    if (a > b) X[e] = (a >= lo && a < lo + nl) ? Wl(c, a - lo, c.colmap[b]) : mk(0.0, 0.0);
  }
  cl.sync();
  SP(spw, 5);
  // (2) fixed rank order sum, identical in every CTA
  for (int e = threadIdx.x; e < r * r; e += CT) {
    const int a = e / r, b = e - a * r;
    if (a == b) continue;
    cplx s = mk(0.0, 0.0);
    for (int k = 0; k < c.C; ++k) s = cadd(s, cl.map_shared_rank(X, k)[e]);
    P[e] = s;
  }
  __syncthreads();
  SP(spw, 6);
  // (3) zlarft (forward, columnwise): T(i,i) = tau_i,
  //     T(0:i, i) = -tau_i T(0:i, 0:i) G(0:i, i).  Lane owns rows of T.
  if (warp == 0) {
    for (int i = 0; i < r; ++i) {
      const cplx ti = c.tau[i];
      for (int a = lane; a < r; a += 32) {
        cplx v = mk(0.0, 0.0);
        if (a < i) {
          for (int b = a; b < i; ++b) v = cfma(T[a * r + b], P[b * r + i], v);
          v = cneg(cmul(ti, v));
        } else if (a == i) {
          v = ti;
        }
        T[a * r + i] = v;
      }
      __syncwarp();
    }
  }
  cl.sync();  // every CTA finished reading the remote partials in X
  SP(spw, 14);
  // (4) M = T V1^H (upper triangular) into X
  cplx* M = X;
  for (int e = threadIdx.x; e < r * r; e += CT) {
    const int a = e / r, b = e - a * r;
    cplx s = mk(0.0, 0.0);
    if (a <= b) {
      // V1(b, cc): 1 at cc == b, P[b*r+cc] for cc < b
      for (int cc = a; cc < b; ++cc) s = cfmac(P[b * r + cc], T[a * r + cc], s);
      s = cadd(s, T[a * r + b]);
    }
    M[e] = s;
  }
  __syncthreads();
  SP(spw, 15);
  // (5) Q(g, b) = delta(g, b) - sum_{a <= b} V(g, a) M(a, b), written to Qg
  //     in logical column order; outputs in blocks of 8 per row thread.
  constexpr int OB = 8;
  FOR_MY_ROWS(l, nl, g_serpentine) {  // the Gram pass ran ascending
    const int g = lo + l;
    double nsq = 0.0, nmx = 0.0;  // sum of squares in column order, largest component
    for (int b0 = 0; b0 < r; b0 += OB) {
      cplx acc[OB];
#pragma unroll
      for (int q = 0; q < OB; ++q) acc[q] = mk(0.0, 0.0);
      const int amax = min(r, b0 + OB);
      if (g >= r) {
#ifndef QF_LOADS
#define QF_LOADS 4
#endif
        constexpr int QL = QF_LOADS;  // V loads in flight per row
        int a = 0;
        for (; a + QL <= amax; a += QL) {
          cplx x[QL];
#pragma unroll
          for (int u = 0; u < QL; ++u) x[u] = Wl(c, l, c.colmap[a + u]);
#pragma unroll
          for (int u = 0; u < QL; ++u)
#pragma unroll
            for (int q = 0; q < OB; ++q)
              if (b0 + q < r) acc[q] = cfma(x[u], M[(a + u) * r + b0 + q], acc[q]);
        }
        for (; a < amax; ++a) {
          const cplx x = Wl(c, l, c.colmap[a]);
#pragma unroll
          for (int q = 0; q < OB; ++q)
            if (b0 + q < r) acc[q] = cfma(x, M[a * r + b0 + q], acc[q]);
        }
      } else {
        for (int a = 0; a < amax; ++a) {
          const cplx x = vref(c, l, g, a);
#pragma unroll
          for (int q = 0; q < OB; ++q)
            if (b0 + q < r) acc[q] = cfma(x, M[a * r + b0 + q], acc[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < OB; ++q)
        if (b0 + q < r) {
          const cplx qv = csub(mk(g == b0 + q ? 1.0 : 0.0, 0.0), acc[q]);
          c.Qg[(long long)(b0 + q) * m + g] = qv;
          nsq = fma(qv.x, qv.x, fma(qv.y, qv.y, nsq));
          nmx = fmax(nmx, fmax(fabs(qv.x), fabs(qv.y)));
        }
    }
    if (norms) {
      // plain sum of squares where no scaling is needed; else the scaled
      // two-pass form over the row just written
      double n2 = nsq;
      if (!(nmx == 0.0 || (nmx > 1e-140 && nmx < 1e140))) {
        __threadfence_block();
        n2 = ssq_norm2(ssq_of(Qrow(c, g), m, r));
      }
      c.vn1[l] = n2;
      c.vn2[l] = n2;
      c.rpos[l] = g;
      c.rpos2[l] = g;
    }
  }
  __threadfence();
  __syncthreads();
}

// ------------------------------------------------------------ phase A
// Distributed zlaqp2 + zung2r on the block.  Returns false (cluster-uniform)
// when the block is zero / rank deficient by rank_tol.
// conj(y_p) y_t products of 8 columns (v[0..8)) summed over the warp's 32
// lanes by a transposed butterfly: afterwards lane L holds the sum for
// column (L >> 2) & 7 (fixed order, 18 shuffles)
__device__ __forceinline__ cplx warp_transpose_sum8(const cplx* v) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  cplx k4[4], k2[2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const cplx send = b4 ? v[j] : v[j + 4];
    cplx got;
    got.x = __shfl_xor_sync(0xffffffffu, send.x, 16);
    got.y = __shfl_xor_sync(0xffffffffu, send.y, 16);
    k4[j] = cadd(b4 ? v[j + 4] : v[j], got);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const cplx send = b3 ? k4[j] : k4[j + 2];
    cplx got;
    got.x = __shfl_xor_sync(0xffffffffu, send.x, 8);
    got.y = __shfl_xor_sync(0xffffffffu, send.y, 8);
    k2[j] = cadd(b3 ? k4[j + 2] : k4[j], got);
  }
  cplx k1;
  {
    const cplx send = b2 ? k2[0] : k2[1];
    cplx got;
    got.x = __shfl_xor_sync(0xffffffffu, send.x, 4);
    got.y = __shfl_xor_sync(0xffffffffu, send.y, 4);
    k1 = cadd(b2 ? k2[1] : k2[0], got);
  }
#pragma unroll
  for (int o = 2; o > 0; o >>= 1) {
    cplx got;
    got.x = __shfl_xor_sync(0xffffffffu, k1.x, o);
    got.y = __shfl_xor_sync(0xffffffffu, k1.y, o);
    k1 = cadd(k1, got);
  }
  return k1;
}

// 16-column version: lane L ends with the sum for column (L >> 1) & 15
__device__ __forceinline__ cplx warp_transpose_sum16(const cplx* v) {
  const int lane = threadIdx.x & 31;
  cplx k8[8], k4[4], k2[2];
  auto xch = [](cplx send, int o) {
    cplx got;
    got.x = __shfl_xor_sync(0xffffffffu, send.x, o);
    got.y = __shfl_xor_sync(0xffffffffu, send.y, o);
    return got;
  };
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int j = 0; j < 8; ++j) k8[j] = cadd(b4 ? v[j + 8] : v[j], xch(b4 ? v[j] : v[j + 8], 16));
#pragma unroll
  for (int j = 0; j < 4; ++j) k4[j] = cadd(b3 ? k8[j + 4] : k8[j], xch(b3 ? k8[j] : k8[j + 4], 8));
#pragma unroll
  for (int j = 0; j < 2; ++j) k2[j] = cadd(b2 ? k4[j + 2] : k4[j], xch(b2 ? k4[j] : k4[j + 2], 4));
  cplx k1 = cadd(b1 ? k2[1] : k2[0], xch(b1 ? k2[0] : k2[1], 2));
  return cadd(k1, xch(k1, 1));
}

__device__ bool column_basis(cg::cluster_group& cl, CC& c, int& par, double rank_tol, bool wy, bool fuse_qr,
                             bool norms_in_q) {
  const int r = c.r, m = c.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lo = c.row0, nl = c.nrows;
  // initial column norms
  {
    Rec* me = &c.rec[par];
    for (int j = warp; j < r; j += CW) {
      Ssq s = ssq_of(&c.Ws[(long long)j * c.ldw + lane], 32, nl > lane ? (nl - lane + 31) / 32 : 0);
      s = warp_ssq(s);
      if (lane == 0) me->data[j] = mk(s.scale, s.ssq);
    }
    cl.sync();
    // cn1/cn2 hold SQUARED partial column norms: the zlaqp2 downdate
    // becomes s1' = max(0, s1 - |a|^2), recompute iff s1' <= tol3z * s2
    // (division free; the idamax choice is order preserving).
    for (int j = warp; j < r; j += CW) {
      const double n2 = ssq_norm2(rank_ssq(cl, c, par, j));
      if (lane == 0) {
        c.cn1[j] = n2;
        c.cn2[j] = n2;
        c.colmap[j] = j;
      }
    }
    par ^= 1;
    __syncthreads();
  }
  SP_BEGIN(spt);
  bool fused = false;  // this step's pivot and partials came out of the previous update pass
  for (int i = 0; i < r; ++i) {
    if (!fused) {
    if (warp == 0) {
      ArgMax am{-1.0, LLONG_MAX};
      for (int j = i + lane; j < r; j += 32)
        if (argmax_better(c.cn1[j], j, am.v, am.key)) am = ArgMax{c.cn1[j], j};
      am = warp_argmax(am);  // idamax: first maximum
      const int p = (int)am.key;
      if (lane == 0 && p != i) {
        const int t = c.colmap[p];
        c.colmap[p] = c.colmap[i];
        c.colmap[i] = t;
        c.cn1[p] = c.cn1[i];
        c.cn2[p] = c.cn2[i];
      }
    }
    __syncthreads();
    }
    SP(spt, 0);
    const int ci = c.colmap[i];
    const bool own_i = (i >= lo && i < lo + nl);
    const int li = i - lo;
    const int lstart = max(0, i + 1 - lo);  // first local row with global index > i
    const int ntr = r - i - 1;
    Rec* me = &c.rec[par];
    if (!fused) {
    // partials: item 0 = Ssq of x, item g >= 1 = conj(x) . columns i+q for
    // the PG tasks q of group g (column x read once per group; PG sized so
    // that every item gets its own warp)
    const int PG = min(8, max(1, (ntr + CW - 2) / (CW - 1)));
    const int ngrp = (ntr + PG - 1) / PG;
    for (int it = warp; it <= ngrp; it += CW) {
      if (it == 0) {
        const int f0 = lstart + lane;
        Ssq s = ssq_of(&c.Ws[(long long)ci * c.ldw + f0], 32, nl > f0 ? (nl - f0 + 31) / 32 : 0);
        s = warp_ssq(s);
        if (lane == 0) {
          me->data[0] = mk(s.scale, s.ssq);
          me->data[1] = own_i ? Wl(c, li, ci) : mk(0.0, 0.0);
        }
      } else {
        const int q0 = 1 + (it - 1) * PG;
        const int n = min(PG, ntr - q0 + 1);
        cplx acc[8];
        const int* cols = c.colmap + i + q0;
        switch (PG) {
          case 1: col_dotc_group<1>(c, ci, cols, n, lstart + lane, nl, acc); break;
          case 2: col_dotc_group<2>(c, ci, cols, n, lstart + lane, nl, acc); break;
          case 3: col_dotc_group<3>(c, ci, cols, n, lstart + lane, nl, acc); break;
          case 4: col_dotc_group<4>(c, ci, cols, n, lstart + lane, nl, acc); break;
          case 5: col_dotc_group<5>(c, ci, cols, n, lstart + lane, nl, acc); break;
          default: col_dotc_group<8>(c, ci, cols, n, lstart + lane, nl, acc); break;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k < n) {
            const cplx sum = warp_sum(acc[k]);
            if (lane == 0) {
              me->data[q0 + k + 1] = sum;
              me->data[1 + r + q0 + k] = own_i ? Wl(c, li, c.colmap[i + q0 + k]) : mk(0.0, 0.0);
            }
          }
        }
      }
    }
    }
    SP(spt, 1);
    cl.sync();
    SP(spt, 2);
    // Every warp derives the reflector itself (lanes = cluster ranks, fixed
    // merge order, identical bits everywhere), then finishes its own items:
    // no block barrier between the cluster barrier and the update.
    const Ssq sx = rank_ssq(cl, c, par, 0);
    const cplx alpha = rank_sum(cl, c, par, 1);
    const Reflector h = (sx.scale > 1e-140 && sx.scale < 1e140) ? zlarfg_fast(alpha, ssq_norm2(sx))
                                                                  : zlarfg_core(alpha, ssq_norm(sx));
    const cplx tau = h.tau;
    const bool ident = is_zero(tau);
    const cplx scal = reflector_scale(h);
    if (threadIdx.x == 0) {
      c.tau[i] = h.tau;
      c.betas[i] = fabs(h.beta);
      c.cbc[0] = scal;
    }
    for (int q = 1 + warp; q <= ntr; q += CW) {
      const cplx dots = rank_sum(cl, c, par, 1 + q);
      const cplx arow = rank_sum(cl, c, par, 1 + r + q);
      if (lane == 0) {
        // v = [1; x*scal]:  s_j = A[i,j] + conj(scal) * (x^H A[:,j])
        const cplx sj = cadd(arow, cmulc(scal, dots));
        const cplx tj = ident ? mk(0.0, 0.0) : cmul(cconj(tau), sj);
        c.vec[q - 1] = tj;
        const cplx newrow = csub(arow, tj);
        c.vec2[q - 1] = newrow;
        // zlaqp2 partial column-norm downdate on squared norms (replicated)
        const int j = i + q;
        int flag = 0;
        const double s1 = c.cn1[j];
        if (s1 != 0.0) {
          const double s1n = fmax(s1 - cabs2(newrow), 0.0);
          if (s1n <= TOL3Z * c.cn2[j]) flag = 1;
          else c.cn1[j] = s1n;
        }
        c.flags[q - 1] = flag;
      }
    }
    par ^= 1;
    __syncthreads();
    SP(spt, 3);
    int anyflag = 0;
    for (int q = 0; q < ntr; ++q) anyflag |= c.flags[q];
    // Fused: when no norm recompute is pending the next pivot is already
    // known, so this step's update pass also produces the next step's
    // partials (the reflector's dot products and norm, the pivot row) and
    // the separate partials pass disappears.
    fused = fuse_qr && !anyflag && ntr >= 1 && ntr <= 32 && !ident;
    if (fused) {
      // pivot of step i+1 (idamax over the downdated norms), swapped into
      // position i+1 together with its update coefficients
      if (warp == 0) {
        ArgMax am{-1.0, LLONG_MAX};
        for (int j = i + 1 + lane; j < r; j += 32)
          if (argmax_better(c.cn1[j], j, am.v, am.key)) am = ArgMax{c.cn1[j], j};
        am = warp_argmax(am);
        const int p = (int)am.key;
        if (lane == 0 && p != i + 1) {
          const int t = c.colmap[p];
          c.colmap[p] = c.colmap[i + 1];
          c.colmap[i + 1] = t;
          c.cn1[p] = c.cn1[i + 1];
          c.cn2[p] = c.cn2[i + 1];
          const int qa = 0, qb = p - i - 1;
          const cplx va = c.vec[qa], wa = c.vec2[qa];
          c.vec[qa] = c.vec[qb];
          c.vec2[qa] = c.vec2[qb];
          c.vec[qb] = va;
          c.vec2[qb] = wa;
        }
      }
      __syncthreads();
      const int* cols = c.colmap + i + 1;  // cols[0]: pivot of step i+1
#ifndef FQ_CH
#define FQ_CH 8
#endif
      constexpr int FQ = FQ_CH;        // trailing entries per chunk (loads in flight)
      constexpr int NCH = 32 / FQ;
      const int nch = (ntr + FQ - 1) / FQ;  // <= NCH
      const int ldw = c.ldw;
      Rec* nx = &c.rec[par];  // step i+1's record
      cplx acc[NCH];
#pragma unroll
      for (int u = 0; u < NCH; ++u) acc[u] = mk(0.0, 0.0);
      double s2 = 0.0, mx = 0.0;
      const int nk = (nl + CT - 1) / CT;
      const bool rev = g_serpentine && (i & 1) == 0;
      for (int k = 0; k < nk; ++k) {
        const int l = threadIdx.x + (rev ? nk - 1 - k : k) * CT;
        const bool act = l < nl;
        const int g = lo + l;
        cplx* prow = c.Ws + (act ? l : 0);
        if (act && g == i) {
          prow[ci * ldw] = mk(h.beta, 0.0);
          for (int q = 1; q <= ntr; ++q) prow[cols[q - 1] * ldw] = c.vec2[q - 1];
        }
        const bool upd = act && g > i;
        const bool prod = act && g > i + 1;
        cplx x = mk(0.0, 0.0), yp = mk(0.0, 0.0);
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          if (ch < nch) {
            const int t0 = ch * FQ;
            cplx y[FQ];
#pragma unroll
            for (int u = 0; u < FQ; ++u) y[u] = (upd && t0 + u < ntr) ? prow[cols[t0 + u] * ldw] : mk(0.0, 0.0);
            if (ch == 0) {
              if (upd) x = cmul(prow[ci * ldw], scal);
            }
#pragma unroll
            for (int u = 0; u < FQ; ++u)
              if (upd && t0 + u < ntr) {
                y[u] = csub(y[u], cmul(x, c.vec[t0 + u]));
                prow[cols[t0 + u] * ldw] = y[u];
              }
            if (ch == 0) {
              if (upd) prow[ci * ldw] = x;
              yp = y[0];
              if (prod) {
                s2 = fma(yp.x, yp.x, fma(yp.y, yp.y, s2));
                mx = fmax(mx, fmax(fabs(yp.x), fabs(yp.y)));
              }
              if (act && g == i + 1) {
                nx->data[1] = yp;
                for (int u = 1; u < FQ; ++u)
                  if (u < ntr) nx->data[1 + r + u] = y[u];
              }
            } else if (act && g == i + 1) {
#pragma unroll
              for (int u = 0; u < FQ; ++u)
                if (t0 + u < ntr) nx->data[1 + r + t0 + u] = y[u];
            }
#pragma unroll
            for (int u = 0; u < FQ; ++u)
              y[u] = (prod && t0 + u < ntr && t0 + u > 0) ? cmulc(yp, y[u]) : mk(0.0, 0.0);
            if constexpr (FQ == 16) acc[ch] = cadd(acc[ch], warp_transpose_sum16(y));
            else acc[ch] = cadd(acc[ch], warp_transpose_sum8(y));
          }
        }
      }
      // per-warp partials -> shared memory, then every CTA's record in
      // warp order (lanes 4v hold column v of each chunk)
      cplx* part = c.wrow;  // CW x r, free during the column basis
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        // lane L holds column (L >> 2) & 7 (8-wide chunks) or (L >> 1) & 15
        const int sh = FQ == 16 ? 1 : 2;
        const int t = ch * FQ + (lane >> sh);
        if (ch < nch && (lane & ((1 << sh) - 1)) == 0 && t < ntr) part[warp * r + t] = acc[ch];
      }
      s2 = warp_sum(s2);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) c.wss[warp] = Ssq{mx, s2};
      __syncthreads();
      if (warp == 0) {
        for (int t = 1 + lane; t < ntr; t += 32) {
          cplx d = mk(0.0, 0.0);
          for (int w = 0; w < CW; ++w) d = cadd(d, part[w * r + t]);
          nx->data[1 + t] = d;
        }
        const bool own_n = (i + 1 >= lo && i + 1 < lo + nl);
        if (!own_n) {
          if (lane == 0) nx->data[1] = mk(0.0, 0.0);
          for (int t = 1 + lane; t < ntr; t += 32) nx->data[1 + r + t] = mk(0.0, 0.0);
        }
        double sum = 0.0, m2 = 0.0;
        for (int w = 0; w < CW; ++w) {
          sum += c.wss[w].ssq;
          m2 = fmax(m2, c.wss[w].scale);
        }
        if (m2 == 0.0) {
          if (lane == 0) nx->data[0] = mk(0.0, 1.0);
        } else if (m2 > 1e-140 && m2 < 1e140) {
          if (lane == 0) nx->data[0] = mk(1.0, sum);  // scale 1: the plain sum of squares
        } else {
          // out of the safe range: the scaled two-pass sum of squares
          const int cpn = cols[0];
          const int ls2 = max(0, i + 2 - lo);
          const int f0 = ls2 + lane;
          Ssq sq = ssq_of(&c.Ws[(long long)cpn * ldw + f0], 32, nl > f0 ? (nl - f0 + 31) / 32 : 0);
          sq = warp_ssq(sq);
          if (lane == 0) nx->data[0] = mk(sq.scale, sq.ssq);
        }
      }
      __syncthreads();
      SP(spt, 4);
      continue;
    }
    // local update of my rows (descending: the partials pass ran ascending)
    FOR_MY_ROWS(l, nl, g_serpentine) {
      const int g = lo + l;
      if (g < i) continue;
      if (g == i) {
        Wl(c, l, ci) = mk(h.beta, 0.0);
        for (int q = 1; q <= ntr; ++q) Wl(c, l, c.colmap[i + q]) = c.vec2[q - 1];
      } else if (!ident) {
        // issue the pivot entry and the first KB trailing entries together
        // (the store of the new pivot entry would otherwise order the
        // trailing loads after the pivot load's round trip)
#ifndef UPD_UB
#define UPD_UB KB
#endif
        constexpr int UB = UPD_UB;  // trailing loads in flight per row chunk
        cplx* prow = c.Ws + l;
        const int ld = c.ldw;
        const int* cols = c.colmap + i + 1;
        const int n0 = min(ntr, UB);
        cplx y[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) y[u] = (u < n0) ? prow[cols[u] * ld] : mk(0.0, 0.0);
        const cplx x = cmul(prow[ci * ld], scal);
#pragma unroll
        for (int u = 0; u < UB; ++u)
          if (u < n0) prow[cols[u] * ld] = csub(y[u], cmul(x, c.vec[u]));
        prow[ci * ld] = x;
        for (int q = n0; q < ntr; q += UB) {
          const int n1 = min(UB, ntr - q);
#pragma unroll
          for (int u = 0; u < UB; ++u) y[u] = (u < n1) ? prow[cols[q + u] * ld] : mk(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < UB; ++u)
            if (u < n1) prow[cols[q + u] * ld] = csub(y[u], cmul(x, c.vec[q + u]));
        }
      }
    }
    __syncthreads();
    SP(spt, 4);
    // norm recompute round (only if some column flagged; replicated decision)
    if (anyflag) {
      Rec* me2 = &c.rec[par];
      for (int q = warp; q < ntr; q += CW) {
        if (!c.flags[q]) continue;
        const int cj = c.colmap[i + 1 + q];
        const int f0 = lstart + lane;
        Ssq s = ssq_of(&c.Ws[(long long)cj * c.ldw + f0], 32, nl > f0 ? (nl - f0 + 31) / 32 : 0);
        s = warp_ssq(s);
        if (lane == 0) me2->data[q] = mk(s.scale, s.ssq);
      }
      cl.sync();
      for (int q = warp; q < ntr; q += CW) {
        if (!c.flags[q]) continue;
        const Ssq s = rank_ssq(cl, c, par, q);
        if (lane == 0) {
          const double n2 = (i < m - 1) ? ssq_norm2(s) : 0.0;
          c.cn1[i + 1 + q] = n2;
          c.cn2[i + 1 + q] = n2;
        }
      }
      par ^= 1;
      __syncthreads();
    }
  }
  SP(spt, 5);
  // rank check of _column_basis (cross.py:110-118)
  double lead = 0.0, mn = INFINITY;
  for (int t = 0; t < r; ++t) {
    lead = fmax(lead, c.betas[t]);
    mn = fmin(mn, c.betas[t]);
  }
  if (lead == 0.0 || mn < rank_tol * lead) return false;
  if (wy) {
    form_q_wy(cl, c, norms_in_q);
    return true;
  }
  // zung2r: Q = H(0)...H(r-1) [I; 0]
  for (int i = r - 1; i >= 0; --i) {
    const int ci = c.colmap[i];
    const bool own_i = (i >= lo && i < lo + nl);
    const int li = i - lo;
    const int lstart = max(0, i + 1 - lo);
    const int ntr = r - i - 1;
    const cplx ti = c.tau[i];
    if (ntr > 0) {
      Rec* me = &c.rec[par];
      for (int q = warp; q < ntr; q += CW) {
        const int cj = c.colmap[i + 1 + q];
        cplx acc = mk(0.0, 0.0);
        acc = col_dotc(c, ci, cj, lstart + lane, nl);
        acc = warp_sum(acc);
        if (lane == 0) me->data[q] = own_i ? cadd(acc, Wl(c, li, cj)) : acc;
      }
      cl.sync();
      for (int q = warp; q < ntr; q += CW) {
        const cplx s = rank_sum(cl, c, par, q);
        if (lane == 0) c.vec[q] = cmul(ti, s);
      }
      par ^= 1;
      __syncthreads();
    }
    // apply H(i) to the trailing columns and overwrite column i with
    // H(i) e_i in one pass per row (each thread owns its rows)
    const cplx mt = cneg(ti);
    for (int l = threadIdx.x; l < nl; l += CT) {
      const int g = lo + l;
      cplx& a = Wl(c, l, ci);
      if (g < i) {
        a = mk(0.0, 0.0);
        continue;
      }
      const cplx v = (g == i) ? mk(1.0, 0.0) : a;
      row_sub_cols(c, c.colmap + i + 1, c.vec, v, l, ntr);
      a = (g > i) ? cmul(a, mt) : mk(1.0 - ti.x, -ti.y);
    }
    __syncthreads();
  }
  SP(spt, 6);
  // publish Q (logical column order) to global memory for the later phases
  for (long long e = threadIdx.x; e < (long long)nl * r; e += CT) {
    const int t = (int)(e / nl), l = (int)(e - (long long)t * nl);
    c.Qg[(long long)t * m + lo + l] = Wl(c, l, c.colmap[t]);
  }
  __threadfence();
  __syncthreads();
  return true;
}

#include "k_tsqr.cuh"

// ------------------------------------------------------------ phase D
// X = Q[rows]^-1 into aug's right half (every CTA, redundantly); returns
// log|det Q[rows]|.
__device__ double invert_rows(const CC& c, const int* rows) {
  const int r = c.r, ld = 2 * r;
  for (int e = threadIdx.x; e < r * ld; e += CT) {
    const int i = e / ld, j = e - i * ld;
    c.aug[e] = (j < r) ? Qrow(c, rows[i])[(long long)j * c.m] : mk((j - r == i) ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  return gauss_jordan_fast<CT>(c.aug, r, c.vec2, c.ibc);
}

// My rows of Q X on the FP64 tensor cores (DMMA m8n8k4), r <= 32: Q rows
// are staged QX_ROWS at a time as interleaved reals (the A operand as
// stored); X (complex r x r, ld ldx) is expanded once per call into the
// B-fragment registers of each warp (warp w owns real n-tile w & 7 and
// m-tiles (w >> 3) + 2i of every staged tile).  sink(l, j, value) receives
// every output entry.  Same products as rowblock_X up to the association of
// the r-term sums.
template <class Sink>
__device__ void qx_dmma(const CC& c, const cplx* X, int ldx, Sink sink) {
  const int r = c.r, lo = c.row0, nl = c.nrows, m = c.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int Kp = (2 * r + 3) & ~3, ldA = Kp + 4, nks = Kp / 4;
  const int ntn = (2 * r + 7) / 8;
  const int nt = warp & 7, mgrp = warp >> 3;
  constexpr int MG = CW / 8;  // warp groups over m-tiles
  const bool active = nt < ntn && warp < 8 * MG;  // CW need not be a multiple of 8
  double breg[16];
#pragma unroll
  for (int ks = 0; ks < 16; ++ks) {
    const int k = 4 * ks + tig, n = nt * 8 + gid;
    const int a = k >> 1, col = n >> 1;
    double b = 0.0;
    if (ks < nks && a < r && col < r) {
      const cplx x = X[a * ldx + col];
      b = ((k & 1) == (n & 1)) ? x.x : ((n & 1) ? x.y : -x.y);
    }
    breg[ks] = b;
  }
  // two staging buffers: the Q row tile of step t+1 streams in (cp.async)
  // while step t runs on the tensor cores
  double* tiles[2] = {c.qtile, c.qtile + QX_ROWS * ldA};
  __syncthreads();  // the region is shared with the starts' per-row state
  for (int e = threadIdx.x; e < 2 * QX_ROWS * (Kp - 2 * r); e += CT) {
    const int bb = e / (QX_ROWS * (Kp - 2 * r)), e2 = e - bb * QX_ROWS * (Kp - 2 * r);
    const int row = e2 / (Kp - 2 * r), k = 2 * r + (e2 - row * (Kp - 2 * r));
    tiles[bb][row * ldA + k] = 0.0;
  }
  // rows past nl are zero-filled by cp.async with a 0-byte source
  auto issue = [&](int l0, double* dst) {
    for (int e = threadIdx.x; e < QX_ROWS * r; e += CT) {
      const int t = e / QX_ROWS, row = e - t * QX_ROWS;
      const int l = l0 + row;
      const cplx* src = c.Qg + (long long)t * m + lo + min(l, nl - 1);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + row * ldA + 2 * t);
      const int bytes = (l < nl) ? 16 : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(bytes));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  issue(0, tiles[0]);
  int buf = 0;
  for (int l0 = 0; l0 < nl; l0 += QX_ROWS, buf ^= 1) {
    if (l0 + QX_ROWS < nl) {
      issue(l0 + QX_ROWS, tiles[buf ^ 1]);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* tile = tiles[buf];
    if (active) {
      for (int mi = mgrp; mi < QX_ROWS / 8; mi += MG) {
        const int m0 = mi * 8;
        double c0 = 0.0, c1 = 0.0;
        const double* arow = tile + (m0 + gid) * ldA + tig;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          if (ks < nks) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c0), "+d"(c1) : "d"(arow[4 * ks]), "d"(breg[ks]));
          }
        }
        const int l = l0 + m0 + gid, j = nt * 4 + tig;
        if (l < nl && j < r) sink(l, j, mk(c0, c1));
      }
    }
    __syncthreads();  // tile buf is refilled by the issue two steps later
  }
}

// B = Q X for my rows (into Ws) and for the selected rows (selb); returns my
// best |B| candidate (key = global row-major index).
__device__ Cand form_B(const CC& c) {
  const int r = c.r, lo = c.row0, nl = c.nrows, ld = 2 * r;
  const cplx* X = c.aug + r;
  Cand a{-1.0, LLONG_MAX, -1};
  constexpr int JB = 16;
  if (c.qtile) {
    qx_dmma(c, X, ld, [&](int l, int j, cplx v) {
      Wl(c, l, j) = v;
      const Cand b{cabs2(v), (long long)(lo + l) * r + j, l};
      if (cand_better(b, a)) a = b;
    });
  } else
  for (int l = threadIdx.x; l < nl; l += CT) {
    const cplx* q = Qrow(c, lo + l);
    for (int j0 = 0; j0 < r; j0 += JB) {
      cplx acc[JB];
      rowblock_X<JB>(q, c.m, X, ld, j0, r, acc);
#pragma unroll
      for (int jj = 0; jj < JB; ++jj) {
        const int j = j0 + jj;
        if (j < r) {
          Wl(c, l, j) = acc[jj];
          Cand b{cabs2(acc[jj]), (long long)(lo + l) * r + j, l};
          if (cand_better(b, a)) a = b;
        }
      }
    }
  }
  const int nch = (r + JB - 1) / JB;
  for (int e = threadIdx.x; e < r * nch; e += CT) {
    const int q = e / nch, j0 = (e - q * nch) * JB;
    cplx acc[JB];
    rowblock_X<JB>(Qrow(c, c.sel[q]), c.m, X, ld, j0, r, acc);
#pragma unroll
    for (int jj = 0; jj < JB; ++jj)
      if (j0 + jj < r) c.selb[q * r + j0 + jj] = acc[jj];
  }
  __syncthreads();
  return a;
}

// ======================================================================
// Warp-granular rounds.  Every warp publishes its own best candidate and
// that row's data; after the cluster barrier every warp independently finds
// the cluster-wide winner among the C*CW records and loads the winning row,
// so a step needs exactly one barrier (the cluster barrier) and no block
// barrier.
// ======================================================================
__device__ __forceinline__ void warp_publish(const CC& c, int par, const Cand& a) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WCand* slot = &c.wrec[par * CW + w];
  if (lane == 0) {
    slot->v = a.v;
    slot->key = a.key;
    slot->row = a.row >= 0 ? c.row0 + a.row : -1;
  }
  if (a.row >= 0) {
    cplx* dst = c.wrow + ((long long)par * CW + w) * c.r;
    for (int t = lane; t < c.r; t += 32) dst[t] = Wl(c, a.row, t);
  }
}

struct Winner {
  Cand w;
  int rank, slot;
};

__device__ __forceinline__ Winner warp_winner_in(cg::cluster_group& cl, WCand* recs, int par);

__device__ __forceinline__ Winner warp_winner(cg::cluster_group& cl, const CC& c, int par) {
  return warp_winner_in(cl, c.wrec, par);
}

// C*CW per-warp records of buffer `par` at recs (same offset in every CTA)
__device__ __forceinline__ Winner warp_winner_in(cg::cluster_group& cl, WCand* recs, int par) {
  const int lane = threadIdx.x & 31;
  const int C = (int)cl.num_blocks();
  const int total = C * CW;
  Cand best{-1.0, LLONG_MAX, -1};
  int bidx = -1;
  // issue every remote load first (one DSMEM round trip), then compare
  constexpr int PER = (16 * CW + 31) / 32;
  double vv[PER];
  long long kk[PER];
  int rw[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int e = lane + 32 * q;
    rw[q] = -1;
    if (e < total) {
      const int rk = e / CW, sl = e - rk * CW;
      const WCand* p = cl.map_shared_rank(&recs[par * CW + sl], rk);
      vv[q] = p->v;
      kk[q] = p->key;
      rw[q] = p->row;
    }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const Cand x{vv[q], kk[q], rw[q]};
    if (x.row >= 0 && (bidx < 0 || cand_better(x, best))) {
      best = x;
      bidx = lane + 32 * q;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand b;
    b.v = __shfl_xor_sync(0xffffffffu, best.v, o);
    b.key = __shfl_xor_sync(0xffffffffu, best.key, o);
    b.row = __shfl_xor_sync(0xffffffffu, best.row, o);
    const int bi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (bi >= 0 && (bidx < 0 || cand_better(b, best))) {
      best = b;
      bidx = bi;
    }
  }
  Winner W;
  W.w = best;
  W.rank = bidx / CW;
  W.slot = bidx - W.rank * CW;
  return W;
}

// entries t = lane and t = lane + 32 of the winner's published row
__device__ __forceinline__ void winner_row(cg::cluster_group& cl, const CC& c, int par, const Winner& W,
                                           cplx& x0, cplx& x1) {
  const int lane = threadIdx.x & 31;
  const cplx* src = cl.map_shared_rank(c.wrow + ((long long)par * CW + W.slot) * c.r, W.rank);
  x0 = (lane < c.r) ? src[lane] : mk(0.0, 0.0);
  x1 = (lane + 32 < c.r) ? src[lane + 32] : mk(0.0, 0.0);
}

__device__ __forceinline__ cplx lane_entry(cplx x0, cplx x1, int t) {
  const cplx s = (t < 32) ? x0 : x1;
  cplx v;
  v.x = __shfl_sync(0xffffffffu, s.x, t & 31);
  v.y = __shfl_sync(0xffffffffu, s.y, t & 31);
  return v;
}

__device__ __forceinline__ int lane_first(int f0, int f1, int t) {
  return __shfl_sync(0xffffffffu, (t < 32) ? f0 : f1, t & 31);
}

// LAPACK interchange of positions i <-> pvt, tracked by warp 0 in registers
// (lane t holds first[t], first[t+32]); returns the row A previously at i.
__device__ __forceinline__ int swap_first(const CC& c, int& f0, int& f1, int i, int B, int pvt) {
  const int lane = threadIdx.x & 31;
  const int A = lane_first(f0, f1, i);
  if (lane == (i & 31)) {
    if (i < 32) f0 = B;
    else f1 = B;
  }
  if (pvt < c.r && lane == (pvt & 31)) {
    if (pvt < 32) f0 = A;
    else f1 = A;
  }
  return A;
}

// Position bookkeeping for the rows this thread owns (after the barrier).
__device__ __forceinline__ void apply_positions(const CC& c, int i, int A, int B, int pvt) {
  const int la = A - c.row0, lb = B - c.row0;
  if (la >= 0 && la < c.nrows && (la % CT) == (int)threadIdx.x) c.rpos[la] = pvt;
  if (lb >= 0 && lb < c.nrows && (lb % CT) == (int)threadIdx.x) c.rpos[lb] = i;
}

// ======================================================================
// Shared-winner rounds: every warp publishes its candidate (no block barrier
// before the cluster barrier); after it, warp 0 alone reads the C*CW records
// and the winning row over DSMEM (one remote read per CTA, so the winner's
// shared-memory port is not flooded), prepares the broadcast vector in local
// shared memory S = c.vec2, and one block barrier hands it to all warps.
// ======================================================================
struct Bcast {
  int i, A, B, pvt;
};

__device__ __forceinline__ Bcast read_bcast(const CC& c) {
  return Bcast{c.ibc[4], c.ibc[5], c.ibc[6], c.ibc[7]};
}

// ---------------------------------------------------------- phase B
__device__ void start_qrcp_qh_s(cg::cluster_group& cl, CC& c, int& par) {
  const int r = c.r, lo = c.row0, nl = c.nrows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // vn1/vn2 hold SQUARED partial norms here: zlaqp2's downdate
  //   temp = max(0, 1 - (|a|/vn1)^2); recompute iff temp*(vn1/vn2)^2 <= tol3z
  // is exactly  s1' = max(0, s1 - |a|^2); recompute iff s1' <= tol3z * s2,
  // which needs no division, sqrt or hypot (the argmax is order-preserving).
  for (int l = threadIdx.x; l < nl; l += CT) {
    for (int t = 0; t < r; ++t) Wl(c, l, t) = cconj(Qrow(c, lo + l)[(long long)t * c.m]);
    const double n2 = ssq_norm2(ssq_of(&Wl(c, l, 0), c.ldw, r));
    c.vn1[l] = n2;
    c.vn2[l] = n2;
    c.rpos[l] = lo + l;
  }
  int f0 = lane, f1 = lane + 32;  // warp 0 only
  cplx* S = c.vec2;               // v (reflector) of the previous step
  SP_BEGIN(spt);
  for (int i = 0; i <= r; ++i) {
    Cand a{-1.0, LLONG_MAX, -1};
    const cplx tc = cconj(c.cbc[1]);
    for (int l = threadIdx.x; l < nl; l += CT) {
      const int p = c.rpos[l];
      if (i > 0 && p > i - 1) {
        // H(i-1)^H applied to this column of Q^H, then the zlaqp2 norm update
        const int i0 = i - 1;
        const cplx sacc = row_dotc(c, S, l, i0, r);
        const cplx tt = cmul(tc, sacc);
        row_sub_scaled(c, S, tt, l, i0, r);
        const double s1 = c.vn1[l];
        if (s1 != 0.0) {
          const double s1n = fmax(s1 - cabs2(Wl(c, l, i0)), 0.0);
          if (s1n <= TOL3Z * c.vn2[l]) {
            const double n2 = (i0 < r - 1) ? ssq_norm2(ssq_of(&Wl(c, l, i0 + 1), c.ldw, r - i0 - 1)) : 0.0;
            c.vn1[l] = n2;
            c.vn2[l] = n2;
          } else {
            c.vn1[l] = s1n;
          }
        }
      }
      if (i < r && p >= i) {
        const Cand b{c.vn1[l], p, l};
        if (cand_better(b, a)) a = b;
      }
    }
    SP(spt, 8);
    if (i == r) break;
    a = warp_cand(a);
    __syncwarp();
    warp_publish(c, par, a);
    SP(spt, 9);
    cl.sync();
    SP(spt, 10);
    if (warp == 0) {
      const Winner W = warp_winner(cl, c, par);
      cplx x0, x1;
      winner_row(cl, c, par, W, x0, x1);
      SP(spt, 11);
      double s2 = 0.0;
      if (lane > i && lane < r) s2 += cabs2(x0);
      if (lane + 32 > i && lane + 32 < r) s2 += cabs2(x1);
      s2 = warp_sum(s2);
      const cplx alpha = lane_entry(x0, x1, i);
      const Reflector h = zlarfg_fast(alpha, s2);
      const cplx sc = reflector_scale(h);
      const bool ident = is_zero(h.tau);
      if (lane >= i && lane < r) S[lane] = (lane == i) ? mk(1.0, 0.0) : (ident ? x0 : cmul(x0, sc));
      if (lane + 32 >= i && lane + 32 < r) S[lane + 32] = (lane + 32 == i) ? mk(1.0, 0.0) : (ident ? x1 : cmul(x1, sc));
      const int A = swap_first(c, f0, f1, i, W.w.row, (int)W.w.key);
      if (lane == 0) {
        c.cbc[1] = h.tau;
        c.ibc[4] = i;
        c.ibc[5] = A;
        c.ibc[6] = W.w.row;
        c.ibc[7] = (int)W.w.key;
      }
      SP(spt, 12);
    }
    __syncthreads();
    SP(spt, 13);
    const Bcast bc = read_bcast(c);
    apply_positions(c, bc.i, bc.A, bc.B, bc.pvt);
    par ^= 1;
  }
  if (warp == 0) {
    c.starts[lane] = f0;
    if (lane + 32 < r) c.starts[lane + 32] = f1;
  }
  __syncthreads();
}

// ---------------------------------------------------------- phase C
__device__ void start_lu_s(cg::cluster_group& cl, CC& c, int& par) {
  const int r = c.r, lo = c.row0, nl = c.nrows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int l = threadIdx.x; l < nl; l += CT) {
    for (int t = 0; t < r; ++t) Wl(c, l, t) = Qrow(c, lo + l)[(long long)t * c.m];
    c.rpos[l] = lo + l;
  }
  int f0 = lane, f1 = lane + 32;
  cplx* S = c.vec2;  // pivot row of the previous step
  for (int k = 0; k <= r; ++k) {
    Cand a{-1.0, LLONG_MAX, -1};
    const cplx rp = c.cbc[1];
    const bool nz = (k > 0) && !is_zero(rp);
    for (int l = threadIdx.x; l < nl; l += CT) {
      const int p = c.rpos[l];
      if (nz && p > k - 1) {
        const cplx mult = cmul(Wl(c, l, k - 1), rp);
        Wl(c, l, k - 1) = mult;
        row_sub_scaled(c, S, mult, l, k, r);
      }
      if (k < r && p >= k) {
        const Cand b{cabs1(Wl(c, l, k)), p, l};
        if (cand_better(b, a)) a = b;
      }
    }
    if (k == r) break;
    a = warp_cand(a);
    __syncwarp();
    warp_publish(c, par, a);
    cl.sync();
    if (warp == 0) {
      const Winner W = warp_winner(cl, c, par);
      cplx x0, x1;
      winner_row(cl, c, par, W, x0, x1);
      if (lane < r) S[lane] = x0;
      if (lane + 32 < r) S[lane + 32] = x1;
      const cplx piv = lane_entry(x0, x1, k);
      const int A = swap_first(c, f0, f1, k, W.w.row, (int)W.w.key);
      if (lane == 0) {
        c.cbc[1] = is_zero(piv) ? mk(0.0, 0.0) : cdiv(mk(1.0, 0.0), piv);
        c.ibc[4] = k;
        c.ibc[5] = A;
        c.ibc[6] = W.w.row;
        c.ibc[7] = (int)W.w.key;
      }
    }
    __syncthreads();
    const Bcast bc = read_bcast(c);
    apply_positions(c, bc.i, bc.A, bc.B, bc.pvt);
    par ^= 1;
  }
  if (warp == 0) {
    c.starts[r + lane] = f0;
    if (lane + 32 < r) c.starts[r + lane + 32] = f1;
  }
  __syncthreads();
}

// ---------------------------------------------------------- phase B+C fused
// Both starts of _dominant_rows (cross.py:172-177) in ONE sequence of r
// rounds that only READ Q:
//
//  * QRCP of Q^H (zlaqp2): after i reflectors the transformed column of
//    row g is  T_i conj(q_g),  T_i = H_{i-1}^H..H_0^H, so the entry step i
//    downdates with is  (Pi_{i+1} e_i)^H conj(q_g) = conj(sum_c Pi[c,i] q_g[c])
//    where Pi_i = H_0..H_{i-1} (r x r, shared memory).  The winner's
//    transformed column (for zlarfg) is Pi_i^H conj(q_p); a recompute
//    (tol3z) takes the trailing norm of Pi_{i+1}[:, i+1:]^H conj(q_g).
//  * LU with partial pivoting (zgetrf): the Schur entry of row g at step k
//    is  s_gk = q_g[k] - q_g[:k] M_k[:, k],  M_k = U_k^-1 U[:k, :]
//    (k x r, shared memory), updated by one rank-1 step per pivot; the
//    winner's U row is  q_p[c] - q_p[:k] M_k[:, c].
//
// Every round is one pass over the Q rows (no copies, no writes), one
// cluster barrier for both arg-maxes, and warps 0 / 1 derive the two
// winners concurrently.  Pivot decisions are those of the two LAPACK
// factorizations; the entries agree with the rank-1-updated ones to
// rounding (same argument as the compact-WY Q).
constexpr int PLD_PAD = 1;  // Pi / M leading dimension r + 1: conflict-free rows and columns

__device__ __forceinline__ int pi_ld(int r) { return r + PLD_PAD; }

__device__ __forceinline__ void load_qrow_lanes(const CC& c, int g, cplx* dst) {
  const int lane = threadIdx.x & 31;
  const cplx* q = Qrow(c, g);
  for (int t = lane; t < c.r; t += 32) dst[t] = q[(long long)t * c.m];
  __syncwarp();
}

__device__ void start_pair_s(cg::cluster_group& cl, CC& c, int& par, bool norms_ready) {
  const int r = c.r, lo = c.row0, nl = c.nrows, m = c.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = pi_ld(r);
  cplx* Pi = c.aug;    // Pi(c, c') at c' * ld + c   (r x (r+1) <= 2 r^2)
  cplx* Mm = c.selb;   // M(j, c) at j * r + c        (r x r)
  cplx* u = c.sp;            // [r]  Pi_{i+1}[:, i] for the next downdate
  cplx* w2 = c.sp + r;       // [r]  M_{k+1}[:, k+1] for the next Schur column
  cplx* qr1 = c.sp + 2 * r;  // [r]  winner Q rows
  cplx* qr2 = c.sp + 3 * r;
  cplx* vv = c.sp + 4 * r;   // [r]  reflector v (entries >= i)
  cplx* yy = c.sp + 5 * r;   // [r]  Pi v
  cplx* mrow = c.sp + 6 * r; // [r]  new M row U[k, :] / U[k, k]
  cplx* mcol = c.sp + 7 * r; // [r]  M_k[:, k]
  for (int e = threadIdx.x; e < r * ld; e += CT) {
    const int cc = e / ld, rr = e - cc * ld;
    Pi[e] = mk((rr == cc) ? 1.0 : 0.0, 0.0);
  }
  if (!norms_ready)
    for (int l = threadIdx.x; l < nl; l += CT) {
      const double n2 = ssq_norm2(ssq_of(Qrow(c, lo + l), m, r));
      c.vn1[l] = n2;
      c.vn2[l] = n2;
      c.rpos[l] = lo + l;
      c.rpos2[l] = lo + l;
    }
  int f0 = lane, f1 = lane + 32;  // warp 0: QRCP first[]; warp 1: LU first[]
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    // ---- row pass: downdate with step k-1 (QRCP), Schur column k (LU)
    Cand a1{-1.0, LLONG_MAX, -1}, a2{-1.0, LLONG_MAX, -1};
    FOR_MY_ROWS(l, nl, g_serpentine && ((k & 1) == 0)) {  // the norm pass before round 0 ran ascending
      const int p1 = c.rpos[l], p2 = c.rpos2[l];
      const bool dd = (k > 0 && p1 > k - 1);
      const bool lu = (p2 >= k);
      if (!dd && !lu) {
        if (p1 >= k) {
          const Cand b{c.vn1[l], p1, l};
          if (cand_better(b, a1)) a1 = b;
        }
        continue;
      }
      const cplx* q = Qrow(c, lo + l);
      cplx t1 = mk(0.0, 0.0), s2 = mk(0.0, 0.0);
      int t = 0;
      constexpr int KS = 2 * KB;  // 16 loads in flight per thread
      for (; t + KS <= r; t += KS) {
        cplx x[KS];
#pragma unroll
        for (int qq = 0; qq < KS; ++qq) x[qq] = q[(long long)(t + qq) * m];
#pragma unroll
        for (int qq = 0; qq < KS; ++qq) {
          t1 = cfma(u[t + qq], x[qq], t1);
          if (t + qq < k) s2 = cfma(x[qq], w2[t + qq], s2);
          else if (t + qq == k) s2 = csub(x[qq], s2);
        }
      }
      for (; t < r; ++t) {
        const cplx x = q[(long long)t * m];
        t1 = cfma(u[t], x, t1);
        if (t < k) s2 = cfma(x, w2[t], s2);
        else if (t == k) s2 = csub(x, s2);
      }
      if (dd) {
        const double s1 = c.vn1[l];
        if (s1 != 0.0) {
          const double s1n = fmax(s1 - cabs2(t1), 0.0);
          if (s1n <= TOL3Z * c.vn2[l]) {
            // trailing norm of the transformed column: entries k .. r-1
            Ssq s = ssq_init();
            for (int cc = k; cc < r; ++cc) {
              cplx e = mk(0.0, 0.0);
              for (int j = 0; j < r; ++j) e = cfma(Pi[cc * ld + j], q[(long long)j * m], e);
              ssq_addc(s, e);
            }
            const double n2 = (k - 1 < r - 1) ? ssq_norm2(s) : 0.0;
            c.vn1[l] = n2;
            c.vn2[l] = n2;
          } else {
            c.vn1[l] = s1n;
          }
        }
      }
      if (p1 >= k) {
        const Cand b{c.vn1[l], p1, l};
        if (cand_better(b, a1)) a1 = b;
      }
      if (lu) {
        const Cand b{cabs1(s2), p2, l};
        if (cand_better(b, a2)) a2 = b;
      }
    }
    a1 = warp_cand(a1);
    a2 = warp_cand(a2);
    if (lane == 0) {
      WCand* s1p = &c.wrec[par * CW + warp];
      s1p->v = a1.v;
      s1p->key = a1.key;
      s1p->row = a1.row >= 0 ? lo + a1.row : -1;
      WCand* s2p = &c.wrec2[par * CW + warp];
      s2p->v = a2.v;
      s2p->key = a2.key;
      s2p->row = a2.row >= 0 ? lo + a2.row : -1;
    }
    cl.sync();
    if (warp == 0) {
      // ---- QRCP winner: reflector H_k from Pi_k^H conj(q_p)
      const Winner W = warp_winner_in(cl, c.wrec, par);
      load_qrow_lanes(c, W.w.row, qr1);
      cplx x0 = mk(0.0, 0.0), x1 = mk(0.0, 0.0);
      for (int cc = lane; cc < r; cc += 32) {
        cplx e = mk(0.0, 0.0);
        for (int j = 0; j < r; ++j) e = cfma(Pi[cc * ld + j], qr1[j], e);
        if (cc < 32) x0 = cconj(e);
        else x1 = cconj(e);
      }
      double sx = 0.0;
      if (lane > k && lane < r) sx += cabs2(x0);
      if (lane + 32 > k && lane + 32 < r) sx += cabs2(x1);
      sx = warp_sum(sx);
      const cplx alpha = lane_entry(x0, x1, k);
      const Reflector h = zlarfg_fast(alpha, sx);
      const cplx sc = reflector_scale(h);
      const bool ident = is_zero(h.tau);
      for (int cc = lane; cc < r; cc += 32) {
        const cplx xv = (cc < 32) ? x0 : x1;
        vv[cc] = (cc < k) ? mk(0.0, 0.0) : (cc == k) ? mk(1.0, 0.0) : (ident ? xv : cmul(xv, sc));
      }
      __syncwarp();
      // y = Pi v; u = Pi_{k+1}[:, k] = Pi[:, k] - tau y  (v[k] = 1)
      for (int cc = lane; cc < r; cc += 32) {
        cplx y = mk(0.0, 0.0);
        for (int j = k; j < r; ++j) y = cfma(Pi[j * ld + cc], vv[j], y);
        yy[cc] = y;
        u[cc] = csub(Pi[k * ld + cc], cmul(h.tau, y));
      }
      const int A = swap_first(c, f0, f1, k, W.w.row, (int)W.w.key);
      if (lane == 0) {
        c.cbc[1] = h.tau;
        c.ibc[4] = k;
        c.ibc[5] = A;
        c.ibc[6] = W.w.row;
        c.ibc[7] = (int)W.w.key;
      }
    } else if (warp == 1) {
      // ---- LU winner: U row k, pivot, next Schur multipliers
      const Winner W = warp_winner_in(cl, c.wrec2, par);
      load_qrow_lanes(c, W.w.row, qr2);
      cplx u0 = mk(0.0, 0.0), u1 = mk(0.0, 0.0);
      for (int cc = lane; cc < r; cc += 32) {
        cplx e = mk(0.0, 0.0);
        if (cc >= k) {
          for (int j = 0; j < k; ++j) e = cfma(qr2[j], Mm[j * r + cc], e);
          e = csub(qr2[cc], e);
        }
        if (cc < 32) u0 = e;
        else u1 = e;
      }
      const cplx piv = lane_entry(u0, u1, k);
      const bool zp = is_zero(piv);
      const cplx rp = zp ? mk(0.0, 0.0) : cdiv(mk(1.0, 0.0), piv);
      for (int cc = lane; cc < r; cc += 32) {
        const cplx e = (cc < 32) ? u0 : u1;
        mrow[cc] = (cc < k || zp) ? mk(0.0, 0.0) : (cc == k ? mk(1.0, 0.0) : cmul(e, rp));
        if (cc < k) mcol[cc] = Mm[cc * r + k];
      }
      __syncwarp();
      // w2 = M_{k+1}[:, k+1]
      if (k + 1 < r) {
        for (int j = lane; j <= k; j += 32)
          w2[j] = (j < k) ? csub(Mm[j * r + k + 1], cmul(mcol[j], mrow[k + 1])) : mrow[k + 1];
      }
      const int A = swap_first(c, f0, f1, k, W.w.row, (int)W.w.key);
      if (lane == 0) {
        c.ibc[8] = k;
        c.ibc[9] = A;
        c.ibc[10] = W.w.row;
        c.ibc[11] = (int)W.w.key;
      }
    }
    __syncthreads();
    // ---- replicated bookkeeping and the two small rank-1 updates
    {
      const int i = c.ibc[4], A = c.ibc[5], B = c.ibc[6], pvt = c.ibc[7];
      const int la = A - lo, lb = B - lo;
      if (la >= 0 && la < nl && (la % CT) == (int)threadIdx.x) c.rpos[la] = pvt;
      if (lb >= 0 && lb < nl && (lb % CT) == (int)threadIdx.x) c.rpos[lb] = i;
      const int i2 = c.ibc[8], A2 = c.ibc[9], B2 = c.ibc[10], pvt2 = c.ibc[11];
      const int la2 = A2 - lo, lb2 = B2 - lo;
      if (la2 >= 0 && la2 < nl && (la2 % CT) == (int)threadIdx.x) c.rpos2[la2] = pvt2;
      if (lb2 >= 0 && lb2 < nl && (lb2 % CT) == (int)threadIdx.x) c.rpos2[lb2] = i2;
    }
    const cplx tau = c.cbc[1];
    const int ncol = r - k;
    for (int e = threadIdx.x; e < r * ncol; e += CT) {
      const int cp = k + e / r, cc = e - (e / r) * r;  // Pi(cc, cp) -= tau y[cc] conj(v[cp])
      Pi[cp * ld + cc] = csub(Pi[cp * ld + cc], cmul(cmul(tau, yy[cc]), cconj(vv[cp])));
    }
    for (int e = threadIdx.x; e < (k + 1) * ncol; e += CT) {
      const int j = e / ncol, cc = k + (e - j * ncol);
      if (j < k) Mm[j * r + cc] = csub(Mm[j * r + cc], cmul(mcol[j], mrow[cc]));
      else Mm[k * r + cc] = mrow[cc];
    }
    par ^= 1;
    __syncthreads();
  }
  if (warp == 0) {
    if (lane < r) c.starts[lane] = f0;
    if (lane + 32 < r) c.starts[lane + 32] = f1;
  } else if (warp == 1) {
    if (lane < r) c.starts[r + lane] = f0;
    if (lane + 32 < r) c.starts[r + lane + 32] = f1;
  }
  __syncthreads();
}

// ---------------------------------------------------------- phase D
// Split cluster barrier (all threads of every CTA): arrive has release and
// wait acquire semantics, so memory reads before a peer's arrive happen
// before writes after my wait.
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One row pass of the swaps over my rows with NP updates still to apply:
// entry (l, t) of the current B is
//   B_W[l, t] + sum_{s < NP} c_s(l) w_s[t],   c_s(l) = B_{s-1}[l, j_s],
// with B_W the slice as stored and c_s(l) accumulated by the same fma chain
// the eager updates would have run, so every value (and the argmax) is
// bitwise the eager one.  flush: write the current B back (B_W := B).
// Returns my best |B|^2 candidate.
// BND: also leave each row's max |B(l, t)| in c.vn1 (the exact bound the
// filtered passes below start from; vn1 is free once the starts are done).
template <int NP, bool BND>
__device__ __forceinline__ Cand swap_pass(const CC& c, const cplx* pw, const int* pj, bool flush, bool rev) {
  const int r = c.r, lo = c.row0, nl = c.nrows;
  // running best as (|v|^2, 32-bit row-major key): fewer live registers
  // than a Cand in the hottest loop; the row follows from the key
  double bv = -1.0;
  int bk = INT_MAX;
  FOR_MY_ROWS(l, nl, rev) {
    cplx* p = c.Ws + l;
    const long long ld = c.ldw;
    cplx cs[NP];
#pragma unroll
    for (int s = 0; s < NP; ++s) cs[s] = p[pj[s] * ld];
#pragma unroll
    for (int s = 1; s < NP; ++s)
#pragma unroll
      for (int u = 0; u < s; ++u) cs[s] = cfma(cs[u], pw[u * r + pj[s]], cs[s]);
    const int rk = (lo + l) * r;
    double rm = 0.0;
    int t = 0;
    // the hottest loop: 16 loads in flight (8 with three or more pending
    // updates, whose coefficients take the registers)
#ifndef SW_KS34
#define SW_KS34 KB
#endif
    constexpr int KS = NP <= 2 ? 2 * KB : SW_KS34;
    for (; t + KS <= r; t += KS) {
      cplx x[KS];
#pragma unroll
      for (int q = 0; q < KS; ++q) x[q] = p[(t + q) * ld];
#pragma unroll
      for (int q = 0; q < KS; ++q) {
        cplx v = x[q];
#pragma unroll
        for (int s = 0; s < NP; ++s) v = cfma(cs[s], pw[s * r + t + q], v);
        if (flush) p[(t + q) * ld] = v;
        const double v2 = cabs2(v);
        if (BND) rm = fmax(rm, v2);
        if (v2 > bv || (v2 == bv && rk + t + q < bk)) {
          bv = v2;
          bk = rk + t + q;
        }
      }
    }
    for (; t < r; ++t) {
      cplx v = p[t * ld];
#pragma unroll
      for (int s = 0; s < NP; ++s) v = cfma(cs[s], pw[s * r + t], v);
      if (flush) p[t * ld] = v;
      const double v2 = cabs2(v);
      if (BND) rm = fmax(rm, v2);
      if (v2 > bv || (v2 == bv && rk + t < bk)) {
        bv = v2;
        bk = rk + t;
      }
    }
    if (BND) c.vn1[l] = sqrt(rm);
  }
  Cand a{-1.0, LLONG_MAX, -1};
  if (bk != INT_MAX) a = Cand{bv, (long long)bk, bk / r - lo};
  return a;
}

// Bound-filtered row pass (global-slice mode, no flush).  c.vn1[l] holds an
// upper bound on max_t |B(l, t)|; the newest update B += c_n(l) w_n raises it
// by at most |c_n(l)| max_t |w_n[t]|.  T is a running lower bound on the
// warp's maximum: the warp's best entry of the previous pass, re-evaluated,
// then every exact entry this pass has formed so far.  A row first forms its
// update coefficients (NP column loads, as in swap_pass) and its entry in the
// newest pivot column; only if its bound reaches T (with a 1e-11 relative
// margin over the rounding of the bounds) are its other entries read.  Every
// skipped row's entries are below T, and every evaluated entry runs the same
// fma chain as swap_pass, so the warp's best (value, row-major key) is
// bitwise the one the full pass returns.  A row costs the full pass's loads
// at worst (the cluster barrier waits for the slowest warp), and one
// coalesced load per pending update when skipped.
template <int NP>
__device__ __forceinline__ Cand swap_pass_filt(const CC& c, const cplx* pw, const int* pj, double wmax,
                                               const Cand prev, bool rev) {
  const int r = c.r, lo = c.row0, nl = c.nrows;
  const long long ld = c.ldw;
  const int jn = pj[NP - 1];
  const cplx wnj = pw[(NP - 1) * r + jn];
  double* bnd = c.vn1;
  double bv = -1.0;
  int bk = INT_MAX;
  auto take = [&](double v2, int key) {
    if (v2 > bv || (v2 == bv && key < bk)) {
      bv = v2;
      bk = key;
    }
  };
  // chain of the row's update coefficients (same fma order as swap_pass)
  auto coeffs = [&](const cplx* p, cplx* cs) {
#pragma unroll
    for (int s = 0; s < NP; ++s) cs[s] = p[pj[s] * ld];
#pragma unroll
    for (int s = 1; s < NP; ++s)
#pragma unroll
      for (int u = 0; u < s; ++u) cs[s] = cfma(cs[u], pw[u * r + pj[s]], cs[s]);
  };
  const int prow = prev.row;  // the warp's previous best (local row), or -1
  if (prow >= 0 && prow % CT == (int)threadIdx.x) {
    const int pt = (int)(prev.key - (long long)(lo + prow) * r);
    const cplx* p = c.Ws + prow;
    cplx cs[NP];
    coeffs(p, cs);
    cplx v = p[pt * ld];
#pragma unroll
    for (int s = 0; s < NP; ++s) v = cfma(cs[s], pw[s * r + pt], v);
    take(cabs2(v), (lo + prow) * r + pt);
  }
  double T2 = bv;
  const int nk = (nl + CT - 1) / CT;
  constexpr int KS = NP <= 2 ? 2 * KB : KB;
  for (int k = 0; k < nk; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) T2 = fmax(T2, __shfl_xor_sync(0xffffffffu, T2, o));
    const int l = (int)threadIdx.x + (rev ? nk - 1 - k : k) * CT;
    if (l < nl) {
      const cplx* p = c.Ws + l;
      cplx cs[NP];
      coeffs(p, cs);
      const double bo = bnd[l];
      const cplx cn = cs[NP - 1];
      const int rk = (lo + l) * r;
      take(cabs2(cfma(cn, wnj, cn)), rk + jn);  // entry (l, jn) after the update
      double bound = fma(sqrt(cabs2(cn)), wmax, bo);
      if (!(bound * bound < T2 * (1.0 - 1e-11))) {
        double rm = 0.0;
        int t = 0;
        for (; t + KS <= r; t += KS) {
          cplx x[KS];
#pragma unroll
          for (int q = 0; q < KS; ++q) x[q] = p[(t + q) * ld];
#pragma unroll
          for (int q = 0; q < KS; ++q) {
            cplx v = x[q];
#pragma unroll
            for (int s = 0; s < NP; ++s) v = cfma(cs[s], pw[s * r + t + q], v);
            const double v2 = cabs2(v);
            rm = fmax(rm, v2);
            take(v2, rk + t + q);
          }
        }
        for (; t < r; ++t) {
          cplx v = p[t * ld];
#pragma unroll
          for (int s = 0; s < NP; ++s) v = cfma(cs[s], pw[s * r + t], v);
          const double v2 = cabs2(v);
          rm = fmax(rm, v2);
          take(v2, rk + t);
        }
        bound = sqrt(rm);
      }
      bnd[l] = bound;
    }
    T2 = fmax(T2, bv);
  }
  Cand a{-1.0, LLONG_MAX, -1};
  if (bk != INT_MAX) a = Cand{bv, (long long)bk, bk / r - lo};
  return a;
}

// _swap_to_dominance (cross.py:122-139).  In global-slice mode the rank-1
// updates are deferred: up to g_lazy_f of them are folded into read-only row
// passes, and every g_lazy_f-th pass writes the slice back, which halves the
// slice traffic of most passes (the passes are HBM bound at full occupancy).
__device__ int swap_to_dominance_s(cg::cluster_group& cl, CC& c, int& par, double slack, long long limit) {
  const int r = c.r, lo = c.row0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  cplx* S = c.vec2;  // [0, r): B[i, :] before the update; [r, 2r): w (eager mode)
  const bool lazy = c.pend != nullptr;
  cplx* pw = lazy ? c.pend : S + r;      // pending w_s, s < np
  int* pj = lazy ? c.pendj : c.ibc + 8;  // pending j_s
  const int F = lazy ? max(1, min(LAZY_MAX, g_lazy_f)) : 1;
  int np = 0;  // updates not yet written to the slice
  const bool filter = lazy && g_swap_filter;
  bool bvalid = false;  // c.vn1 holds row bounds of the current B
  // global-slice mode: peers read winner rows straight from my slice, so no
  // CTA may rewrite its slice (form_B, a flushing pass) while a peer can
  // still be reading the previous winner row from it
  if (c.ns_global) cl.sync();
  invert_rows(c, c.sel);
  Cand a = form_B(c);
  int status = TTP_ERR_MAXVOL_ITER;
  SP_BEGIN(spt);
  for (long long it = 0;; ++it) {
    a = warp_cand(a);
    const Cand wb = a;  // this warp's best entry (the filtered pass re-evaluates it)
    __syncwarp();
    if (c.ns_global) {
      // global-slice mode: the winner's row is read straight from its
      // owner's slice after the barrier, so only the record is published
      WCand* slot = &c.wrec[par * CW + warp];
      if (lane == 0) {
        slot->v = a.v;
        slot->key = a.key;
        slot->row = a.row >= 0 ? lo + a.row : -1;
      }
    } else {
      warp_publish(c, par, a);
    }
    SP(spt, 8);
    cl.sync();
    SP(spt, 9);
    if (warp == 0) {
      const Winner W = warp_winner(cl, c, par);
      const int i = W.w.row;
      const int j = (int)(W.w.key - (long long)i * r);
      cplx x0, x1;
      if (c.ns_global) {
        const cplx* rowp = c.Ws + (long long)(W.rank - c.crank) * c.ldw * r + (i - W.rank * c.ldw);
        x0 = (lane < r) ? rowp[(long long)lane * c.ldw] : mk(0.0, 0.0);
        x1 = (lane + 32 < r) ? rowp[(long long)(lane + 32) * c.ldw] : mk(0.0, 0.0);
        // the pending updates, in order (the owner's row pass ran the same chain)
        for (int s = 0; s < np; ++s) {
          const cplx cv = lane_entry(x0, x1, pj[s]);
          if (lane < r) x0 = cfma(cv, pw[s * r + lane], x0);
          if (lane + 32 < r) x1 = cfma(cv, pw[s * r + lane + 32], x1);
        }
      } else {
        winner_row(cl, c, par, W, x0, x1);
      }
      const cplx pivot = lane_entry(x0, x1, j);
      // candidates are ranked by |b|^2; the stopping test uses |b| (hypot, as numpy abs)
      const int done = (cabsh(pivot) <= 1.0 + slack) ? 1 : 0;
      if (!done && it < limit) {
        // w[t] = (B[sel[j], t] - B[i, t]) / pivot: one fma per entry in the update
        cplx* w = pw + np * r;
        if (lane < r) {
          S[lane] = x0;
          w[lane] = cdiv(csub(c.selb[j * r + lane], x0), pivot);
        }
        if (lane + 32 < r) {
          S[lane + 32] = x1;
          w[lane + 32] = cdiv(csub(c.selb[j * r + lane + 32], x1), pivot);
        }
        if (lane == 0) pj[np] = j;
        if (filter) {
          // max_t |w[t]| for the filtered passes' bounds, rounded up
          double wm = 0.0;
          if (lane < r) wm = cabsh(w[lane]);
          if (lane + 32 < r) wm = fmax(wm, cabsh(w[lane + 32]));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) wm = fmax(wm, __shfl_xor_sync(0xffffffffu, wm, o));
          if (lane == 0) c.dbc[6] = wm * (1.0 + 1e-12);
        }
      }
      if (lane == 0) {
        c.ibc[4] = i;
        c.ibc[5] = j;
        c.ibc[6] = done;
      }
      SP(spt, 10);
    }
    __syncthreads();
    SP(spt, 11);
    const int i = c.ibc[4], j = c.ibc[5], done = c.ibc[6];
    if (it >= limit) break;  // guard exhausted (cross.py:127-139)
    if (done) {
      status = TTP_OK;
      break;
    }
    par ^= 1;
    const int nq = np + 1;
    const bool flush = nq >= F;
    const bool refresh = (it + 1) % 64 == 0;
    // this iteration rewrites the slice: every CTA must be done reading the
    // winner row first (the barrier latency overlaps the B[sel, :] update)
    const bool fence = c.ns_global && (flush || refresh);
    if (fence) cluster_arrive();
    const cplx* w = pw + np * r;
    // replicated B[sel, :]: rank-1 update of every row, row j <- updated B[i, :]
    for (int q = warp; q < r; q += CW) {
      const cplx bqj = (q == j) ? S[j] : c.selb[q * r + j];
      const cplx* base = (q == j) ? S : c.selb + q * r;
      cplx y0 = mk(0.0, 0.0), y1 = mk(0.0, 0.0);
      if (lane < r) y0 = cfma(bqj, w[lane], base[lane]);
      if (lane + 32 < r) y1 = cfma(bqj, w[lane + 32], base[lane + 32]);
      __syncwarp();
      if (lane < r) c.selb[q * r + lane] = y0;
      if (lane + 32 < r) c.selb[q * r + lane + 32] = y1;
    }
    if (threadIdx.x == 0) c.sel[j] = i;
    if (fence) cluster_wait();
    SP(spt, 12);
    const bool rev = g_serpentine && ((it & 1) == 0);
    if (filter && bvalid && !flush) {
      const double wmax = c.dbc[6];
      switch (nq) {
        case 1: a = swap_pass_filt<1>(c, pw, pj, wmax, wb, rev); break;
        case 2: a = swap_pass_filt<2>(c, pw, pj, wmax, wb, rev); break;
        case 3: a = swap_pass_filt<3>(c, pw, pj, wmax, wb, rev); break;
        default: a = swap_pass_filt<4>(c, pw, pj, wmax, wb, rev); break;
      }
    } else {
      // full pass; its row bounds are only used in global-slice mode (vn1 is
      // free during the swaps in every mode)
      switch (nq) {
        case 1: a = swap_pass<1, true>(c, pw, pj, flush, rev); break;
        case 2: a = swap_pass<2, true>(c, pw, pj, flush, rev); break;
        case 3: a = swap_pass<3, true>(c, pw, pj, flush, rev); break;
        default: a = swap_pass<4, true>(c, pw, pj, flush, rev); break;
      }
      bvalid = filter;
    }
    np = flush ? 0 : nq;
    SP(spt, 13);
    if (refresh) {
      __syncthreads();
      invert_rows(c, c.sel);
      a = form_B(c);
      np = 0;
      bvalid = false;
    }
  }
  par ^= 1;
  __syncthreads();
  if (status == TTP_OK && threadIdx.x == 0) insertion_sort(c.sel, r);
  __syncthreads();
  return status;
}

// _pairwise_refine (cross.py:147-169); only reached with C == 1 (m <= 96).
__device__ int pairwise_refine(cg::cluster_group& cl, CC& c, int& par, double slack, long long limit) {
  const int m = c.m, r = c.r;
  for (long long round = 0; round < limit; ++round) {
    const int st = swap_to_dominance_s(cl, c, par, slack, limit);
    if (st != TTP_OK) return st;
    invert_rows(c, c.sel);
    form_B(c);
    ArgMax a{-1.0, LLONG_MAX};
    const long long total = (long long)m * m * r * r;
    for (long long f = threadIdx.x; f < total; f += CT) {
      const int l2 = (int)(f % r);
      long long q = f / r;
      const int l1 = (int)(q % r);
      q /= r;
      const int i2 = (int)(q % m);
      const int i1 = (int)(q / m);
      const cplx v = csub(cmul(Wl(c, i1, l1), Wl(c, i2, l2)), cmul(Wl(c, i1, l2), Wl(c, i2, l1)));
      const double av = cabsh(v);
      if (argmax_better(av, f, a.v, a.key)) a = ArgMax{av, f};
    }
    Cand ca{a.v, a.key, 0};
    ca = block_cand(ca, c.wcand);
    if (ca.v <= 1.0 + 1e-9) return TTP_OK;
    if (threadIdx.x == 0) {
      const long long f = ca.key;
      const int j2 = (int)(f % r);
      long long q = f / r;
      const int j1 = (int)(q % r);
      q /= r;
      const int i2 = (int)(q % m);
      const int i1 = (int)(q / m);
      c.sel[j1] = i1;
      c.sel[j2] = i2;
    }
    __syncthreads();
  }
  return TTP_ERR_MAXVOL_ITER;
}

__global__ void __launch_bounds__(CT, CLUSTER_MIN_BLOCKS) cluster_bond_kernel(ClusterJob J) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  const BondJob& job = J.b;
  const int C = J.cl;
  const int inst = blockIdx.x / C;
  // cluster-uniform early exit
  if (job.active && !job.active[inst]) return;
  if (job.status[inst] != TTP_OK) return;
  CC c;
  c.m = job.m;
  c.r = job.r;
  c.C = C;
  c.crank = (int)cl.block_rank();
  const int ms = (job.m + C - 1) / C;
  c.row0 = c.crank * ms;
  c.nrows = max(0, min(job.m, c.row0 + ms) - c.row0);
  c.ldw = ms;
  c.Qg = J.Qg + inst * J.q_stride;
  carve(smem_raw, ms, job.r, &c, J.Wg != nullptr, J.big);
  if (J.Wg) c.Ws = J.Wg + inst * J.wg_stride + (long long)c.crank * ms * job.r;
  c.ns_global = J.Wg != nullptr;
  if (J.big & 1) {
    c.vn1 = job.dwork + inst * job.dw_stride + (long long)c.crank * 2 * ms;
    c.vn2 = c.vn1 + ms;
    c.rpos = job.iwork + inst * job.iw_stride + (long long)c.crank * 2 * ms;
    c.rpos2 = c.rpos + ms;
  }
  if (J.big & 2) c.selb = J.Sg + inst * J.wg_stride + (long long)c.crank * job.r * job.r;
  int par = 0;
  const int r = c.r, m = c.m;

  PHASE_MARK(0);
  INST_MARK(0);
  load_block(c, J, inst);
  PHASE_MARK(1);
  // the WY Q pass also leaves the fused starts' row norms (m > r only)
  const bool norms_in_q = J.q_wy != 0 && J.fused_starts != 0 && job.m != job.r;
  const bool basis_ok = tsqr_usable(c, J) ? tsqr_basis(cl, c, J, inst, job.rank_tol, norms_in_q)
                                           : column_basis(cl, c, par, job.rank_tol, J.q_wy != 0, J.fused_qr != 0, norms_in_q);
  if (!basis_ok) {
    if (c.crank == 0 && threadIdx.x == 0) set_error(job, inst, TTP_ERR_SINGULAR);
    cl.sync();
    return;
  }
  cl.sync();  // Q rows of every CTA are now visible in global memory
  if (J.basis_only) return;  // every CTA passed the barrier above
  if (m == r) {
    for (int t = threadIdx.x; t < r; t += CT) c.best[t] = t;
    __syncthreads();
  } else {
    PHASE_MARK(2);
    if (J.fused_starts) {
      start_pair_s(cl, c, par, norms_in_q);
      PHASE_MARK(3);
    } else {
      start_qrcp_qh_s(cl, c, par);
      PHASE_MARK(3);
      start_lu_s(cl, c, par);
    }
    PHASE_MARK(4);
    if (threadIdx.x == 0) {
      insertion_sort(c.starts, r);
      insertion_sort(c.starts + r, r);
      int same = 1;
      for (int t = 0; t < r; ++t) same &= (c.starts[t] == c.starts[r + t]);
      c.ibc[2] = same ? 1 : 2;
    }
    __syncthreads();
    const int nstart = c.ibc[2];
    const long long limit = job.max_iters >= 0 ? job.max_iters : 10LL * m;
    double best_vol = -INFINITY;
    bool have = false;
    int err = TTP_OK;
    for (int s = 0; s < nstart; ++s) {
      for (int t = threadIdx.x; t < r; t += CT) c.sel[t] = c.starts[s * r + t];
      __syncthreads();
      const int st = swap_to_dominance_s(cl, c, par, job.slack, limit);
      PHASE_MARK(5 + s);
      if (st != TTP_OK) {
        err = st;
        continue;
      }
      const double vol = invert_rows(c, c.sel);
      if (vol > best_vol) {
        best_vol = vol;
        have = true;
        for (int t = threadIdx.x; t < r; t += CT) c.best[t] = c.sel[t];
      }
      __syncthreads();
    }
    if (!have) {
      if (c.crank == 0 && threadIdx.x == 0) set_error(job, inst, err != TTP_OK ? err : TTP_ERR_SINGULAR);
      cl.sync();
      return;
    }
    if (job.pairwise && m <= 96 && r <= 8 && C == 1) {
      for (int t = threadIdx.x; t < r; t += CT) c.sel[t] = c.best[t];
      __syncthreads();
      const int st = pairwise_refine(cl, c, par, job.slack, limit);
      if (st != TTP_OK) {
        if (threadIdx.x == 0) set_error(job, inst, st);
        return;
      }
      for (int t = threadIdx.x; t < r; t += CT) c.best[t] = c.sel[t];
      __syncthreads();
    }
  }
  if (job.sel_out && c.crank == 0)
    for (int t = threadIdx.x; t < r; t += CT) job.sel_out[inst * job.sel_stride + t] = c.best[t];
  if (job.write_mode == 0) {
    cl.sync();
    return;
  }
  // phase E: factor with the conditioning check (cross.py:349-355)
  PHASE_MARK(7);
  invert_rows(c, c.best);
  {
    double fa = 0.0, fx = 0.0;
    if (threadIdx.x < 32) {
      for (int e = threadIdx.x; e < r * r; e += 32) {
        const int i = e / r, j = e - i * r;
        fa += cabs2(Qrow(c, c.best[i])[(long long)j * m]);
        fx += cabs2(c.aug[i * 2 * r + r + j]);
      }
      fa = warp_sum(fa);
      fx = warp_sum(fx);
      if (threadIdx.x == 0) c.dbc[1] = sqrt(fa) * sqrt(fx);
    }
    __syncthreads();
    if (!(c.dbc[1] <= 1e12)) {
      for (int e = threadIdx.x; e < r * r; e += CT) {
        const int i = e / r, j = e - i * r;
        c.aug[i * 2 * r + j] = Qrow(c, c.best[i])[(long long)j * m];
      }
      __syncthreads();
      if (threadIdx.x < 32) jacobi_cond_warp(c.aug, r, &c.dbc[2]);
      __syncthreads();
      if (!(c.dbc[2] <= 1e12)) {
        if (c.crank == 0 && threadIdx.x == 0) set_error(job, inst, TTP_ERR_SINGULAR);
        cl.sync();
        return;
      }
      invert_rows(c, c.best);
    }
  }
  cplx* core = job.core_out + inst * job.core_stride;
  const cplx* X = c.aug + r;
  if (c.qtile) {
    const int wm = job.write_mode;
    qx_dmma(c, X, 2 * r, [&](int l, int j, cplx v) {
      const int g = c.row0 + l;
      if (wm == 1) core[(long long)g * r + j] = v;
      else core[(long long)j * m + g] = v;
    });
  } else
  for (int l = threadIdx.x; l < c.nrows; l += CT) {
    const int g = c.row0 + l;
    const cplx* q = Qrow(c, g);
    for (int j0 = 0; j0 < r; j0 += 16) {
      cplx acc[16];
      rowblock_X<16>(q, m, X, 2 * r, j0, r, acc);
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int j = j0 + jj;
        if (j >= r) break;
        if (job.write_mode == 1) core[(long long)g * r + j] = acc[jj];
        else core[(long long)j * m + g] = acc[jj];
      }
    }
  }
  if (job.set_out && c.crank == 0) {
    const int d = job.set_d;
    for (int t = threadIdx.x; t < r; t += CT) {
      const int row = c.best[t];
      int* dst = job.set_out + inst * job.set_stride + job.set_out_off + (long long)t * d;
      if (job.write_mode == 1) {
        const int a = row / job.na, s = row - a * job.na;
        const int* src = job.set_in + inst * job.set_stride + job.set_in_off + (long long)a * d;
        for (int q = 0; q < job.klen - 1; ++q) dst[q] = src[q];
        dst[job.klen - 1] = s;
      } else {
        const int s = row / job.rr, b = row - s * job.rr;
        const int* src = job.set_in + inst * job.set_stride + job.set_in_off + (long long)b * d;
        dst[0] = s;
        for (int q = 1; q < job.klen; ++q) dst[q] = src[q - 1];
      }
    }
  }
  PHASE_MARK(8);
  INST_MARK(1);
  cl.sync();  // no CTA may exit while a peer can still read its shared memory
}

}  // namespace

namespace CK_NS {

int max_active_clusters_query(int C, size_t smem);

size_t cluster_smem_bytes(int m, int r, int C, bool global_slice, int big) {
  const int ms = (m + C - 1) / C;
  return carve(nullptr, ms, r, nullptr, global_slice, big);
}

static size_t cluster_smem_limit() {
  static std::mutex mu;
  static std::map<std::pair<int, int>, size_t> memo;
  return ttp_device_memo(memo, mu, 0, [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, (const void*)cluster_bond_kernel);
    return (size_t)v - fa.sharedSizeBytes;
  });
}

// Global-slice jobs move per-row state to global memory (the instance's
// dwork/iwork, B[sel,:] into the B buffer) until the carve fits the
// per-CTA budget of CLUSTER_MIN_BLOCKS resident CTAs per SM, or at least
// the opt-in limit of one.
static size_t cluster_smem_target() {
  static std::mutex mu;
  static std::map<std::pair<int, int>, size_t> memo;
  const size_t lim = cluster_smem_limit();
  return ttp_device_memo(memo, mu, 0, [lim] {
    int dev = 0, per_sm = 0, resv = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, (const void*)cluster_bond_kernel);
    const long long share = (long long)per_sm / CLUSTER_MIN_BLOCKS - resv - (long long)fa.sharedSizeBytes;
    return std::min(lim, (size_t)std::max(0LL, share));
  });
}

static void resolve_big(ClusterJob& job) {
  job.big = 0;
  if (!(job.Wg && job.Sg && job.b.dwork && job.b.iwork)) return;
  static const int forced = [] {  // TTP_BIG=0|1|3: A/B knob
    const char* e = ttp_dev_env("TTP_BIG");
    return e ? atoi(e) & 3 : -1;
  }();
  if (forced >= 0 && cluster_smem_bytes(job.b.m, job.b.r, job.cl, true, forced) <= cluster_smem_limit()) {
    job.big = forced;
    return;
  }
  // several CTAs per SM: the smallest carve (every byte of shared memory
  // taken from the unified L1 hurts the row passes); one: the largest
  const int order[3] = {CLUSTER_MIN_BLOCKS > 1 ? 3 : 0, 1, CLUSTER_MIN_BLOCKS > 1 ? 0 : 3};
  for (size_t lim : {cluster_smem_target(), cluster_smem_limit()})
    for (int b : order)
      if (cluster_smem_bytes(job.b.m, job.b.r, job.cl, true, b) <= lim) {
        job.big = b;
        return;
      }
  job.big = 3;
}

int pick_cluster_size(int m, int r, size_t smem_limit) {
  for (int C = 1; C <= 16; C *= 2) {
    const int ms = (m + C - 1) / C;
    if (C > 1 && ms < 1) break;
    if (cluster_smem_bytes(m, r, C) <= smem_limit) return C;
  }
  return 0;
}

// TTP_QFORM=zung2r selects the r-round reflector application (A/B checks);
// the default forms Q in compact-WY form.
static bool q_wy_enabled() {
  static const bool on = [] {
    const char* e = ttp_dev_env("TTP_QFORM");
    return !(e && strcmp(e, "zung2r") == 0);
  }();
  return on;
}

// TTP_STARTS=split runs the two starts as separate in-place factorizations.
static bool fused_starts_enabled() {
  static const bool on = [] {
    const char* e = ttp_dev_env("TTP_STARTS");
    return !(e && strcmp(e, "split") == 0);
  }();
  return on;
}

// TTP_TSQR=0 keeps the restated zlaqp2 column basis in global-slice mode
// (A/B knob); default: TSQR + zlaqp2 on the triangle (k_tsqr.cuh).
static bool tsqr_enabled() {
  static const bool on = [] {
    const char* e = ttp_dev_env("TTP_TSQR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// TTP_LAZY=F (1..LAZY_MAX): flush cadence of the deferred swap updates in
// global-slice mode (1 = the eager update of every row pass); A/B knob.
static cudaError_t apply_lazy_knob() {
#ifdef TTP_DEV
  static const cudaError_t st = [] {
    const char* e = ttp_dev_env("TTP_LAZY");
    if (!e) return cudaSuccess;
    const int f = std::max(1, std::min(LAZY_MAX, atoi(e)));
    return cudaMemcpyToSymbol(g_lazy_f, &f, sizeof(int));
  }();
  return st;
#else
  return cudaSuccess;
#endif
}

// TTP_SWAP_FILTER=0 runs every deferred swap pass over all rows (A/B knob);
// default: bound-filtered passes between the flushing ones.
static cudaError_t apply_swap_filter_knob() {
#ifdef TTP_DEV
  static const cudaError_t st = [] {
    const char* e = ttp_dev_env("TTP_SWAP_FILTER");
    if (!e) return cudaSuccess;
    const int f = e[0] == '0' ? 0 : 1;
    return cudaMemcpyToSymbol(g_swap_filter, &f, sizeof(int));
  }();
  return st;
#else
  return cudaSuccess;
#endif
}

// TTP_FUSED_QR=0 runs the column basis with a separate partials pass per
// step (A/B knob); default: each update pass also produces the next step's
// partials.
static bool fused_qr_enabled() {
  static const bool on = [] {
    const char* e = ttp_dev_env("TTP_FUSED_QR");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t launch_cluster_bond(const ClusterJob& job_in, int n_inst, cudaStream_t s) {
  ClusterJob job = job_in;
  job.fused_qr = fused_qr_enabled() ? 1 : 0;
  {
    cudaError_t e = apply_lazy_knob();
    if (e == cudaSuccess) e = apply_swap_filter_knob();
    if (e != cudaSuccess) return e;
  }
  resolve_big(job);
  job.q_wy = q_wy_enabled() ? 1 : 0;
  job.fused_starts = fused_starts_enabled() ? 1 : 0;
  job.tsqr = tsqr_enabled() ? 1 : 0;
  const int C = job.cl;
  const size_t smem = cluster_smem_bytes(job.b.m, job.b.r, C, job.Wg != nullptr, job.big);
  cudaError_t e = ensure_max_smem((const void*)cluster_bond_kernel);
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(cluster_bond_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_inst * C));
  cfg.blockDim = dim3(CT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  {
    LaunchScope _ls(KC_CLUSTER_BOND, s);
    e = cudaLaunchKernelEx(&cfg, cluster_bond_kernel, job);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int max_active_clusters(const ClusterJob& job_in) {
  ClusterJob job = job_in;
  resolve_big(job);
  const int C = job.cl;
  const size_t smem = cluster_smem_bytes(job.b.m, job.b.r, C, job.Wg != nullptr, job.big);
  if (smem > cluster_smem_limit()) return 0;
  static std::mutex mu;
  static std::map<std::pair<int, std::pair<int, size_t>>, int> cache;
  return ttp_device_memo(cache, mu, std::make_pair(C, smem), [&] { return max_active_clusters_query(C, smem); });
}

int max_active_clusters_query(int C, size_t smem) {
  if (ensure_max_smem((const void*)cluster_bond_kernel) != cudaSuccess) return 0;
  if (C > 8 && cudaFuncSetAttribute(cluster_bond_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * 64));
  cfg.blockDim = dim3(CT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, cluster_bond_kernel, &cfg) != cudaSuccess) return 0;
  // The occupancy calculator assumes one CTA per SM for kernels that
  // allocate tensor memory (measured: tools/micro/tmem_occ.cu reports 1
  // block/SM while the hardware keeps two 256-column CTAs resident).  Scale
  // its answer by the residency the registers, shared memory, threads and
  // TMEM columns (TW_NCOLS per CTA of 512) actually allow.
  int api = 0, dev = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&api, cluster_bond_kernel, CT, smem) != cudaSuccess || api <= 0)
    return n;
  cudaFuncAttributes fa{};
  int regs_sm = 0, smem_sm = 0, thr_sm = 0, resv = 0;
  cudaGetDevice(&dev);
  cudaFuncGetAttributes(&fa, (const void*)cluster_bond_kernel);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
  cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
  int bps = std::min(thr_sm / CT, regs_sm / std::max(1, regs_warp * CW));
  bps = std::min(bps, (int)(smem_sm / std::max<size_t>(1, smem + fa.sharedSizeBytes + resv)));
  bps = std::min(bps, 512 / TW_NCOLS);
  return bps > api ? n * bps / api : n;
}

#ifdef TTP_DEV
// Phase clocks of this instantiation: out[0..16) phase marks, out[16..32)
// sub-phase accumulators; enable also clears both.
int debug_phase_clocks(int enable, int64_t* out, int32_t n) {
  const int en = enable ? 1 : 0;
  if (out && n > 0) {
    long long tmp[32];
    if (cudaMemcpyFromSymbol(tmp, g_phase_clock, 16 * sizeof(long long)) != cudaSuccess) return TTP_ERR_CUDA;
    if (cudaMemcpyFromSymbol(tmp + 16, g_sub_clock, 16 * sizeof(long long)) != cudaSuccess) return TTP_ERR_CUDA;
    for (int i = 0; i < n && i < 32; ++i) out[i] = tmp[i];
  }
  if (en) {
    unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(g_sub_clock, z, sizeof(z)) != cudaSuccess) return TTP_ERR_CUDA;
    if (cudaMemcpyToSymbol(g_phase_clock, z, sizeof(z)) != cudaSuccess) return TTP_ERR_CUDA;
  }
  if (cudaMemcpyToSymbol(g_phase_enable, &en, sizeof(int)) != cudaSuccess) return TTP_ERR_CUDA;
  return TTP_OK;
}

// Per-instance [start, end, sm] of the last enabled launches (n instances).
int debug_inst_times(int64_t* out, int32_t n) {
  n = std::min(n, INST_T_MAX);
  for (int k = 0; k < 3; ++k)
    if (cudaMemcpyFromSymbol(out + (size_t)k * n, g_inst_t, sizeof(long long) * n, sizeof(long long) * k * INST_T_MAX) !=
        cudaSuccess)
      return TTP_ERR_CUDA;
  return TTP_OK;
}

#endif

}  // namespace CK_NS
