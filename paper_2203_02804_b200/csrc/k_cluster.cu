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
// Phases per bond (reference decision order, as in k_bond_v0.cu):
//   0  fibers: the oracle is evaluated straight into shared memory (no HBM
//      round trip for the sampled block; pricers.py:234-253 via cross.py:310-332)
//   A  zgeqp3 (zlaqp2: pivot, zlarfg, zlarf, partial-norm downdate/recompute)
//      + zung2r, distributed: 1 round per step (+1 when a norm recompute fires)
//      -> orthonormal Q (written once to global, L2-resident)       cross.py:103-119
//   B  start 1: zlaqp2 on Q^H (right-looking, reflectors of length r)  cross.py:184-185
//   C  start 2: zgetrf partial pivoting (|Re|+|Im|)                  cross.py:186-187
//   D  _swap_to_dominance from each start; every CTA keeps a replicated
//      copy of B[sel, :] so the rank-1 update needs only the winning row,
//      which travels with the argmax record                        cross.py:122-139
//   E  slogdet choice, cond screen, factor Q Q[sel]^-1 -> TT core     cross.py:191-205,349-355
#include <cooperative_groups.h>

#include <map>
#include <mutex>

#include "ttp_internal.h"
#include "bond_common.cuh"
#include "k_bond.h"
#include "launch.h"

namespace cg = cooperative_groups;

// Phase clocks of instance 0 / cluster rank 0 (diagnostic; ttp_debug_phase_clocks).
__device__ long long g_phase_clock[16];
__device__ int g_phase_enable;
#define PHASE_MARK(k)                                                           \
  do {                                                                          \
    if (g_phase_enable && inst == 0 && c.crank == 0 && threadIdx.x == 0)        \
      g_phase_clock[k] = clock64();                                             \
  } while (0)

// Sub-phase cycle accumulators (cluster rank 0, thread 0 of instance 0).
__device__ unsigned long long g_sub_clock[8];
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

namespace {

constexpr int CT = CLUSTER_THREADS;
constexpr int CW = CT / 32;
constexpr int RMAX = 64;

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
  Cand* wcand;     // CW
  Ssq* wss;        // CW
  int* ibc;        // 8
  double* dbc;     // 8
  cplx* cbc;       // 8
};

__device__ __forceinline__ cplx& Wl(const CC& c, int l, int t) { return c.Ws[(long long)t * c.ldw + l]; }
__device__ __forceinline__ const cplx* Qrow(const CC& c, int g) { return c.Qg + g; }  // stride m

__host__ __device__ size_t carve(unsigned char* base, int ldw, int r, CC* c) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* p = base ? base + off : nullptr;
    off += (bytes + 15) & ~(size_t)15;
    return p;
  };
  CC t;
  t.Ws = (cplx*)take(sizeof(cplx) * (size_t)ldw * r);
  t.aug = (cplx*)take(sizeof(cplx) * 2 * r * r);
  t.selb = (cplx*)take(sizeof(cplx) * r * r);
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
  t.vn1 = (double*)take(sizeof(double) * ldw);
  t.vn2 = (double*)take(sizeof(double) * ldw);
  t.rpos = (int*)take(sizeof(int) * ldw);
  t.rec = (Rec*)take(sizeof(Rec) * 2);
  t.wcand = (Cand*)take(sizeof(Cand) * CW);
  t.wss = (Ssq*)take(sizeof(Ssq) * CW);
  t.ibc = (int*)take(sizeof(int) * 8);
  t.dbc = (double*)take(sizeof(double) * 8);
  t.cbc = (cplx*)take(sizeof(cplx) * 8);
  if (c) {
    c->Ws = t.Ws; c->aug = t.aug; c->selb = t.selb; c->vec = t.vec; c->vec2 = t.vec2;
    c->tau = t.tau; c->betas = t.betas; c->cn1 = t.cn1; c->cn2 = t.cn2; c->colmap = t.colmap;
    c->flags = t.flags; c->first = t.first; c->sel = t.sel; c->best = t.best; c->starts = t.starts;
    c->vn1 = t.vn1; c->vn2 = t.vn2; c->rpos = t.rpos; c->rec = t.rec; c->wcand = t.wcand;
    c->wss = t.wss; c->ibc = t.ibc; c->dbc = t.dbc; c->cbc = t.cbc;
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
  if (J.src_mode == 0) {
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

// ------------------------------------------------------------ phase A
// Distributed zlaqp2 + zung2r on the block.  Returns false (cluster-uniform)
// when the block is zero / rank deficient by rank_tol.
__device__ bool column_basis(cg::cluster_group& cl, CC& c, int& par, double rank_tol) {
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
    for (int j = warp; j < r; j += CW) {
      const double nrm = ssq_norm(rank_ssq(cl, c, par, j));
      if (lane == 0) {
        c.cn1[j] = nrm;
        c.cn2[j] = nrm;
        c.colmap[j] = j;
      }
    }
    par ^= 1;
    __syncthreads();
  }
  SP_BEGIN(spt);
  for (int i = 0; i < r; ++i) {
    if (threadIdx.x == 0) {
      int p = i;
      for (int j = i + 1; j < r; ++j)
        if (c.cn1[j] > c.cn1[p]) p = j;
      if (p != i) {
        const int t = c.colmap[p];
        c.colmap[p] = c.colmap[i];
        c.colmap[i] = t;
        c.cn1[p] = c.cn1[i];
        c.cn2[p] = c.cn2[i];
      }
    }
    __syncthreads();
    SP(spt, 0);
    const int ci = c.colmap[i];
    const bool own_i = (i >= lo && i < lo + nl);
    const int li = i - lo;
    const int lstart = max(0, i + 1 - lo);  // first local row with global index > i
    const int ntr = r - i - 1;
    Rec* me = &c.rec[par];
    // partials: task 0 = Ssq of x, task q>=1 = conj(x) . column (i+q)
    for (int q = warp; q <= ntr; q += CW) {
      if (q == 0) {
        const int f0 = lstart + lane;
        Ssq s = ssq_of(&c.Ws[(long long)ci * c.ldw + f0], 32, nl > f0 ? (nl - f0 + 31) / 32 : 0);
        s = warp_ssq(s);
        if (lane == 0) {
          me->data[0] = mk(s.scale, s.ssq);
          me->data[1] = own_i ? Wl(c, li, ci) : mk(0.0, 0.0);
        }
      } else {
        const int cj = c.colmap[i + q];
        cplx acc = mk(0.0, 0.0);
        for (int l = lstart + lane; l < nl; l += 32) acc = cfmac(Wl(c, l, ci), Wl(c, l, cj), acc);
        acc = warp_sum(acc);
        if (lane == 0) {
          me->data[1 + q] = acc;
          me->data[1 + r + q] = own_i ? Wl(c, li, cj) : mk(0.0, 0.0);
        }
      }
    }
    SP(spt, 1);
    cl.sync();
    SP(spt, 2);
    // cross-rank reductions, one warp per item (identical in every CTA)
    for (int q = warp; q <= ntr; q += CW) {
      if (q == 0) {
        const Ssq s = rank_ssq(cl, c, par, 0);
        const cplx alpha = rank_sum(cl, c, par, 1);
        if (lane == 0) {
          Reflector h = zlarfg_core(alpha, ssq_norm(s));
          c.tau[i] = h.tau;
          c.betas[i] = fabs(h.beta);
          c.cbc[0] = reflector_scale(h);
          c.dbc[0] = h.beta;
        }
      } else {
        const cplx dq = rank_sum(cl, c, par, 1 + q);
        const cplx aq = rank_sum(cl, c, par, 1 + r + q);
        if (lane == 0) {
          c.vec[q - 1] = dq;
          c.vec2[q - 1] = aq;
        }
      }
    }
    __syncthreads();
    const cplx tau = c.tau[i];
    const bool ident = is_zero(tau);
    const cplx scal = c.cbc[0];
    for (int q = 1 + (int)threadIdx.x; q <= ntr; q += CT) {
      const cplx dots = c.vec[q - 1], arow = c.vec2[q - 1];
      // v = [1; x*scal]:  s_j = A[i,j] + conj(scal) * (x^H A[:,j])
      const cplx sj = cadd(arow, cmulc(scal, dots));
      const cplx tj = ident ? mk(0.0, 0.0) : cmul(cconj(tau), sj);
      c.vec[q - 1] = tj;
      const cplx newrow = csub(arow, tj);
      c.vec2[q - 1] = newrow;
      // zlaqp2 partial column-norm downdate (replicated)
      const int j = i + q;
      int flag = 0;
      const double v1 = c.cn1[j];
      if (v1 != 0.0) {
        double temp = cabsh(newrow) / v1;
        temp = fmax(1.0 - temp * temp, 0.0);
        const double rq = v1 / c.cn2[j];
        if (temp * rq * rq <= TOL3Z) flag = 1;
        else c.cn1[j] = v1 * sqrt(temp);
      }
      c.flags[q - 1] = flag;
    }
    par ^= 1;
    __syncthreads();
    SP(spt, 3);
    // local update of my rows
    for (int l = threadIdx.x; l < nl; l += CT) {
      const int g = lo + l;
      if (g < i) continue;
      if (g == i) {
        Wl(c, l, ci) = mk(c.dbc[0], 0.0);
        for (int q = 1; q <= ntr; ++q) Wl(c, l, c.colmap[i + q]) = c.vec2[q - 1];
      } else if (!ident) {
        const cplx x = cmul(Wl(c, l, ci), scal);
        Wl(c, l, ci) = x;
        for (int q = 1; q <= ntr; ++q) {
          cplx& a = Wl(c, l, c.colmap[i + q]);
          a = csub(a, cmul(x, c.vec[q - 1]));
        }
      }
    }
    __syncthreads();
    SP(spt, 4);
    // norm recompute round (only if some column flagged; replicated decision)
    int anyflag = 0;
    for (int q = 0; q < ntr; ++q) anyflag |= c.flags[q];
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
          const double nrm = (i < m - 1) ? ssq_norm(s) : 0.0;
          c.cn1[i + 1 + q] = nrm;
          c.cn2[i + 1 + q] = nrm;
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
        for (int l = lstart + lane; l < nl; l += 32) acc = cfmac(Wl(c, l, ci), Wl(c, l, cj), acc);
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
      for (int l = threadIdx.x; l < nl; l += CT) {
        const int g = lo + l;
        if (g < i) continue;
        const cplx v = (g == i) ? mk(1.0, 0.0) : Wl(c, l, ci);
        for (int q = 0; q < ntr; ++q) {
          cplx& a = Wl(c, l, c.colmap[i + 1 + q]);
          a = csub(a, cmul(v, c.vec[q]));
        }
      }
      __syncthreads();
    }
    const cplx mt = cneg(ti);
    for (int l = threadIdx.x; l < nl; l += CT) {
      const int g = lo + l;
      cplx& a = Wl(c, l, ci);
      if (g > i) a = cmul(a, mt);
      else if (g == i) a = mk(1.0 - ti.x, -ti.y);
      else a = mk(0.0, 0.0);
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

// ------------------------------------------------------------ phase B
__device__ void start_qrcp_qh(cg::cluster_group& cl, CC& c, int& par) {
  const int r = c.r, lo = c.row0, nl = c.nrows;
  for (int l = threadIdx.x; l < nl; l += CT) {
    for (int t = 0; t < r; ++t) Wl(c, l, t) = cconj(Qrow(c, lo + l)[(long long)t * c.m]);
    const double nrm = ssq_norm(ssq_of(&Wl(c, l, 0), c.ldw, r));
    c.vn1[l] = nrm;
    c.vn2[l] = nrm;
    c.rpos[l] = lo + l;
  }
  for (int t = threadIdx.x; t < r; t += CT) c.first[t] = t;
  __syncthreads();
  for (int i = 0; i < r; ++i) {
    Cand a{-1.0, LLONG_MAX, -1};
    for (int l = threadIdx.x; l < nl; l += CT)
      if (c.rpos[l] >= i) {
        Cand b{c.vn1[l], c.rpos[l], l};
        if (cand_better(b, a)) a = b;
      }
    a = block_cand(a, c.wcand);
    Rec* me = &c.rec[par];
    if (threadIdx.x == 0) {
      me->v = a.v;
      me->key = a.key;
      me->row = a.row >= 0 ? lo + a.row : -1;
    }
    if (a.row >= 0)
      for (int t = threadIdx.x; t < r; t += CT) me->data[t] = Wl(c, a.row, t);
    cl.sync();
    int wr;
    const Cand w = cluster_winner(cl, c, par, &wr);
    const Rec* wrec = cl.map_shared_rank(&c.rec[par], wr);
    if (threadIdx.x < 32) {
      // winner's column of Q^H (rows i..r-1) -> reflector, one warp
      const int ln = threadIdx.x;
      cplx x0 = mk(0.0, 0.0), x1 = mk(0.0, 0.0);
      const int t0 = i + 1 + ln, t1 = i + 33 + ln;
      Ssq s = ssq_init();
      if (t0 < r) {
        x0 = wrec->data[t0];
        ssq_addc(s, x0);
      }
      if (t1 < r) {
        x1 = wrec->data[t1];
        ssq_addc(s, x1);
      }
      s = warp_ssq(s);
      const cplx alpha = wrec->data[i];
      Reflector h = zlarfg_core(alpha, ssq_norm(s));
      const cplx sc = reflector_scale(h);
      const bool ident = is_zero(h.tau);
      if (t0 < r) c.vec2[t0] = ident ? x0 : cmul(x0, sc);
      if (t1 < r) c.vec2[t1] = ident ? x1 : cmul(x1, sc);
      if (ln == 0) {
        c.vec2[i] = mk(1.0, 0.0);
        c.cbc[0] = h.tau;
        const int B = w.row, pvt = (int)w.key;
        const int A = c.first[i];
        c.first[i] = B;
        if (pvt < r) c.first[pvt] = A;
        if (A >= lo && A < lo + nl) c.rpos[A - lo] = pvt;
        if (B >= lo && B < lo + nl) c.rpos[B - lo] = i;
      }
    }
    __syncthreads();
    par ^= 1;
    const cplx tc = cconj(c.cbc[0]);
    const bool last = (i == r - 1);
    for (int l = threadIdx.x; l < nl; l += CT) {
      if (c.rpos[l] <= i) continue;
      cplx sacc = mk(0.0, 0.0);
      for (int t = i; t < r; ++t) sacc = cfmac(c.vec2[t], Wl(c, l, t), sacc);
      const cplx tt = cmul(tc, sacc);
      for (int t = i; t < r; ++t) Wl(c, l, t) = csub(Wl(c, l, t), cmul(c.vec2[t], tt));
      const double v1 = c.vn1[l];
      if (v1 != 0.0) {
        double temp = cabsh(Wl(c, l, i)) / v1;
        temp = fmax(1.0 - temp * temp, 0.0);
        const double q = v1 / c.vn2[l];
        if (temp * q * q <= TOL3Z) {
          double nrm = 0.0;
          if (!last) nrm = ssq_norm(ssq_of(&Wl(c, l, i + 1), c.ldw, r - i - 1));
          c.vn1[l] = nrm;
          c.vn2[l] = nrm;
        } else {
          c.vn1[l] = v1 * sqrt(temp);
        }
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < r; t += CT) c.starts[t] = c.first[t];
  __syncthreads();
}

// ------------------------------------------------------------ phase C
__device__ void start_lu(cg::cluster_group& cl, CC& c, int& par) {
  const int r = c.r, lo = c.row0, nl = c.nrows;
  Cand a{-1.0, LLONG_MAX, -1};
  for (int l = threadIdx.x; l < nl; l += CT) {
    for (int t = 0; t < r; ++t) Wl(c, l, t) = Qrow(c, lo + l)[(long long)t * c.m];
    c.rpos[l] = lo + l;
    Cand b{cabs1(Wl(c, l, 0)), lo + l, l};
    if (cand_better(b, a)) a = b;
  }
  for (int t = threadIdx.x; t < r; t += CT) c.first[t] = t;
  for (int k = 0; k < r; ++k) {
    a = block_cand(a, c.wcand);
    Rec* me = &c.rec[par];
    if (threadIdx.x == 0) {
      me->v = a.v;
      me->key = a.key;
      me->row = a.row >= 0 ? lo + a.row : -1;
    }
    if (a.row >= 0)
      for (int t = threadIdx.x; t < r; t += CT) me->data[t] = Wl(c, a.row, t);
    cl.sync();
    int wr;
    const Cand w = cluster_winner(cl, c, par, &wr);
    const Rec* wrec = cl.map_shared_rank(&c.rec[par], wr);
    for (int t = threadIdx.x; t < r; t += CT) c.vec[t] = wrec->data[t];
    __syncthreads();
    if (threadIdx.x == 0) {
      const int B = w.row, pvt = (int)w.key;
      const int A = c.first[k];
      c.first[k] = B;
      if (pvt < r) c.first[pvt] = A;
      if (A >= lo && A < lo + nl) c.rpos[A - lo] = pvt;
      if (B >= lo && B < lo + nl) c.rpos[B - lo] = k;
    }
    __syncthreads();
    par ^= 1;
    const cplx piv = c.vec[k];
    const bool nz = !is_zero(piv);
    const cplx rp = nz ? cdiv(mk(1.0, 0.0), piv) : mk(0.0, 0.0);
    a = Cand{-1.0, LLONG_MAX, -1};
    for (int l = threadIdx.x; l < nl; l += CT) {
      const int p = c.rpos[l];
      if (p <= k) continue;
      if (nz) {
        const cplx mult = cmul(Wl(c, l, k), rp);
        Wl(c, l, k) = mult;
        for (int t = k + 1; t < r; ++t) Wl(c, l, t) = csub(Wl(c, l, t), cmul(mult, c.vec[t]));
      }
      if (k + 1 < r) {
        Cand b{cabs1(Wl(c, l, k + 1)), p, l};
        if (cand_better(b, a)) a = b;
      }
    }
  }
  for (int t = threadIdx.x; t < r; t += CT) c.starts[r + t] = c.first[t];
  __syncthreads();
}

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

// B = Q X for my rows (into Ws) and for the selected rows (selb); returns my
// best |B| candidate (key = global row-major index).
__device__ Cand form_B(const CC& c) {
  const int r = c.r, lo = c.row0, nl = c.nrows, ld = 2 * r;
  const cplx* X = c.aug + r;
  Cand a{-1.0, LLONG_MAX, -1};
  constexpr int JB = 16;
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

__device__ int swap_to_dominance(cg::cluster_group& cl, CC& c, int& par, double slack, long long limit) {
  const int r = c.r, lo = c.row0, nl = c.nrows;
  invert_rows(c, c.sel);
  Cand a = form_B(c);
  int status = TTP_ERR_MAXVOL_ITER;
  for (long long it = 0;; ++it) {
    a = block_cand(a, c.wcand);
    Rec* me = &c.rec[par];
    if (threadIdx.x == 0) {
      me->v = a.v;
      me->key = a.key;
      me->row = a.row >= 0 ? lo + a.row : -1;
    }
    if (a.row >= 0)
      for (int t = threadIdx.x; t < r; t += CT) me->data[t] = Wl(c, a.row, t);
    cl.sync();
    int wr;
    const Cand w = cluster_winner(cl, c, par, &wr);
    if (it >= limit) break;  // guard exhausted (cross.py:127-139)
    const Rec* wrec = cl.map_shared_rank(&c.rec[par], wr);
    const int i = (int)(w.key / r), j = (int)(w.key - (long long)(w.key / r) * r);
    for (int t = threadIdx.x; t < r; t += CT) c.vec2[t] = wrec->data[t];  // B[i, :] before the update
    __syncthreads();
    const cplx pivot = c.vec2[j];
    // candidates are ranked by |b|^2; the stopping test uses |b| (numpy abs = hypot)
    if (cabsh(pivot) <= 1.0 + slack) {
      status = TTP_OK;
      break;
    }
    // w[t] = (B[sel[j], t] - B[i, t]) / pivot, so the update is one fma per entry
    for (int t = threadIdx.x; t < r; t += CT) c.vec[t] = cdiv(csub(c.selb[j * r + t], c.vec2[t]), pivot);
    __syncthreads();
    par ^= 1;
    a = Cand{-1.0, LLONG_MAX, -1};
    for (int l = threadIdx.x; l < nl; l += CT) {
      const cplx blj = Wl(c, l, j);
      for (int t = 0; t < r; ++t) {
        const cplx v = cfma(blj, c.vec[t], Wl(c, l, t));
        Wl(c, l, t) = v;
        Cand b{cabs2(v), (long long)(lo + l) * r + t, l};
        if (cand_better(b, a)) a = b;
      }
    }
    // replicated B[sel, :]: rank-1 update of every row, then row j <- new B[i, :]
    for (int q = threadIdx.x; q < r; q += CT) {
      const cplx bqj = c.selb[q * r + j];
      for (int t = 0; t < r; ++t) c.selb[q * r + t] = cfma(bqj, c.vec[t], c.selb[q * r + t]);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < r; t += CT) c.selb[j * r + t] = cfma(c.vec2[j], c.vec[t], c.vec2[t]);
    if (threadIdx.x == 0) c.sel[j] = i;
    __syncthreads();
    if ((it + 1) % 64 == 0) {
      invert_rows(c, c.sel);
      a = form_B(c);
    }
  }
  par ^= 1;
  if (status == TTP_OK && threadIdx.x == 0) insertion_sort(c.sel, r);
  __syncthreads();
  return status;
}

// _pairwise_refine (cross.py:147-169); only reached with C == 1 (m <= 96).
__device__ int pairwise_refine(cg::cluster_group& cl, CC& c, int& par, double slack, long long limit) {
  const int m = c.m, r = c.r;
  for (long long round = 0; round < limit; ++round) {
    const int st = swap_to_dominance(cl, c, par, slack, limit);
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

__global__ void __launch_bounds__(CT, 1) cluster_bond_kernel(ClusterJob J) {
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
  carve(smem_raw, ms, job.r, &c);
  int par = 0;
  const int r = c.r, m = c.m;

  PHASE_MARK(0);
  load_block(c, J, inst);
  PHASE_MARK(1);
  if (!column_basis(cl, c, par, job.rank_tol)) {
    if (c.crank == 0 && threadIdx.x == 0) set_error(job, inst, TTP_ERR_SINGULAR);
    cl.sync();
    return;
  }
  cl.sync();  // Q rows of every CTA are now visible in global memory
  if (m == r) {
    for (int t = threadIdx.x; t < r; t += CT) c.best[t] = t;
    __syncthreads();
  } else {
    PHASE_MARK(2);
    start_qrcp_qh(cl, c, par);
    PHASE_MARK(3);
    start_lu(cl, c, par);
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
      const int st = swap_to_dominance(cl, c, par, job.slack, limit);
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
  cl.sync();  // no CTA may exit while a peer can still read its shared memory
}

}  // namespace

int max_active_clusters_query(int C, size_t smem);

size_t cluster_smem_bytes(int m, int r, int C) {
  const int ms = (m + C - 1) / C;
  return carve(nullptr, ms, r, nullptr);
}

int pick_cluster_size(int m, int r, size_t smem_limit) {
  for (int C = 1; C <= 16; C *= 2) {
    const int ms = (m + C - 1) / C;
    if (C > 1 && ms < 1) break;
    if (cluster_smem_bytes(m, r, C) <= smem_limit) return C;
  }
  return 0;
}

cudaError_t launch_cluster_bond(const ClusterJob& job, int n_inst, cudaStream_t s) {
  const int C = job.cl;
  const size_t smem = cluster_smem_bytes(job.b.m, job.b.r, C);
  cudaError_t e = cudaFuncSetAttribute(cluster_bond_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
    LaunchScope _ls(KC_BOND, s);
    e = cudaLaunchKernelEx(&cfg, cluster_bond_kernel, job);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int max_active_clusters(const ClusterJob& job) {
  const int C = job.cl;
  const size_t smem = cluster_smem_bytes(job.b.m, job.b.r, C);
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, int> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({C, smem});
    if (it != cache.end()) return it->second;
  }
  const int n = max_active_clusters_query(C, smem);
  std::lock_guard<std::mutex> lk(mu);
  cache[{C, smem}] = n;
  return n;
}

int max_active_clusters_query(int C, size_t smem) {
  if (cudaFuncSetAttribute(cluster_bond_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
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
  return n;
}

extern "C" int ttp_debug_phase_clocks(int enable, int64_t* out, int32_t n) {
  const int en = enable ? 1 : 0;
  if (out && n > 0) {
    long long tmp[24];
    if (cudaMemcpyFromSymbol(tmp, g_phase_clock, 16 * sizeof(long long)) != cudaSuccess) return TTP_ERR_CUDA;
    if (cudaMemcpyFromSymbol(tmp + 16, g_sub_clock, 8 * sizeof(long long)) != cudaSuccess) return TTP_ERR_CUDA;
    for (int i = 0; i < n && i < 24; ++i) out[i] = tmp[i];
  }
  if (en) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(g_sub_clock, z, sizeof(z)) != cudaSuccess) return TTP_ERR_CUDA;
  }
  if (cudaMemcpyToSymbol(g_phase_enable, &en, sizeof(int)) != cudaSuccess) return TTP_ERR_CUDA;
  return TTP_OK;
}
