// K3-K5: the per-bond linear algebra of TT-cross, one CTA per instance.
//
// For every sampled unfolding block M (m x r, m >= r) this kernel performs,
// entirely on the device and in the reference's decision order:
//   1. column basis:   zgeqp3 (unblocked zlaqp2) + zung2r   (_column_basis,
//                      cross.py:103-119; scipy.linalg.qr(pivoting=True))
//   2. maxvol starts:  first r pivots of QRCP(Q^H)           (cross.py:184-185)
//                      partial-pivot LU rows, |Re|+|Im| rule (cross.py:186-187)
//   3. swaps:          B = Q Q[sel]^-1, argmax |B| (first in row-major order),
//                      rank-1 updates, refresh every 64      (cross.py:122-139)
//   4. best start by slogdet, strict >                       (cross.py:191-202)
//   5. pairwise refine for m <= 96, r <= 8                   (cross.py:147-169)
//   6. cond2(Q[sel]) <= 1e12 check, factor Q Q[sel]^-1      (cross.py:349-355)
// and writes the factor straight into the TT core layout.
//
// Layout: M / W / B are column-major (ld = m) complex128 in global memory;
// a warp covers 32 consecutive rows so every column access coalesces.
// Row-parallel phases (LU, QRCP of Q^H, swaps) keep physical rows in place
// and track LAPACK's row/column interchanges through pos2row/row2pos, so
// "first maximum" tie-breaks follow the reference's scan order exactly.
// All reductions are fixed-order (warp xor trees + ordered warp merge).
//
// Compiled twice with different CTA shapes (V0_NS / V0_THREADS /
// V0_MIN_BLOCKS set by the including .cu): 512 threads x 2 CTAs per SM for
// blocks of more than 64 KB (k_bond_v0.cu) and 128 threads x 8 CTAs per SM
// for smaller ones (k_bond_v0_small.cu); launch_bond in k_bond_v0.cu picks by
// the block shape alone, so results do not depend on the batch.  Measured on
// configs 1-3 (profiles/r02/s4/ab_v0_shape.log).
#include "ttp_internal.h"
#include "bond_common.cuh"
#include "launch.h"
#include "k_bond.h"

#include <float.h>
#include <limits.h>

#if !defined(V0_NS) || !defined(V0_THREADS) || !defined(V0_MIN_BLOCKS)
#error "define V0_NS, V0_THREADS and V0_MIN_BLOCKS before including k_bond_v0_impl.cuh"
#endif

namespace {

constexpr int NT = V0_THREADS;
constexpr int NW = NT / 32;

struct Ctx {
  int m, r;
  cplx* A;  // sampled block -> Q (physical column colmap[t] holds Q[:, t])
  cplx* W;  // working copy
  cplx* B;  // maxvol interpolation matrix
  int* pos2row;
  int* row2pos;
  double* vn1;
  double* vn2;
  // shared memory
  cplx* aug;   // r x 2r augmented matrix (Gauss-Jordan)
  cplx* vec;   // r
  cplx* rowv;  // r
  cplx* tau;   // r
  double* cn1; // r
  double* cn2; // r
  double* betas;  // r
  int* colmap;  // r
  int* sel;     // r
  int* best;    // r
  int* starts;  // 2r
  ArgMax* red;  // NW
  Ssq* rss;     // NW
  cplx* rc;     // NW
  int* ibc;     // small int broadcast area (8)
  double* dbc;  // small double broadcast area (8)
  cplx* cbc;    // small complex broadcast area (8)
};

__device__ __forceinline__ cplx& Qat(const Ctx& c, int l, int t) {
  return c.A[(long long)c.colmap[t] * c.m + l];
}
__device__ __forceinline__ cplx& Wat(const Ctx& c, int l, int t) { return c.W[(long long)t * c.m + l]; }
__device__ __forceinline__ cplx& Bat(const Ctx& c, int l, int t) { return c.B[(long long)t * c.m + l]; }

// ------------------------------------------------------ block reductions
__device__ ArgMax block_argmax(ArgMax a, ArgMax* red) {
  a = warp_argmax(a);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  ArgMax b = red[0];
  for (int w = 1; w < NW; ++w)
    if (argmax_better(red[w].v, red[w].key, b.v, b.key)) b = red[w];
  return b;
}

__device__ Ssq block_ssq(Ssq s, Ssq* red) {
  s = warp_ssq(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  Ssq b = red[0];
  for (int w = 1; w < NW; ++w) b = ssq_merge(b, red[w]);
  return b;
}

// ------------------------------------------- small dense LA in shared memory
__device__ double gauss_jordan(const Ctx& c, int r) { return ::gauss_jordan<NT>(c.aug, r, c.vec, c.ibc); }

// aug <- [Q[rows] | I] with Q in logical column order.
__device__ void load_aug_from_Q(const Ctx& c, const int* rows) {
  const int r = c.r, ld = 2 * r;
  for (int e = threadIdx.x; e < r * ld; e += NT) {
    const int i = e / ld, j = e - i * ld;
    c.aug[e] = (j < r) ? Qat(c, rows[i], j) : mk((j - r == i) ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
}

// Running argmax of |z| (numpy abs = hypot, first maximum) with a squared-
// modulus screen: hypot is only evaluated when z2 = re^2 + im^2 comes within
// rounding of the running best's.  Below that, hypot(z) < a.v strictly (both
// are accurate to an ulp and the margin is ~50 ulp), so the (value, key)
// winner is bitwise the unscreened one; ties and non-finite values take the
// exact path.  a2: squared modulus of a's entry, -1 before the first.
__device__ __forceinline__ void argmax_abs_update(cplx z, long long key, ArgMax& a, double& a2) {
  const double z2 = fma(z.x, z.x, z.y * z.y);
  if (z2 >= a2 * (1.0 - 1e-14)) {
    const double v = cabsh(z);
    if (argmax_better(v, key, a.v, a.key)) {
      a = ArgMax{v, key};
      a2 = z2;
    }
  }
}

// B = Q X with X = right half of aug; returns the block argmax of |B|
// (key = row-major flat index, numpy argmax order).
__device__ ArgMax form_B(const Ctx& c) {
  const int m = c.m, r = c.r, ld = 2 * r;
  ArgMax a{-1.0, LLONG_MAX};
  double a2 = -1.0;
  for (int l = threadIdx.x; l < m; l += NT) {
    for (int j = 0; j < r; ++j) {
      cplx acc = mk(0.0, 0.0);
      for (int t = 0; t < r; ++t) acc = cfma(Qat(c, l, t), c.aug[t * ld + r + j], acc);
      Bat(c, l, j) = acc;
      argmax_abs_update(acc, (long long)l * r + j, a, a2);
    }
  }
  return block_argmax(a, c.red);
}

// ------------------------------------------------------------ phase 1 + 2
// zgeqp3 (unblocked zlaqp2 path; r <= 64 <= nx) on the block, then zung2r.
// Returns the R diagonal moduli in betas[] (for the rank check).
__device__ void column_basis(const Ctx& c) {
  const int m = c.m, r = c.r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  cplx* A = c.A;
  // initial column norms
  for (int j = warp; j < r; j += NW) {
    Ssq s = ssq_init();
    for (int l = lane; l < m; l += 32) ssq_addc(s, A[(long long)j * m + l]);
    s = warp_ssq(s);
    if (lane == 0) {
      const double nrm = ssq_norm(s);
      c.cn1[j] = nrm;
      c.cn2[j] = nrm;
      c.colmap[j] = j;
    }
  }
  __syncthreads();
  const int mn = min(m, r);
  for (int i = 0; i < mn; ++i) {
    if (threadIdx.x == 0) {
      int p = i;
      for (int j = i + 1; j < r; ++j)
        if (c.cn1[j] > c.cn1[p]) p = j;  // idamax: first maximum
      if (p != i) {
        const int t = c.colmap[p];
        c.colmap[p] = c.colmap[i];
        c.colmap[i] = t;
        c.cn1[p] = c.cn1[i];
        c.cn2[p] = c.cn2[i];
      }
    }
    __syncthreads();
    cplx* col = A + (long long)c.colmap[i] * m;
    // xnorm over rows i+1..m-1
    Ssq s = ssq_init();
    for (int l = i + 1 + threadIdx.x; l < m; l += NT) ssq_addc(s, col[l]);
    s = block_ssq(s, c.rss);
    if (threadIdx.x == 0) {
      Reflector h = zlarfg_core(col[i], ssq_norm(s));
      c.tau[i] = h.tau;
      c.betas[i] = fabs(h.beta);
      c.cbc[0] = h.scal;
      c.ibc[1] = h.knt;
      c.dbc[0] = h.beta;
    }
    __syncthreads();
    {
      cplx scal = c.cbc[0];
      const int knt = c.ibc[1];
      for (int q = 0; q < knt; ++q) scal = cscale(scal, 1.0 / SAFMIN_RFG);
      if (!(c.tau[i].x == 0.0 && c.tau[i].y == 0.0))
        for (int l = i + 1 + threadIdx.x; l < m; l += NT) col[l] = cmul(col[l], scal);
    }
    __syncthreads();
    if (threadIdx.x == 0) col[i] = mk(c.dbc[0], 0.0);
    __syncthreads();
    // apply H(i)^H = I - conj(tau) v v^H to trailing columns; update norms
    const cplx tc = cconj(c.tau[i]);
    for (int j = i + 1 + warp; j < r; j += NW) {
      cplx* cj = A + (long long)c.colmap[j] * m;
      cplx sacc = mk(0.0, 0.0);
      if (lane == 0) sacc = cj[i];  // v_i = 1
#pragma unroll 4
      for (int l = i + 1 + lane; l < m; l += 32) sacc = cfmac(col[l], cj[l], sacc);
      sacc = warp_sum(sacc);
      const cplx t = cmul(tc, sacc);
      if (lane == 0) cj[i] = csub(cj[i], t);
#pragma unroll 4
      for (int l = i + 1 + lane; l < m; l += 32) cj[l] = csub(cj[l], cmul(col[l], t));
      __syncwarp();
      // zlaqp2 partial column norm update
      double v1 = c.cn1[j];
      if (v1 != 0.0) {
        double temp = cabsh(cj[i]) / v1;
        temp = 1.0 - temp * temp;
        temp = fmax(temp, 0.0);
        const double q = v1 / c.cn2[j];
        const double temp2 = temp * q * q;
        if (temp2 <= TOL3Z) {
          double nrm = 0.0;
          if (i < m - 1) {
            Ssq s2 = ssq_init();
            for (int l = i + 1 + lane; l < m; l += 32) ssq_addc(s2, cj[l]);
            s2 = warp_ssq(s2);
            nrm = ssq_norm(s2);
          }
          if (lane == 0) {
            c.cn1[j] = nrm;
            c.cn2[j] = nrm;
          }
        } else if (lane == 0) {
          c.cn1[j] = v1 * sqrt(temp);
        }
      }
    }
    __syncthreads();
  }
  // zung2r: Q = H(0) ... H(r-1) [I; 0], in place
  for (int i = r - 1; i >= 0; --i) {
    cplx* col = A + (long long)c.colmap[i] * m;
    const cplx ti = c.tau[i];
    for (int j = i + 1 + warp; j < r; j += NW) {
      cplx* cj = A + (long long)c.colmap[j] * m;
      cplx sacc = mk(0.0, 0.0);
      if (lane == 0) sacc = cj[i];
#pragma unroll 4
      for (int l = i + 1 + lane; l < m; l += 32) sacc = cfmac(col[l], cj[l], sacc);
      sacc = warp_sum(sacc);
      const cplx t = cmul(ti, sacc);
      if (lane == 0) cj[i] = csub(cj[i], t);
#pragma unroll 4
      for (int l = i + 1 + lane; l < m; l += 32) cj[l] = csub(cj[l], cmul(col[l], t));
    }
    __syncthreads();
    const cplx mt = cneg(ti);
    for (int l = threadIdx.x; l < m; l += NT) {
      if (l > i) col[l] = cmul(col[l], mt);
      else if (l == i) col[l] = mk(1.0 - ti.x, -ti.y);
      else col[l] = mk(0.0, 0.0);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ phase 2a
// First r pivots of zgeqp3 on Q^H (r x m): W[l, t] holds column l of the
// working Q^H.  Result: c.starts[0..r-1] (unsorted pivot rows).
__device__ void start_qrcp_qh(const Ctx& c) {
  const int m = c.m, r = c.r;
  for (int l = threadIdx.x; l < m; l += NT) {
    Ssq s = ssq_init();
    for (int t = 0; t < r; ++t) {
      const cplx q = cconj(Qat(c, l, t));
      Wat(c, l, t) = q;
      ssq_addc(s, q);
    }
    const double nrm = ssq_norm(s);
    c.vn1[l] = nrm;
    c.vn2[l] = nrm;
    c.pos2row[l] = l;
    c.row2pos[l] = l;
  }
  __syncthreads();
  for (int i = 0; i < r; ++i) {
    ArgMax a{-1.0, LLONG_MAX};
    for (int l = threadIdx.x; l < m; l += NT) {
      const int p = c.row2pos[l];
      if (p >= i && argmax_better(c.vn1[l], p, a.v, a.key)) a = ArgMax{c.vn1[l], p};
    }
    a = block_argmax(a, c.red);
    if (threadIdx.x == 0) {
      const int p = (int)a.key;
      const int ri = c.pos2row[i], rp = c.pos2row[p];
      c.pos2row[i] = rp;
      c.pos2row[p] = ri;
      c.row2pos[rp] = i;
      c.row2pos[ri] = p;
      c.starts[i] = rp;
    }
    __syncthreads();
    const int lp = c.starts[i];
    // reflector from column lp, rows i..r-1 of Q^H (one warp)
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      Ssq s = ssq_init();
      for (int t = i + 1 + lane; t < r; t += 32) ssq_addc(s, Wat(c, lp, t));
      s = warp_ssq(s);
      const cplx alpha = Wat(c, lp, i);
      Reflector h = zlarfg_core(alpha, ssq_norm(s));
      cplx scal = h.scal;
      for (int q = 0; q < h.knt; ++q) scal = cscale(scal, 1.0 / SAFMIN_RFG);
      const bool ident = (h.tau.x == 0.0 && h.tau.y == 0.0);
      for (int t = i + 1 + lane; t < r; t += 32)
        c.vec[t] = ident ? Wat(c, lp, t) : cmul(Wat(c, lp, t), scal);
      if (lane == 0) {
        c.vec[i] = mk(1.0, 0.0);
        c.cbc[0] = h.tau;
      }
    }
    __syncthreads();
    const cplx tc = cconj(c.cbc[0]);
    const bool last = (i == r - 1);
    for (int l = threadIdx.x; l < m; l += NT) {
      if (c.row2pos[l] <= i) continue;
      cplx sacc = mk(0.0, 0.0);
      for (int t = i; t < r; ++t) sacc = cfmac(c.vec[t], Wat(c, l, t), sacc);
      const cplx tt = cmul(tc, sacc);
      for (int t = i; t < r; ++t) Wat(c, l, t) = csub(Wat(c, l, t), cmul(c.vec[t], tt));
      double v1 = c.vn1[l];
      if (v1 != 0.0) {
        double temp = cabsh(Wat(c, l, i)) / v1;
        temp = 1.0 - temp * temp;
        temp = fmax(temp, 0.0);
        const double q = v1 / c.vn2[l];
        const double temp2 = temp * q * q;
        if (temp2 <= TOL3Z) {
          double nrm = 0.0;
          if (!last) {
            Ssq s = ssq_init();
            for (int t = i + 1; t < r; ++t) ssq_addc(s, Wat(c, l, t));
            nrm = ssq_norm(s);
          }
          c.vn1[l] = nrm;
          c.vn2[l] = nrm;
        } else {
          c.vn1[l] = v1 * sqrt(temp);
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ phase 2b
// zgetrf partial pivoting on a copy of Q; result c.starts[r..2r-1].
__device__ void start_lu(const Ctx& c) {
  const int m = c.m, r = c.r;
  ArgMax a{-1.0, LLONG_MAX};
  for (int l = threadIdx.x; l < m; l += NT) {
    for (int t = 0; t < r; ++t) Wat(c, l, t) = Qat(c, l, t);
    c.pos2row[l] = l;
    c.row2pos[l] = l;
    const double v = cabs1(Wat(c, l, 0));
    if (argmax_better(v, l, a.v, a.key)) a = ArgMax{v, l};
  }
  for (int k = 0; k < r; ++k) {
    a = block_argmax(a, c.red);
    if (threadIdx.x == 0) {
      const int p = (int)a.key;
      const int rk = c.pos2row[k], rp = c.pos2row[p];
      c.pos2row[k] = rp;
      c.pos2row[p] = rk;
      c.row2pos[rp] = k;
      c.row2pos[rk] = p;
      c.starts[r + k] = rp;
    }
    __syncthreads();
    const int lp = c.starts[r + k];
    const cplx piv = Wat(c, lp, k);
    const bool nz = (piv.x != 0.0 || piv.y != 0.0);
    const cplx rp = nz ? cdiv(mk(1.0, 0.0), piv) : mk(0.0, 0.0);
    a = ArgMax{-1.0, LLONG_MAX};
    for (int l = threadIdx.x; l < m; l += NT) {
      const int p = c.row2pos[l];
      if (p <= k) continue;
      if (nz) {
        const cplx mult = cmul(Wat(c, l, k), rp);
        Wat(c, l, k) = mult;
        for (int t = k + 1; t < r; ++t) Wat(c, l, t) = csub(Wat(c, l, t), cmul(mult, Wat(c, lp, t)));
      }
      if (k + 1 < r) {
        const double v = cabs1(Wat(c, l, k + 1));
        if (argmax_better(v, p, a.v, a.key)) a = ArgMax{v, p};
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ phase 3
// _swap_to_dominance from the selection in c.sel (r rows).  Returns TTP_OK
// (c.sel sorted ascending) or TTP_ERR_MAXVOL_ITER.
__device__ int swap_to_dominance(const Ctx& c, double slack, long long limit) {
  const int m = c.m, r = c.r;
  load_aug_from_Q(c, c.sel);
  gauss_jordan(c, r);
  ArgMax a = form_B(c);
  int status = TTP_ERR_MAXVOL_ITER;
  for (long long it = 0; it < limit; ++it) {
    if (a.v <= 1.0 + slack) {
      status = TTP_OK;
      break;
    }
    const int i = (int)(a.key / r), j = (int)(a.key - (long long)(a.key / r) * r);
    const int sj = c.sel[j];
    const cplx pivot = Bat(c, i, j);
    for (int t = threadIdx.x; t < r; t += NT) c.vec[t] = csub(Bat(c, sj, t), Bat(c, i, t));
    __syncthreads();
    a = ArgMax{-1.0, LLONG_MAX};
    double a2 = -1.0;
    for (int l = threadIdx.x; l < m; l += NT) {
      const cplx blj = Bat(c, l, j);
      for (int t = 0; t < r; ++t) {
        const cplx nv = cadd(Bat(c, l, t), cdiv(cmul(blj, c.vec[t]), pivot));
        Bat(c, l, t) = nv;
        argmax_abs_update(nv, (long long)l * r + t, a, a2);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) c.sel[j] = i;
    __syncthreads();
    if ((it + 1) % 64 == 0) {
      load_aug_from_Q(c, c.sel);
      gauss_jordan(c, r);
      a = form_B(c);
    } else {
      a = block_argmax(a, c.red);
    }
  }
  if (status == TTP_OK && threadIdx.x == 0) {
    // insertion sort (r <= 64)
    for (int p = 1; p < r; ++p) {
      const int v = c.sel[p];
      int q = p - 1;
      while (q >= 0 && c.sel[q] > v) {
        c.sel[q + 1] = c.sel[q];
        --q;
      }
      c.sel[q + 1] = v;
    }
  }
  __syncthreads();
  return status;
}

// _pairwise_refine (cross.py:147-169): only for m <= 96, r <= 8.
__device__ int pairwise_refine(const Ctx& c, double slack, long long swap_limit, long long limit) {
  const int m = c.m, r = c.r;
  for (long long round = 0; round < limit; ++round) {
    int st = swap_to_dominance(c, slack, swap_limit);
    if (st != TTP_OK) return st;
    load_aug_from_Q(c, c.sel);
    gauss_jordan(c, r);
    form_B(c);
    __syncthreads();
    ArgMax a{-1.0, LLONG_MAX};
    const long long total = (long long)m * m * r * r;
    for (long long f = threadIdx.x; f < total; f += NT) {
      const int l2 = (int)(f % r);
      long long q = f / r;
      const int l1 = (int)(q % r);
      q /= r;
      const int i2 = (int)(q % m);
      const int i1 = (int)(q / m);
      const cplx v = csub(cmul(Bat(c, i1, l1), Bat(c, i2, l2)), cmul(Bat(c, i1, l2), Bat(c, i2, l1)));
      const double av = cabsh(v);
      if (argmax_better(av, f, a.v, a.key)) a = ArgMax{av, f};
    }
    a = block_argmax(a, c.red);
    if (a.v <= 1.0 + 1e-9) return TTP_OK;
    if (threadIdx.x == 0) {
      const long long f = a.key;
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

__device__ double jacobi_cond(const Ctx& c) {
  __shared__ double res;
  if (threadIdx.x < 32) jacobi_cond_warp(c.aug, c.r, &res);
  __syncthreads();
  return res;
}

__device__ void set_error(const BondJob& job, int inst, int code) {
  job.status[inst] = code;
  if (job.err_bond) job.err_bond[inst] = job.bond;
}

__global__ void __launch_bounds__(NT, V0_MIN_BLOCKS) bond_kernel(BondJob job) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int inst = blockIdx.x;
  if (job.active && !job.active[inst]) return;
  if (job.status[inst] != TTP_OK) return;
  const int m = job.m, r = job.r;
  Ctx c;
  c.m = m;
  c.r = r;
  c.A = job.A + inst * job.mat_stride;
  c.W = job.W + inst * job.mat_stride;
  c.B = job.B + inst * job.mat_stride;
  c.pos2row = job.iwork + inst * job.iw_stride;
  c.row2pos = c.pos2row + m;
  c.vn1 = job.dwork + inst * job.dw_stride;
  c.vn2 = c.vn1 + m;
  unsigned char* p = smem_raw;
  auto take = [&](size_t bytes) {
    unsigned char* q = p;
    p += (bytes + 15) & ~(size_t)15;
    return q;
  };
  c.aug = (cplx*)take(sizeof(cplx) * 2 * r * r);
  c.vec = (cplx*)take(sizeof(cplx) * r);
  c.rowv = (cplx*)take(sizeof(cplx) * r);
  c.tau = (cplx*)take(sizeof(cplx) * r);
  c.cn1 = (double*)take(sizeof(double) * r);
  c.cn2 = (double*)take(sizeof(double) * r);
  c.betas = (double*)take(sizeof(double) * r);
  c.colmap = (int*)take(sizeof(int) * r);
  c.sel = (int*)take(sizeof(int) * r);
  c.best = (int*)take(sizeof(int) * r);
  c.starts = (int*)take(sizeof(int) * 2 * r);
  c.red = (ArgMax*)take(sizeof(ArgMax) * NW);
  c.rss = (Ssq*)take(sizeof(Ssq) * NW);
  c.rc = (cplx*)take(sizeof(cplx) * NW);
  c.ibc = (int*)take(sizeof(int) * 8);
  c.dbc = (double*)take(sizeof(double) * 8);
  c.cbc = (cplx*)take(sizeof(cplx) * 8);

  // 1. column basis with rank check
  column_basis(c);
  {
    double lead = 0.0, mn = INFINITY;
    for (int t = 0; t < r; ++t) {
      lead = fmax(lead, c.betas[t]);
      mn = fmin(mn, c.betas[t]);
    }
    if (lead == 0.0 || mn < job.rank_tol * lead) {
      if (threadIdx.x == 0) set_error(job, inst, TTP_ERR_SINGULAR);
      return;
    }
  }
  // 2-5. maxvol row selection (_dominant_rows, cross.py:172-205)
  if (m == r) {
    for (int t = threadIdx.x; t < r; t += NT) c.best[t] = t;
    __syncthreads();
  } else {
    start_qrcp_qh(c);
    start_lu(c);
    if (threadIdx.x == 0) {
      // sort both starts; drop the LU start if identical (cross.py:188-189)
      for (int s = 0; s < 2; ++s) {
        int* v = c.starts + s * r;
        for (int q1 = 1; q1 < r; ++q1) {
          const int x = v[q1];
          int q = q1 - 1;
          while (q >= 0 && v[q] > x) {
            v[q + 1] = v[q];
            --q;
          }
          v[q + 1] = x;
        }
      }
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
      for (int t = threadIdx.x; t < r; t += NT) c.sel[t] = c.starts[s * r + t];
      __syncthreads();
      const int st = swap_to_dominance(c, job.slack, limit);
      if (st != TTP_OK) {
        err = st;
        continue;
      }
      load_aug_from_Q(c, c.sel);
      const double vol = gauss_jordan(c, r);
      // strict '>' keeps the first start on ties; a singular start
      // (slogdet = -inf) is never kept, as in the reference.
      if (vol > best_vol) {
        best_vol = vol;
        have = true;
        for (int t = threadIdx.x; t < r; t += NT) c.best[t] = c.sel[t];
      }
      __syncthreads();
    }
    if (!have) {
      if (threadIdx.x == 0) set_error(job, inst, (err != TTP_OK) ? err : TTP_ERR_SINGULAR);
      return;
    }
    if (job.pairwise && m <= 96 && r <= 8) {
      for (int t = threadIdx.x; t < r; t += NT) c.sel[t] = c.best[t];
      __syncthreads();
      const int st = pairwise_refine(c, job.slack, limit, limit);
      if (st != TTP_OK) {
        if (threadIdx.x == 0) set_error(job, inst, st);
        return;
      }
      for (int t = threadIdx.x; t < r; t += NT) c.best[t] = c.sel[t];
      __syncthreads();
    }
  }
  // output selection
  if (job.sel_out)
    for (int t = threadIdx.x; t < r; t += NT) job.sel_out[inst * job.sel_stride + t] = c.best[t];
  if (job.write_mode == 0) return;
  // 6. interpolation factor with the conditioning check (cross.py:349-355)
  load_aug_from_Q(c, c.best);
  gauss_jordan(c, r);
  {
    double fa = 0.0, fx = 0.0;
    for (int e = threadIdx.x; e < r * r; e += NT) {
      const int i = e / r, j = e - i * r;
      fa += cabs2(Qat(c, c.best[i], j));
      fx += cabs2(c.aug[i * 2 * r + r + j]);
    }
    fa = warp_sum(fa);
    fx = warp_sum(fx);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      c.rc[threadIdx.x >> 5] = mk(fa, fx);
    }
    __syncthreads();
    double ta = 0.0, tx = 0.0;
    for (int w = 0; w < NW; ++w) {
      ta += c.rc[w].x;
      tx += c.rc[w].y;
    }
    const double screen = sqrt(ta) * sqrt(tx);
    if (!(screen <= 1e12)) {
      // exact cond2 on a fresh copy (the inverse in the right half is kept)
      for (int e = threadIdx.x; e < r * r; e += NT) {
        const int i = e / r, j = e - i * r;
        c.aug[i * 2 * r + j] = Qat(c, c.best[i], j);
      }
      __syncthreads();
      const double cond = jacobi_cond(c);
      if (!(cond <= 1e12)) {
        if (threadIdx.x == 0) set_error(job, inst, TTP_ERR_SINGULAR);
        return;
      }
      load_aug_from_Q(c, c.best);
      gauss_jordan(c, r);
    }
  }
  // factor = Q X written in the TT core layout
  cplx* core = job.core_out + inst * job.core_stride;
  for (int l = threadIdx.x; l < m; l += NT) {
    for (int j = 0; j < r; ++j) {
      cplx acc = mk(0.0, 0.0);
      for (int t = 0; t < r; ++t) acc = cfma(Qat(c, l, t), c.aug[t * 2 * r + r + j], acc);
      if (job.write_mode == 1)
        core[(long long)l * r + j] = acc;  // cores[k-1] = factor.reshape(...)
      else
        core[(long long)j * m + l] = acc;  // cores[k] = factor.T.reshape(...)
    }
  }
  // new nested index set
  if (job.set_out) {
    const int d = job.set_d;
    for (int t = threadIdx.x; t < r; t += NT) {
      const int row = c.best[t];
      int* dst = job.set_out + inst * job.set_stride + job.set_out_off + (long long)t * d;
      if (job.write_mode == 1) {
        // left[k][t] = left[k-1][row / na] ++ (row % na)
        const int a = row / job.na, s = row - a * job.na;
        const int* src = job.set_in + inst * job.set_stride + job.set_in_off + (long long)a * d;
        for (int q = 0; q < job.klen - 1; ++q) dst[q] = src[q];
        dst[job.klen - 1] = s;
      } else {
        // right[k][t] = (row / rr,) ++ right[k+1][row % rr]
        const int s = row / job.rr, b = row - s * job.rr;
        const int* src = job.set_in + inst * job.set_stride + job.set_in_off + (long long)b * d;
        dst[0] = s;
        for (int q = 1; q < job.klen; ++q) dst[q] = src[q - 1];
      }
    }
  }
}

}  // namespace

namespace V0_NS {

size_t bond_smem_bytes(int r) {
  auto al = [](size_t b) { return (b + 15) & ~(size_t)15; };
  size_t s = 0;
  s += al(sizeof(cplx) * 2 * r * r);
  s += 3 * al(sizeof(cplx) * r);
  s += 3 * al(sizeof(double) * r);
  s += 3 * al(sizeof(int) * r) + al(sizeof(int) * 2 * r);
  s += al(sizeof(ArgMax) * NW) + al(sizeof(Ssq) * NW) + al(sizeof(cplx) * NW);
  s += al(sizeof(int) * 8) + al(sizeof(double) * 8) + al(sizeof(cplx) * 8);
  return s;
}

cudaError_t launch_bond(const BondJob& job, int n_inst, cudaStream_t s) {
  const size_t smem = bond_smem_bytes(job.r);
  cudaError_t e = ensure_max_smem((const void*)bond_kernel);
  if (e != cudaSuccess) return e;
  {
    LaunchScope _ls(KC_BOND, s);
    bond_kernel<<<n_inst, NT, smem, s>>>(job);
  }
  return cudaGetLastError();
}

}  // namespace V0_NS
