// Device helpers shared by the bond kernels (k_bond.cu: one CTA per
// instance, global-memory working set; k_cluster.cu: one thread-block
// cluster per instance, shared-memory working set).
#pragma once

#include <limits.h>

#include "ttp_common.cuh"

constexpr double TOL3Z = 1.0536712127723509e-08;         // sqrt(dlamch('E')), eps = 2^-53
constexpr double SAFMIN_RFG = 2.0041683600089728e-292;   // dlamch('S') / dlamch('E')

__device__ __forceinline__ double dlapy3(double x, double y, double z) {
  const double xa = fabs(x), ya = fabs(y), za = fabs(z);
  const double w = fmax(xa, fmax(ya, za));
  if (w == 0.0) return xa + ya + za;
  return w * sqrt((xa / w) * (xa / w) + (ya / w) * (ya / w) + (za / w) * (za / w));
}

// LAPACK zlarfg on (alpha, x) given xnorm = ||x||: H = I - tau v v^H with
// v = [1; x * scal_total], H^H [alpha; x] = [beta; 0], beta real.
// scal_total = scal * rsafmn^knt (the safmin rescaling loop of zlarfg).
struct Reflector {
  cplx tau;
  double beta;
  cplx scal;
  int knt;
};

__device__ __forceinline__ Reflector zlarfg_core(cplx alpha, double xnorm) {
  Reflector h;
  h.knt = 0;
  double alphr = alpha.x, alphi = alpha.y;
  if (xnorm == 0.0 && alphi == 0.0) {
    h.tau = mk(0.0, 0.0);
    h.beta = alphr;
    h.scal = mk(1.0, 0.0);
    return h;
  }
  double beta = -copysign(dlapy3(alphr, alphi, xnorm), alphr);
  const double rsafmn = 1.0 / SAFMIN_RFG;
  while (fabs(beta) < SAFMIN_RFG && h.knt < 20) {
    ++h.knt;
    beta *= rsafmn;
    alphi *= rsafmn;
    alphr *= rsafmn;
    xnorm *= rsafmn;
  }
  if (h.knt > 0) beta = -copysign(dlapy3(alphr, alphi, xnorm), alphr);
  h.tau = mk((beta - alphr) / beta, -alphi / beta);
  h.scal = cdiv(mk(1.0, 0.0), mk(alphr - beta, alphi));
  for (int j = 0; j < h.knt; ++j) beta *= SAFMIN_RFG;
  h.beta = beta;
  return h;
}

// zlarfg from the SQUARED norm of x with one sqrt and two divisions (the
// LAPACK routine uses dlapy3 + four divisions); falls back to zlarfg_core
// when any intermediate could leave the safe exponent range.  Same
// reflector up to rounding.
__device__ __forceinline__ Reflector zlarfg_fast(cplx alpha, double xnorm2) {
  const double a2 = alpha.x * alpha.x + alpha.y * alpha.y;
  const double t2 = a2 + xnorm2;
  if (!(t2 > 1e-280 && t2 < 1e280) || (xnorm2 == 0.0 && alpha.y == 0.0))
    return zlarfg_core(alpha, sqrt(xnorm2));
  Reflector h;
  h.knt = 0;
  const double beta = -copysign(sqrt(t2), alpha.x);
  const double ib = 1.0 / beta;
  h.tau = mk((beta - alpha.x) * ib, -alpha.y * ib);
  const double dr = alpha.x - beta;
  const double id = 1.0 / (dr * dr + alpha.y * alpha.y);
  h.scal = mk(dr * id, -alpha.y * id);
  h.beta = beta;
  return h;
}

__device__ __forceinline__ cplx reflector_scale(const Reflector& h) {
  cplx s = h.scal;
  for (int q = 0; q < h.knt; ++q) s = cscale(s, 1.0 / SAFMIN_RFG);
  return s;
}

__device__ __forceinline__ bool is_zero(cplx z) { return z.x == 0.0 && z.y == 0.0; }

// Gauss-Jordan with LAPACK's partial pivoting rule (izamax: |Re|+|Im|, first
// maximum) on M = [S | I] (r x 2r, row stride 2r) in shared memory, all NT
// threads cooperating.  On return the right half holds S^-1; returns
// log|det S| (numpy slogdet's logabsdet; -inf when singular), identical in
// every thread.  colbuf: r complex scratch, ibc: 1 int scratch.
template <int NT>
__device__ double gauss_jordan(cplx* M, int r, cplx* colbuf, int* ibc) {
  const int ld = 2 * r;
  double logdet = 0.0;
  for (int k = 0; k < r; ++k) {
    if (threadIdx.x < 32) {
      ArgMax a{-1.0, LLONG_MAX};
      for (int i = k + (int)threadIdx.x; i < r; i += 32) {
        const double v = cabs1(M[i * ld + k]);
        if (argmax_better(v, i, a.v, a.key)) a = ArgMax{v, i};
      }
      a = warp_argmax(a);
      if (threadIdx.x == 0) *ibc = (int)a.key;
    }
    __syncthreads();
    const int p = *ibc;
    if (p != k) {
      for (int j = threadIdx.x; j < ld; j += NT) {
        const cplx t = M[k * ld + j];
        M[k * ld + j] = M[p * ld + j];
        M[p * ld + j] = t;
      }
    }
    __syncthreads();
    const cplx piv = M[k * ld + k];
    const double apiv = cabsh(piv);
    logdet += log(apiv);
    if (apiv == 0.0) {
      __syncthreads();
      continue;
    }
    const cplx rp = cdiv(mk(1.0, 0.0), piv);
    for (int i = threadIdx.x; i < r; i += NT) colbuf[i] = (i == k) ? mk(0.0, 0.0) : M[i * ld + k];
    __syncthreads();
    for (int j = threadIdx.x; j < ld; j += NT) M[k * ld + j] = cmul(M[k * ld + j], rp);
    __syncthreads();
    for (int e = threadIdx.x; e < r * ld; e += NT) {
      const int i = e / ld, j = e - i * ld;
      if (i != k) M[e] = csub(M[e], cmul(colbuf[i], M[k * ld + j]));
    }
    __syncthreads();
  }
  return logdet;
}

// Same result as gauss_jordan (same pivots, same arithmetic per entry) with
// three barriers per column instead of five: the pivot row is scaled into a
// scratch copy and the interchange is folded into the elimination pass.
// scratch: 5r complex (scaled pivot row 2r, old row k 2r, multipliers r).
template <int NT>
__device__ double gauss_jordan_fast(cplx* M, int r, cplx* scratch, int* ibc) {
  const int ld = 2 * r;
  cplx* prow = scratch;
  cplx* oldk = scratch + ld;
  cplx* colb = scratch + 2 * ld;
  double logdet = 0.0;
  for (int k = 0; k < r; ++k) {
    __syncthreads();
    if (threadIdx.x < 32) {
      ArgMax a{-1.0, LLONG_MAX};
      for (int i = k + (int)threadIdx.x; i < r; i += 32) {
        const double v = cabs1(M[i * ld + k]);
        if (argmax_better(v, i, a.v, a.key)) a = ArgMax{v, i};
      }
      a = warp_argmax(a);
      if (threadIdx.x == 0) *ibc = (int)a.key;
    }
    __syncthreads();
    const int p = *ibc;
    const cplx piv = M[p * ld + k];
    const double apiv = cabsh(piv);
    logdet += log(apiv);
    if (apiv == 0.0) {
      // singular: still perform the interchange so later columns see LAPACK's order
      for (int j = threadIdx.x; j < ld; j += NT) oldk[j] = M[k * ld + j];
      __syncthreads();
      if (p != k)
        for (int j = threadIdx.x; j < ld; j += NT) {
          const cplx t = M[p * ld + j];
          M[k * ld + j] = t;
          M[p * ld + j] = oldk[j];
        }
      continue;
    }
    const cplx rp = cdiv(mk(1.0, 0.0), piv);
    for (int j = threadIdx.x; j < ld; j += NT) {
      prow[j] = cmul(M[p * ld + j], rp);
      oldk[j] = M[k * ld + j];
    }
    for (int i = threadIdx.x; i < r; i += NT)
      colb[i] = (i == k) ? mk(0.0, 0.0) : ((i == p) ? M[k * ld + k] : M[i * ld + k]);
    __syncthreads();
    for (int e = threadIdx.x; e < r * ld; e += NT) {
      const int i = e / ld, j = e - i * ld;
      if (i == k) {
        M[e] = prow[j];
      } else {
        const cplx base = (i == p) ? oldk[j] : M[e];
        M[e] = csub(base, cmul(colb[i], prow[j]));
      }
    }
  }
  __syncthreads();
  return logdet;
}

// One-sided Jacobi on the r x r left half of M (row stride 2r), single warp
// (threads 0..31); writes sigma_max / sigma_min to *res.  Only used when the
// cheap Frobenius screen cannot rule out cond2 > 1e12 (cross.py:350).
__device__ __forceinline__ void jacobi_cond_warp(cplx* M, int r, double* res) {
  const int ld = 2 * r;
  const int lane = threadIdx.x;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < r - 1; ++p) {
      for (int q = p + 1; q < r; ++q) {
        double app = 0.0, aqq = 0.0;
        cplx apq = mk(0.0, 0.0);
        for (int i = lane; i < r; i += 32) {
          const cplx x = M[i * ld + p], y = M[i * ld + q];
          app += cabs2(x);
          aqq += cabs2(y);
          apq = cfmac(x, y, apq);
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        const double g = cabsh(apq);
        if (g == 0.0 || g <= 1e-17 * sqrt(app * aqq)) continue;
        off = fmax(off, g / sqrt(app * aqq));
        const double zeta = (aqq - app) / (2.0 * g);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        const cplx ph = mk(apq.x / g, apq.y / g);
        for (int i = lane; i < r; i += 32) {
          const cplx x = M[i * ld + p], y = M[i * ld + q];
          const cplx yp = cmul(y, cconj(ph));
          M[i * ld + p] = csub(cscale(x, cs), cscale(yp, sn));
          M[i * ld + q] = cmul(cadd(cscale(x, sn), cscale(yp, cs)), ph);
        }
        __syncwarp();
      }
    }
    if (off <= 1e-15) break;
  }
  double smax = 0.0, smin = INFINITY;
  for (int q = 0; q < r; ++q) {
    double s = 0.0;
    for (int i = lane; i < r; i += 32) s += cabs2(M[i * ld + q]);
    s = sqrt(warp_sum(s));
    smax = fmax(smax, s);
    smin = fmin(smin, s);
  }
  if (lane == 0) *res = (smin == 0.0) ? INFINITY : smax / smin;
}

// One row of B = Q X: out[j] = sum_t q[t * qstride] * X[t * xld + j].
// Shared by every code path that must produce bitwise-identical rows.
__device__ __forceinline__ cplx rowdot_X(const cplx* q, long long qstride, const cplx* X, int xld,
                                         int j, int r) {
  cplx acc = mk(0.0, 0.0);
  for (int t = 0; t < r; ++t) acc = cfma(q[t * qstride], X[t * xld + j], acc);
  return acc;
}

// Columns [j0, j0+JB) of one row of Q X with the row read once: acc[jj]
// receives exactly what rowdot_X(q, ..., j0+jj, r) returns (same order of
// fused multiply-adds), so both forms can be mixed bitwise-consistently.
template <int JB>
__device__ __forceinline__ void rowblock_X(const cplx* q, long long qstride, const cplx* X, int xld,
                                           int j0, int r, cplx* acc) {
#pragma unroll
  for (int jj = 0; jj < JB; ++jj) acc[jj] = mk(0.0, 0.0);
  for (int t = 0; t < r; ++t) {
    const cplx qt = q[t * qstride];
    const cplx* xr = X + t * xld + j0;
#pragma unroll
    for (int jj = 0; jj < JB; ++jj)
      if (j0 + jj < r) acc[jj] = cfma(qt, xr[jj], acc[jj]);
  }
}

// The maxvol rank-1 update of one entry (cross.py:134):
//   b[l, c] + (b[l, j] * (b[sel[j], c] - b[i, c])) / pivot
__device__ __forceinline__ cplx swap_update(cplx blc, cplx blj, cplx diffc, cplx pivot) {
  return cadd(blc, cdiv(cmul(blj, diffc), pivot));
}
