// Separable evaluation of the two hot-path oracles over a fiber block.
//
// Every entry of a sampled unfolding is oracle(L[a] ++ (s) ++ R[b]): the
// multi-index splits into coordinates owned by the block ROW and coordinates
// owned by the block COLUMN.  Both grid oracles factor over that split:
//
//   phi(-z):  E = E_X + E_Y - sum_{j in X, k in Y} y_j C_jk y_k      (market.py:216-218)
//             exp(E) with one inner product of length min(|X|, |Y|) per entry
//             once E_X, E_Y and the projected vector are precomputed;
//   vhat:     (-1)^(d-1) K prod_X g_j prod_Y g_j / (1 + i (w_X + w_Y)),
//             g_j = K^{i z_j} / (i z_j)                                (market.py:256-261)
//             i.e. one complex multiply and one complex divide per entry.
//
// Same values as oracle_value() up to rounding (~1e-14 relative on the
// BASELINE grids; SURVEY.md 8(c) P0 measured such re-associations at
// <= 8.5e-14 for cfg4).
#pragma once

#include "oracle_eval.cuh"

constexpr int FF_MAXI = 10;  // largest inner coordinate set handled (d <= 20)

struct FiberSplit {
  // coordinate positions owned by the row / column of the block
  int row_lo, row_hi;  // [row_lo, row_hi)
  int col_lo, col_hi;
  bool inner_is_col;   // inner product runs over the column coordinates
  int ninner;
};

__device__ __forceinline__ FiberSplit fiber_split(int mode, int kl, int d) {
  FiberSplit f;
  if (mode == 0) {  // rows (a, s): positions 0..kl; columns b: kl+1..d-1
    f.row_lo = 0;
    f.row_hi = kl + 1;
    f.col_lo = kl + 1;
    f.col_hi = d;
  } else {          // rows (s, b): positions kl..d-1; columns a: 0..kl-1
    f.row_lo = kl;
    f.row_hi = d;
    f.col_lo = 0;
    f.col_hi = kl;
  }
  const int nr = f.row_hi - f.row_lo, nc = f.col_hi - f.col_lo;
  f.inner_is_col = nc <= nr;
  f.ninner = f.inner_is_col ? nc : nr;
  return f;
}

__device__ __forceinline__ bool fiber_fast_ok(const OracleDev& o) {
  return (o.kind == TTP_ORACLE_PHI_GBM || o.kind == TTP_ORACLE_VHAT_MIN) && o.d <= 2 * FF_MAXI;
}

// y_j = -z_j for phi(-z)
__device__ __forceinline__ cplx phi_y(const double* p, int i) { return cneg(contour_point(p, i)); }

// Part of a phi evaluation owned by one side of the split.
//   e   : i sum_j y_j mu_j - 1/2 sum_{j,k in side} y_j C_jk y_k
//   vec : if the inner set is THIS side: y_j for j in the side
//         else: sum_{j in side} y_j C_jk for k in the OTHER (inner) side
struct PhiPart {
  cplx e;
  cplx vec[FF_MAXI];
};

__device__ __forceinline__ void phi_part(const double* p, int d, const int* idx, int lo, int hi,
                                         bool side_is_inner, int olo, int ohi, PhiPart& out) {
  const double* mu = p + 3;
  const double* C = p + 3 + d;
  cplx lin = mk(0.0, 0.0), quad = mk(0.0, 0.0);
  for (int j = lo; j < hi; ++j) {
    const cplx yj = phi_y(p, idx[j]);
    lin = cadd(lin, cscale(yj, mu[j]));
    cplx row = mk(0.0, 0.0);
    for (int k = lo; k < hi; ++k) row = cadd(row, cscale(phi_y(p, idx[k]), C[j * d + k]));
    quad = cfma(yj, row, quad);
  }
  out.e = mk(-lin.y - 0.5 * quad.x, lin.x - 0.5 * quad.y);
  if (side_is_inner) {
#pragma unroll
    for (int q = 0; q < FF_MAXI; ++q)
      if (lo + q < hi) out.vec[q] = phi_y(p, idx[lo + q]);
  } else {
#pragma unroll
    for (int q = 0; q < FF_MAXI; ++q) {
      if (olo + q < ohi) {
        cplx acc = mk(0.0, 0.0);
        for (int j = lo; j < hi; ++j) acc = cfma(phi_y(p, idx[j]), mk(C[j * d + olo + q], 0.0), acc);
        out.vec[q] = acc;
      }
    }
  }
}

__device__ __forceinline__ cplx phi_combine(const PhiPart& r, const PhiPart& c, int ninner) {
  cplx cross = mk(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < FF_MAXI; ++q)
    if (q < ninner) cross = cfma(r.vec[q], c.vec[q], cross);
  return cexp_d(csub(cadd(r.e, c.e), cross));
}

// column part stored contiguously as (e, vec[0..ninner)) in shared memory
__device__ __forceinline__ cplx phi_combine_packed(const PhiPart& r, const cplx* cb, int ninner) {
  cplx cross = mk(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < FF_MAXI; ++q)
    if (q < ninner) cross = cfma(r.vec[q], cb[1 + q], cross);
  return cexp_d(csub(cadd(r.e, cb[0]), cross));
}

// vhat side: (prod_j g_j, sum_j z_j)
__device__ __forceinline__ void vhat_part(const double* p, const int* idx, int lo, int hi, cplx& prod,
                                          cplx& w) {
  const double lnK = log(p[3]);
  prod = mk(1.0, 0.0);
  w = mk(0.0, 0.0);
  for (int j = lo; j < hi; ++j) {
    const cplx z = contour_point(p, idx[j]);
    w = cadd(w, z);
    // K^{i z} / (i z)
    const cplx kiz = cexp_d(mk(-z.y * lnK, z.x * lnK));
    prod = cmul(prod, cdiv(kiz, mk(-z.y, z.x)));
  }
}

__device__ __forceinline__ cplx vhat_combine(const double* p, int d, cplx prow, cplx wrow, cplx pcol,
                                             cplx wcol) {
  const cplx w = cadd(wrow, wcol);
  const cplx onepiw = mk(1.0 - w.y, w.x);
  cplx v = cdiv(cscale(cmul(prow, pcol), p[3]), onepiw);
  if ((d - 1) & 1) v = cneg(v);
  return (p[4] != 0.0) ? cconj(v) : v;
}
