// Device-side oracle descriptors (the "plugins" of tt_cross).
//
// The reference's oracle convention is a Python callable (m, d) int64 ->
// (m,) complex128 (tensor_train.py:11-13).  On the device the hot-path
// oracles are descriptors evaluated in-kernel; there is no Python callback
// and no host evaluation:
//   PHI_GBM    phi_grid_oracle     (pricers.py:234-240, market.py:204-219)
//   VHAT_MIN   payoff_grid_oracle  (pricers.py:243-253, market.py:237-262)
//   SEPARABLE  prod_k w_k[i_k]     (test helper, test_cross.py:112-119)
//   TT         tt_evaluate_many    (tensor_train.py:126-140; test targets)
//   TABLE      dense C-order lookup (small shapes; test helper)
#pragma once

#include "ttp_common.cuh"
#include "../../include/ttpricer_b200.h"

#ifndef TTP_MAX_D
#define TTP_MAX_D 64
#endif

struct OracleDev {
  int kind;
  int d;
  long long param_stride;
  const double* params;
  long long table_stride;
  const cplx* table;
  const long long* table_offsets;  // d+1 entries
  const int* tt_bonds;             // d+1 entries (TT kind)
  const int* shape;                // d entries
};

inline OracleDev oracle_dev_from(const ttp_oracle& o, const int* d_shape) {
  OracleDev r;
  r.kind = o.kind;
  r.d = o.d;
  r.param_stride = o.param_stride;
  r.params = o.params;
  r.table_stride = o.table_stride;
  r.table = reinterpret_cast<const cplx*>(o.table);
  r.table_offsets = reinterpret_cast<const long long*>(o.table_offsets);
  r.tt_bonds = o.tt_bonds;
  r.shape = d_shape;
  return r;
}

// Contour point z_j = eta * (i_j - n/2) + i*alpha  (GridSpec.contour, pricers.py:83-86).
TTP_D cplx contour_point(const double* p, int i) {
  return mk(p[0] * (double)(i - (int)p[2]), p[1]);
}

// phi_T(-z) = exp(i(-z).mu - (-z)^T C (-z) / 2)   (market.py:216-218).
TTP_D cplx eval_phi(const double* p, int d, const int* idx) {
  const double* mu = p + 3;
  const double* C = p + 3 + d;
  cplx lin = mk(0.0, 0.0);
  cplx quad = mk(0.0, 0.0);
  for (int j = 0; j < d; ++j) {
    const cplx yj = cneg(contour_point(p, idx[j]));
    lin = cadd(lin, cscale(yj, mu[j]));
    cplx row = mk(0.0, 0.0);
    for (int k = 0; k < d; ++k) {
      const cplx yk = cneg(contour_point(p, idx[k]));
      row = cadd(row, cscale(yk, C[j * d + k]));
    }
    quad = cfma(yj, row, quad);
  }
  // i*lin - 0.5*quad
  const cplx e = mk(-lin.y - 0.5 * quad.x, lin.x - 0.5 * quad.y);
  return cexp_d(e);
}

// (-1)^(d-1) K^{1+iw} / ((1+iw) prod_j (i z_j)),  w = sum_j z_j   (market.py:256-261);
// the grid oracle stores its conjugate (pricers.py:251).
TTP_D cplx eval_vhat(const double* p, int d, const int* idx) {
  const double lnK = log(p[3]);
  cplx w = mk(0.0, 0.0);
  cplx prod = mk(1.0, 0.0);
  for (int j = 0; j < d; ++j) {
    const cplx z = contour_point(p, idx[j]);
    w = cadd(w, z);
    prod = cmul(prod, mk(-z.y, z.x));  // i*z
  }
  const cplx onepiw = mk(1.0 - w.y, w.x);  // 1 + i w
  const cplx num = cexp_d(cscale(onepiw, lnK));
  cplx v = cdiv(num, cmul(onepiw, prod));
  if ((d - 1) & 1) v = cneg(v);
  return (p[4] != 0.0) ? cconj(v) : v;
}

TTP_D cplx eval_separable(const OracleDev& o, int inst, const int* idx) {
  const cplx* t = o.table + inst * o.table_stride;
  cplx v = mk(1.0, 0.0);
  for (int k = 0; k < o.d; ++k) v = cmul(v, t[o.table_offsets[k] + idx[k]]);
  return v;
}

TTP_D cplx eval_table(const OracleDev& o, int inst, const int* idx) {
  const cplx* t = o.table + inst * o.table_stride;
  long long flat = 0;
  for (int k = 0; k < o.d; ++k) flat = flat * o.shape[k] + idx[k];
  return t[flat];
}

// Target-train evaluation, left to right (tensor_train.py:136-140).
TTP_D cplx eval_tt(const OracleDev& o, int inst, const int* idx) {
  const cplx* t = o.table + inst * o.table_stride;
  cplx vec[TTP_MAX_D];
  cplx nxt[TTP_MAX_D];
  int r0 = o.tt_bonds[1];
  const cplx* c0 = t + o.table_offsets[0];
  for (int b = 0; b < r0; ++b) vec[b] = c0[(long long)idx[0] * r0 + b];
  for (int k = 1; k < o.d; ++k) {
    const int ra = o.tt_bonds[k], rb = o.tt_bonds[k + 1], nk = o.shape[k];
    const cplx* ck = t + o.table_offsets[k];
    for (int b = 0; b < rb; ++b) {
      cplx acc = mk(0.0, 0.0);
      for (int a = 0; a < ra; ++a)
        acc = cfma(vec[a], ck[((long long)a * nk + idx[k]) * rb + b], acc);
      nxt[b] = acc;
    }
    for (int b = 0; b < rb; ++b) vec[b] = nxt[b];
  }
  return vec[0];
}

TTP_D cplx oracle_value(const OracleDev& o, int inst, const int* idx) {
  switch (o.kind) {
    case TTP_ORACLE_PHI_GBM:
      return eval_phi(o.params + inst * o.param_stride, o.d, idx);
    case TTP_ORACLE_VHAT_MIN:
      return eval_vhat(o.params + inst * o.param_stride, o.d, idx);
    case TTP_ORACLE_SEPARABLE:
      return eval_separable(o, inst, idx);
    case TTP_ORACLE_TABLE:
      return eval_table(o, inst, idx);
    case TTP_ORACLE_TT:
      return eval_tt(o, inst, idx);
    default:
      return mk(nan(""), nan(""));
  }
}
