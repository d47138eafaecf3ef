// Common device helpers for the B200 TT-Fourier pricer kernels.
//
// complex128 values are stored interleaved (re, im) as double2, exactly like
// numpy's complex128 memory layout, so buffers can be exchanged with the
// reference container format (tensor_train.py:228-261) without reshuffling.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define TTP_HD __host__ __device__ __forceinline__
#define TTP_D __device__ __forceinline__

typedef double2 cplx;

TTP_HD cplx mk(double re, double im) { return make_double2(re, im); }
TTP_HD cplx cadd(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
TTP_HD cplx csub(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
TTP_HD cplx cmul(cplx a, cplx b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
TTP_HD cplx cconj(cplx a) { return mk(a.x, -a.y); }
TTP_HD cplx cneg(cplx a) { return mk(-a.x, -a.y); }
TTP_HD cplx cscale(cplx a, double s) { return mk(a.x * s, a.y * s); }
// conj(a) * b
TTP_HD cplx cmulc(cplx a, cplx b) { return mk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x); }
// acc + a*b
TTP_HD cplx cfma(cplx a, cplx b, cplx acc) {
  return mk(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// acc + conj(a)*b
TTP_HD cplx cfmac(cplx a, cplx b, cplx acc) {
  return mk(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}
TTP_HD double cabs1(cplx a) { return fabs(a.x) + fabs(a.y); }  // LAPACK dcabs1 (izamax pivot rule)
TTP_HD double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
TTP_HD double cabsh(cplx a) { return hypot(a.x, a.y); }  // numpy abs(complex) = hypot

// Smith-style division with the same branch structure numpy uses for
// complex128 true_divide, so rank-1 maxvol updates round like the reference.
TTP_HD cplx cdiv(cplx a, cplx b) {
  const double br = fabs(b.x), bi = fabs(b.y);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0) return mk(a.x / br, a.y / bi);
    const double rat = b.y / b.x;
    const double scl = 1.0 / (b.x + b.y * rat);
    return mk((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  }
  const double rat = b.x / b.y;
  const double scl = 1.0 / (b.y + b.x * rat);
  return mk((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

TTP_D cplx cexp_d(cplx z) {
  double s, c;
  sincos(z.y, &s, &c);
  const double e = exp(z.x);
  return mk(e * c, e * s);
}

// ---------------------------------------------------------------------------
// Warp / block reductions (fixed order => bitwise run-to-run determinism).
// ---------------------------------------------------------------------------
TTP_D double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
TTP_D cplx warp_sum(cplx v) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  return v;
}
TTP_D double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Argmax record: larger value wins; on equal values the smaller key wins
// (numpy / LAPACK "first maximum" rule, key = position in scan order).
struct ArgMax {
  double v;
  long long key;
};
TTP_HD bool argmax_better(double v, long long k, double bv, long long bk) {
  return (v > bv) || (v == bv && k < bk);
}
TTP_D ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, a.v, o);
    long long ok = __shfl_xor_sync(0xffffffffu, a.key, o);
    if (argmax_better(ov, ok, a.v, a.key)) {
      a.v = ov;
      a.key = ok;
    }
  }
  return a;
}

// LAPACK-style safe scaled sum of squares: represents scale^2 * ssq.
struct Ssq {
  double scale, ssq;
};
TTP_HD Ssq ssq_init() { return Ssq{0.0, 1.0}; }
TTP_HD void ssq_add(Ssq& s, double x) {
  const double ax = fabs(x);
  if (ax != 0.0 && !isnan(ax)) {
    if (s.scale < ax) {
      const double r = s.scale / ax;
      s.ssq = 1.0 + s.ssq * r * r;
      s.scale = ax;
    } else {
      const double r = ax / s.scale;
      s.ssq += r * r;
    }
  } else if (isnan(ax)) {
    s.scale = ax;
  }
}
TTP_HD void ssq_addc(Ssq& s, cplx z) {
  ssq_add(s, z.x);
  ssq_add(s, z.y);
}
TTP_HD Ssq ssq_merge(Ssq a, Ssq b) {
  if (b.scale == 0.0) return a;
  if (a.scale == 0.0) return b;
  if (a.scale >= b.scale) {
    const double r = b.scale / a.scale;
    return Ssq{a.scale, a.ssq + b.ssq * r * r};
  }
  const double r = a.scale / b.scale;
  return Ssq{b.scale, b.ssq + a.ssq * r * r};
}
TTP_HD double ssq_norm(Ssq s) { return s.scale == 0.0 ? 0.0 : s.scale * sqrt(s.ssq); }
TTP_HD double ssq_norm2(Ssq s) { return s.scale == 0.0 ? 0.0 : (s.scale * s.scale) * s.ssq; }
// Scaled sum of squares of n complex values without per-element divisions:
// pass 1 finds the largest component, pass 2 sums squares scaled by an exact
// power of two.  Same value as the LAPACK-style recurrence up to rounding.
TTP_HD Ssq ssq_of(const cplx* p, long long stride, int n) {
  double mx = 0.0;
  for (int i = 0; i < n; ++i) {
    const cplx z = p[i * stride];
    mx = fmax(mx, fmax(fabs(z.x), fabs(z.y)));
  }
  if (mx == 0.0 || !isfinite(mx)) return Ssq{mx == 0.0 ? 0.0 : mx, 1.0};
  int e;
  frexp(mx, &e);
  const double down = ldexp(1.0, -e);
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const cplx z = p[i * stride];
    const double a = z.x * down, b = z.y * down;
    acc = fma(a, a, fma(b, b, acc));
  }
  return Ssq{ldexp(1.0, e), acc};
}

TTP_D Ssq warp_ssq(Ssq s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Ssq t;
    t.scale = __shfl_xor_sync(0xffffffffu, s.scale, o);
    t.ssq = __shfl_xor_sync(0xffffffffu, s.ssq, o);
    // merge in a lane-order-independent way: both lanes compute the same result
    // because ssq_merge is symmetric up to which side is the larger scale.
    s = ssq_merge(s, t);
  }
  return s;
}

#define TTP_CUDA_CHECK(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ttp_record_cuda_error(_e);   \
  } while (0)
