// Cycles per structured TSQR chunk step (k_tsqr.cuh tw_chunk_fwd, the
// owner-publishes-raw-column form) at 1/8/16 warps per SM, for variants of
// the FP64 instruction stream:
//   V0  the shipped step (csub(X, cmul(tws, b)) update, 2-accumulator dots)
//   V1  update as explicit fma pairs (4 DFMA per complex axpy instead of 6)
//   V2  V1 + the owner's norm folded into the previous step's update
//       (lane j+1 accumulates |x|^2 of its column while updating it)
//   V3  V1 with 4-accumulator dots
// Also checks that every variant leaves the same R and X up to rounding.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
typedef double2 cplx;
__device__ __forceinline__ cplx mk(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx cconj(cplx a) { return mk(a.x, -a.y); }
__device__ __forceinline__ cplx cfmac(cplx a, cplx b, cplx acc) {
  return mk(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}
// x - t*b as two fma pairs
__device__ __forceinline__ cplx caxmy(cplx t, cplx b, cplx x) {
  return mk(fma(-t.x, b.x, fma(t.y, b.y, x.x)), fma(-t.x, b.y, fma(-t.y, b.x, x.y)));
}
struct TmRow { uint32_t q0, q1, q2, q3; };
__device__ __forceinline__ void tm_ld_async(uint32_t a, int row, TmRow& t) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(t.q0), "=r"(t.q1), "=r"(t.q2), "=r"(t.q3) : "r"(a + 4u * row));
}
__device__ __forceinline__ cplx tm_wait_row(TmRow& t) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(t.q0), "+r"(t.q1), "+r"(t.q2), "+r"(t.q3) :: "memory");
  return mk(__hiloint2double((int)t.q1, (int)t.q0), __hiloint2double((int)t.q3, (int)t.q2));
}
__device__ __forceinline__ void tm_st_async(uint32_t a, int row, cplx v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + 4u * row),
               "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y)) : "memory");
}
constexpr int LC = 8;

template <int V>
__global__ void k(long long* cyc, double* out, int chunks) {
  __shared__ uint32_t holder;
  __shared__ cplx vbs[16][2][LC + 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t ta = holder + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  cplx* vb = &vbs[warp][0][0];
  for (int j = 0; j < 32; ++j)
    tm_st_async(ta, j, mk(j == lane ? 2.0 : 0.01 * (j + lane), 0.003 * (lane - j)));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  double accum = 0.0;
  long long t0 = clock64();
  for (int c = 0; c < chunks; ++c) {
    cplx X[LC];
    for (int i = 0; i < LC; ++i) X[i] = mk(0.1 + lane * 0.01 + i * 0.001 + c * 1e-4, 0.05 - i * 0.01);
    cplx myscal = mk(1.0, 0.0);
    double nxt = 0.0;  // V2: this lane's column norm, folded into the update
    if (V == 2) {
      double p = 0.0;
      for (int i = 0; i < LC; ++i) p = fma(X[i].x, X[i].x, fma(X[i].y, X[i].y, p));
      nxt = p;
    }
    TmRow nx;
    tm_ld_async(ta, 0, nx);
    for (int j = 0; j < 32; ++j) {
      cplx Rj = tm_wait_row(nx);
      if (j + 1 < 32) tm_ld_async(ta, j + 1, nx);
      cplx* b = vb + (j & 1) * (LC + 2);
      if (lane == j) {
        double s2;
        if (V == 2) {
          s2 = nxt;
        } else {
          double p[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int i = 0; i < LC; ++i) p[i & 3] = fma(X[i].x, X[i].x, fma(X[i].y, X[i].y, p[i & 3]));
          s2 = (p[0] + p[1]) + (p[2] + p[3]);
        }
#pragma unroll
        for (int i = 0; i < LC; ++i) b[i] = X[i];
        const double a2 = Rj.x * Rj.x + Rj.y * Rj.y;
        const double beta = -copysign(sqrt(a2 + s2), Rj.x);
        const double ib = 1.0 / beta;
        const cplx tau = mk((beta - Rj.x) * ib, -Rj.y * ib);
        const double dr = Rj.x - beta;
        const double id = 1.0 / (dr * dr + Rj.y * Rj.y);
        myscal = mk(dr * id, -Rj.y * id);
        b[LC] = tau;
        b[LC + 1] = myscal;
        Rj = mk(beta, 0.0);
      }
      __syncwarp();
      if (lane > j) {
        const cplx ct = cconj(b[LC]), sc = b[LC + 1];
        cplx w;
        if (V == 3) {
          cplx w0 = mk(0.0, 0.0), w1 = w0, w2 = w0, w3 = w0;
#pragma unroll
          for (int i = 0; i < LC; i += 4) {
            w0 = cfmac(b[i], X[i], w0);
            w1 = cfmac(b[i + 1], X[i + 1], w1);
            w2 = cfmac(b[i + 2], X[i + 2], w2);
            w3 = cfmac(b[i + 3], X[i + 3], w3);
          }
          w = cfmac(sc, cadd(cadd(w0, w1), cadd(w2, w3)), Rj);
        } else {
          cplx w0 = mk(0.0, 0.0), w1 = mk(0.0, 0.0);
#pragma unroll
          for (int i = 0; i < LC; i += 2) {
            w0 = cfmac(b[i], X[i], w0);
            w1 = cfmac(b[i + 1], X[i + 1], w1);
          }
          w = cfmac(sc, cadd(w0, w1), Rj);
        }
        const cplx tw = cmul(ct, w);
        Rj = csub(Rj, tw);
        const cplx tws = cmul(tw, sc);
        if (V == 0) {
#pragma unroll
          for (int i = 0; i < LC; ++i) X[i] = csub(X[i], cmul(tws, b[i]));
        } else if (V == 2) {
          double p = 0.0;
#pragma unroll
          for (int i = 0; i < LC; ++i) {
            X[i] = caxmy(tws, b[i], X[i]);
            p = fma(X[i].x, X[i].x, fma(X[i].y, X[i].y, p));
          }
          nxt = p;
        } else {
#pragma unroll
          for (int i = 0; i < LC; ++i) X[i] = caxmy(tws, b[i], X[i]);
        }
      }
      __syncwarp();
      tm_st_async(ta, j, Rj);
    }
    for (int i = 0; i < LC; ++i) X[i] = cmul(X[i], myscal);
    asm volatile("tcgen05.wait::st.sync.aligned;");
    for (int i = 0; i < LC; ++i) accum += X[i].x + X[i].y;
    // restore the triangle so every chunk sees the same input (not timed separately; small)
    for (int j = 0; j < 32; ++j)
      tm_st_async(ta, j, mk(j == lane ? 2.0 : 0.01 * (j + lane), 0.003 * (lane - j)));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = accum;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
}

static double ref_out[512];
template <int V> void run(const char* name, int warps) {
  long long* cyc; double* out;
  cudaMallocManaged(&cyc, 148 * 16 * 8); cudaMallocManaged(&out, 148 * 512 * 8);
  const int chunks = 20;
  k<V><<<1, warps * 32>>>(cyc, out, chunks); cudaDeviceSynchronize();
  k<V><<<1, warps * 32>>>(cyc, out, chunks); cudaDeviceSynchronize();
  long long mx = 0; for (int w = 0; w < warps; ++w) mx = cyc[w] > mx ? cyc[w] : mx;
  double dev = 0.0;
  if (V == 0 && warps == 1) for (int i = 0; i < 32; ++i) ref_out[i] = out[i];
  if (warps == 1) for (int i = 0; i < 32; ++i) dev = fmax(dev, fabs(out[i] - ref_out[i]) / fmax(1e-300, fabs(ref_out[i])));
  printf("%-34s warps %2d: %6.0f cycles/step  (max rel diff vs V0 %.1e) %s\n", name, warps, (double)mx / (chunks * 32.0),
         dev, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc); cudaFree(out);
}
int main() {
  for (int w : {1, 8, 16}) {
    run<0>("V0 shipped", w);
    run<1>("V1 fma-pair update", w);
    run<2>("V2 V1 + norm folded into update", w);
    run<3>("V3 V1 + 4-acc dots", w);
  }
}
