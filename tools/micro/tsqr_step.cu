// Cycles per structured TSQR step (k_tsqr.cuh tw_chunk_fwd) on one warp, and
// with 8/16 warps per SM, split by component: TMEM row round trip, the owner
// lane's reflector, the broadcast, the update.
#include <cstdio>
#include <cstdint>
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
template <int MODE>  // 0 full, 1 no TMEM (R in a register), 2 reflector+bcast only, 3 update only
__global__ void k(long long* cyc, double* out, int chunks) {
  __shared__ uint32_t holder;
  __shared__ cplx vbs[16][2][LC + 1];
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
  cplx X[LC];
  for (int i = 0; i < LC; ++i) X[i] = mk(1.0 + lane * 0.01 + i * 0.001, 0.5 - i * 0.01);
  for (int j = 0; j < 32; ++j) { asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(ta + 4u * j), "r"(0x3ff00000u)); }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  cplx Rreg = mk(1.0, 0.0);
  long long t0 = clock64();
  for (int c = 0; c < chunks; ++c) {
    TmRow nx;
    if (MODE != 1) tm_ld_async(ta, 0, nx);
    for (int j = 0; j < 32; ++j) {
      cplx Rj = Rreg;
      if (MODE != 1) { Rj = tm_wait_row(nx); if (j + 1 < 32) tm_ld_async(ta, j + 1, nx); }
      cplx* b = vb + (j & 1) * (LC + 1);
      if (MODE != 3 && lane == j) {
        double p[4] = {0, 0, 0, 0};
        for (int i = 0; i < LC; ++i) p[i & 3] = fma(X[i].x, X[i].x, fma(X[i].y, X[i].y, p[i & 3]));
        const double s2 = (p[0] + p[1]) + (p[2] + p[3]);
        const double t2 = Rj.x * Rj.x + Rj.y * Rj.y + s2;
        const double beta = -copysign(sqrt(t2), Rj.x);
        const double ib = 1.0 / beta;
        const cplx tau = mk((beta - Rj.x) * ib, -Rj.y * ib);
        const double dr = Rj.x - beta;
        const double id = 1.0 / (dr * dr + Rj.y * Rj.y);
        const cplx scal = mk(dr * id, -Rj.y * id);
        for (int i = 0; i < LC; ++i) { X[i] = cmul(X[i], scal); b[i] = X[i]; }
        b[LC] = tau;
        Rj = mk(beta, 0.0);
      }
      if (MODE == 3 && lane == j) { for (int i = 0; i < LC; ++i) b[i] = X[i]; b[LC] = Rj; }
      __syncwarp();
      if (MODE != 2 && lane > j) {
        const cplx ct = cconj(b[LC]);
        cplx w0 = Rj, w1 = mk(0.0, 0.0);
        for (int i = 0; i < LC; i += 2) { w0 = cfmac(b[i], X[i], w0); w1 = cfmac(b[i + 1], X[i + 1], w1); }
        const cplx tw = cmul(ct, cadd(w0, w1));
        Rj = csub(Rj, tw);
        for (int i = 0; i < LC; ++i) X[i] = csub(X[i], cmul(tw, b[i]));
      }
      __syncwarp();
      if (MODE != 1) tm_st_async(ta, j, Rj); else Rreg = Rj;
    }
    if (MODE != 1) asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
  double acc = 0; for (int i = 0; i < LC; ++i) acc += X[i].x; out[blockIdx.x * blockDim.x + threadIdx.x] = acc + Rreg.x;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
}
template <int MODE> void run(const char* name, int warps) {
  long long* cyc; double* out;
  cudaMallocManaged(&cyc, 148 * 16 * 8); cudaMalloc(&out, 148 * 512 * 8);
  const int chunks = 20;
  k<MODE><<<1, warps * 32>>>(cyc, out, chunks); cudaDeviceSynchronize();
  k<MODE><<<1, warps * 32>>>(cyc, out, chunks); cudaDeviceSynchronize();
  long long mx = 0; for (int w = 0; w < warps; ++w) mx = cyc[w] > mx ? cyc[w] : mx;
  printf("%-28s warps %2d: %.0f cycles/step (%s)\n", name, warps, (double)mx / (chunks * 32), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int w : {1, 8, 16}) {
    run<0>("full step", w);
    run<1>("R in a register (no TMEM)", w);
    run<2>("reflector + broadcast only", w);
    run<3>("broadcast + update only", w);
  }
}
