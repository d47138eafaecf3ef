// FP64 dependent-chain latencies on this B200 (clock64 around N dependent
// ops, one warp): DFMA, DADD, double shuffle, reciprocal, sqrt, division.
// These set the per-step critical path of the bond kernel's sequential
// Householder / pivot steps.  build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x, int n) {
  double a = x + threadIdx.x * 1e-9, y = 1.0 - 1e-12;
  long long t0, t1;
  // DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, y, x);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DADD
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + y;
  t1 = clock64(); cyc[1] = t1 - t0;
  // shuffle of a double (2 x SHFL) + add
  t0 = clock64();
  for (int i = 0; i < n; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1);
  t1 = clock64(); cyc[2] = t1 - t0;
  // reciprocal
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = 1.0 / (a + 2.0);
  t1 = clock64(); cyc[3] = t1 - t0;
  // sqrt
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = sqrt(a + 2.0);
  t1 = clock64(); cyc[4] = t1 - t0;
  // smem round trip
  __shared__ double sm[64];
  sm[threadIdx.x] = a;
  __syncwarp();
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = sm[idx] + 1.0; sm[idx] = a; __syncwarp(); }
  t1 = clock64(); cyc[5] = t1 - t0;
  // __syncthreads with 8 warps launched
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); cyc[6] = t1 - t0;
  out[threadIdx.x] = a;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 4096 * 8); cudaMallocManaged(&c, 16 * 8);
  const int n = 1000;
  k<<<1, 256>>>(o, c, 1e-3, n);
  cudaDeviceSynchronize();
  k<<<1, 256>>>(o, c, 1e-3, n);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DADD", "SHFL.f64+DADD", "1/x (f64)", "sqrt (f64)", "LDS+DADD+STS", "BAR 8 warps"};
  for (int i = 0; i < 7; ++i) printf("%-16s %.1f cycles per dependent op\n", names[i], (double)c[i] / n);
}
