// FP64 non-tensor (DFMA) peak of this B200: every thread runs 8 independent
// fma chains; flops = 2 per fma.  Companion of dmma_rate.cu (FP64 tensor,
// mma.sync) -- the bond kernel's rank-1 / Householder updates are DFMA work,
// its Q*X products and Gram matrices DMMA work.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_rate dfma_rate.cu
#include <cstdio>
__global__ void k(double* out, int iters, double x) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double y = 1.0 - 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, y, x); a1 = fma(a1, y, x); a2 = fma(a2, y, x); a3 = fma(a3, y, x);
      a4 = fma(a4, y, x); a5 = fma(a5, y, x); a6 = fma(a6, y, x); a7 = fma(a7, y, x);
    }
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* o;
  cudaMalloc(&o, (size_t)sms * 8 * 1024 * sizeof(double));
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  double best = 0;
  for (int blocks_per_sm : {1, 2, 4}) {
    for (int threads : {256, 512, 1024}) {
      if (blocks_per_sm * threads > 2048) continue;
      const int it = 4000, grid = sms * blocks_per_sm;
      k<<<grid, threads>>>(o, it, 1e-3);
      cudaDeviceSynchronize();
      cudaEventRecord(s);
      k<<<grid, threads>>>(o, it, 1e-3);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      float ms;
      cudaEventElapsedTime(&ms, s, e);
      const double fl = 2.0 * 8 * 8 * (double)it * threads * grid;
      const double tf = fl / ms / 1e9;
      best = tf > best ? tf : best;
      printf("DFMA blocks/SM %d threads %d: %.2f TF/s\n", blocks_per_sm, threads, tf);
    }
  }
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("best %.2f TF/s  (%d SMs, attr clock %d kHz) %s\n", best, sms, clk, cudaGetErrorString(cudaGetLastError()));
}
