#include <cstdio>
__global__ void k(double* out, int iters) {
  double a[4] = {1.0, 2.0, 3.0, 4.0}, b[2] = {0.5, 0.25};
  double c[4] = {0, 0, 0, 0};
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = c[0] + c[1] + c[2] + c[3];
}
__global__ void k4(double* out, int iters) {
  double a = threadIdx.x, b = 0.5;
  double c0 = 0, c1 = 0;
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = c0 + c1;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 1024 * 8 * 8);
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  for (int w : {4, 8, 16, 32}) {
    int it = 20000;
    k<<<148 * 2, w * 32>>>(o, it); cudaDeviceSynchronize();
    cudaEventRecord(s); k<<<148 * 2, w * 32>>>(o, it); cudaEventRecord(e); cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    double fl = 2.0 * 16 * 8 * 8 * (double)it * w * 148 * 2;
    printf("m16n8k8 warps/blk %d: %.2f TF/s\n", w, fl / ms / 1e9);
    k4<<<148 * 2, w * 32>>>(o, it); cudaDeviceSynchronize();
    cudaEventRecord(s); k4<<<148 * 2, w * 32>>>(o, it); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    fl = 2.0 * 8 * 8 * 4 * (double)it * w * 148 * 2;
    printf("m8n8k4 warps/blk %d: %.2f TF/s\n", w, fl / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
