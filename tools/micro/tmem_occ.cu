// Does a kernel that allocates tensor memory (tcgen05.alloc) change the
// occupancy the runtime reports / the residency the hardware grants?
#include <cstdio>
#include <cstdint>
template <int USE>
__global__ void __launch_bounds__(256, 2) k(long long* t, int* sm) {
  __shared__ uint32_t holder;
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (USE) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&holder)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  long long t1;
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); } while (t1 - t0 < 200000);
  if (USE) {
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(holder));
  }
  if (threadIdx.x == 0) { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); sm[blockIdx.x] = s; t[blockIdx.x] = t0; }
}
template <int USE> void run(const char* name) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<USE>, 256, 0);
  long long* t; int* sm; const int n = 296;
  cudaMallocManaged(&t, n * 8); cudaMallocManaged(&sm, n * 4);
  k<USE><<<n, 256>>>(t, sm); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<USE><<<n, 256>>>(t, sm); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%s: occupancy API %d blocks/SM; 296 blocks of 0.2 ms took %.2f ms (%s)\n", name, occ, ms, cudaGetErrorString(cudaGetLastError()));
}
int main() { run<0>("plain"); run<1>("tcgen05.alloc 256 cols"); }
