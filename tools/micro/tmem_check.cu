// TMEM region check: 2 CTAs per SM (256 threads, 256 columns each); warp w
// uses lane quarter (w % 4) and columns ((w / 4) * 128, +128): every warp
// writes a pattern row by row (32x32b.x4), waits, reads it back.
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(256, 2) k(int* bad, long long* sample) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = holder;
  const uint32_t a = base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  if (blockIdx.x < 2 && threadIdx.x == 0) sample[blockIdx.x] = base;
  for (int it = 0; it < 50; ++it) {
    for (int row = 0; row < 32; ++row) {
      const uint32_t v0 = blockIdx.x * 1000003u + warp * 7919u + lane * 131u + row * 17u + it;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + 4u * row), "r"(v0), "r"(v0 + 1), "r"(v0 + 2), "r"(v0 + 3));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    for (int row = 0; row < 32; ++row) {
      uint32_t r0, r1, r2, r3;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a + 4u * row));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const uint32_t v0 = blockIdx.x * 1000003u + warp * 7919u + lane * 131u + row * 17u + it;
      if (r0 != v0 || r1 != v0 + 1 || r2 != v0 + 2 || r3 != v0 + 3) atomicAdd(bad, 1);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(base));
}
int main() {
  int* bad; long long* s;
  cudaMallocManaged(&bad, 4); cudaMallocManaged(&s, 16);
  *bad = 0;
  k<<<296 * 4, 256>>>(bad, s);
  cudaDeviceSynchronize();
  printf("mismatches %d (%s); base of CTA0 %llx CTA1 %llx\n", *bad, cudaGetErrorString(cudaGetLastError()), s[0], s[1]);
}
