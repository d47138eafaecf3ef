// Streaming r+w sweeps over per-CTA column-major slices (ms rows x r cols of
// complex128), the access pattern of the bond kernel's row passes, with
// (a) thread-batched loads (KB per thread in flight) and (b) bulk-async
// (cp.async.bulk) row tiles double-buffered in shared memory.
// Reports effective GB/s (read+write) over all SMs.
#include <cstdio>
#include <cuda_runtime.h>
typedef double2 cplx;
constexpr int CT = 512;

template <int KB>
__global__ void __launch_bounds__(CT, 1) sweep_threads(cplx* base, int ms, int r, long long stride, int passes) {
  cplx* W = base + blockIdx.x * stride;
  for (int p = 0; p < passes; ++p) {
    for (int l = threadIdx.x; l < ms; l += CT) {
      cplx* q = W + l;
      for (int t = 0; t < r; t += KB) {
        cplx x[KB];
#pragma unroll
        for (int u = 0; u < KB; ++u) x[u] = q[(long long)(t + u) * ms];
#pragma unroll
        for (int u = 0; u < KB; ++u) { x[u].x = x[u].x * 0.999 + 1e-3; x[u].y = x[u].y * 0.999; q[(long long)(t + u) * ms] = x[u]; }
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(b)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}

// tile = TR rows x r cols (column-major in smem, ld TR); NS stages
template <int TR, int NS>
__global__ void __launch_bounds__(CT, 1) sweep_bulk(cplx* base, int ms, int r, long long stride, int passes) {
  extern __shared__ __align__(128) unsigned char sm[];
  cplx* tiles = (cplx*)sm;
  unsigned long long* bar = (unsigned long long*)(sm + (size_t)NS * TR * r * sizeof(cplx));
  cplx* W = base + blockIdx.x * stride;
  if (threadIdx.x == 0) for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int ntile = ms / TR;
  unsigned phase[NS];
  for (int s = 0; s < NS; ++s) phase[s] = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int p = 0; p < passes; ++p) {
    auto issue = [&](int tile) {
      const int s = tile % NS;
      if (warp == 0) {
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // previous store from this stage drained
          mbar_expect(&bar[s], TR * r * sizeof(cplx));
        }
        __syncwarp();
        for (int t = lane; t < r; t += 32)
          bulk_g2s(tiles + ((size_t)s * r + t) * TR, W + (long long)t * ms + tile * TR, TR * sizeof(cplx), &bar[s]);
      }
    };
    for (int k = 0; k < NS - 1 && k < ntile; ++k) issue(k);
    for (int k = 0; k < ntile; ++k) {
      if (k + NS - 1 < ntile) issue(k + NS - 1);
      const int s = k % NS;
      mbar_wait(&bar[s], phase[s]);
      phase[s] ^= 1;
      cplx* T = tiles + (size_t)s * r * TR;
      for (int e = threadIdx.x; e < TR * r; e += CT) { cplx x = T[e]; x.x = x.x * 0.999 + 1e-3; x.y = x.y * 0.999; T[e] = x; }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (warp == 0) {
        for (int t = lane; t < r; t += 32)
          bulk_s2g(W + (long long)t * ms + k * TR, T + (size_t)t * TR, TR * sizeof(cplx));
        if (lane == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (warp == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
  }
}

int main() {
  const int nblk = 148, ms = 2048, r = 32, passes = 20;
  const long long stride = (long long)ms * r;
  cplx* buf;
  cudaMalloc(&buf, sizeof(cplx) * stride * nblk);
  cudaMemset(buf, 0, sizeof(cplx) * stride * nblk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = 2.0 * sizeof(cplx) * stride * nblk * passes;
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms_;
    cudaEventElapsedTime(&ms_, a, b);
    printf("%-28s %8.1f GB/s  (%.1f us per pass per CTA-slice of %.2f MB)  %s\n", name, bytes / ms_ / 1e6,
           1e3 * ms_ / passes, sizeof(cplx) * stride / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run("threads KB=4", [&] { sweep_threads<4><<<nblk, CT>>>(buf, ms, r, stride, passes); });
  run("threads KB=8", [&] { sweep_threads<8><<<nblk, CT>>>(buf, ms, r, stride, passes); });
  run("threads KB=16", [&] { sweep_threads<16><<<nblk, CT>>>(buf, ms, r, stride, passes); });
  {
    auto k = sweep_bulk<64, 3>;
    size_t sm = 3 * 64 * r * sizeof(cplx) + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    run("bulk TR=64 NS=3 (144KB)", [&] { k<<<nblk, CT, sm>>>(buf, ms, r, stride, passes); });
  }
  {
    auto k = sweep_bulk<32, 6>;
    size_t sm = 6 * 32 * r * sizeof(cplx) + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    run("bulk TR=32 NS=6 (192KB)", [&] { k<<<nblk, CT, sm>>>(buf, ms, r, stride, passes); });
  }
  {
    auto k = sweep_bulk<64, 2>;
    size_t sm = 2 * 64 * r * sizeof(cplx) + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    run("bulk TR=64 NS=2 (64KB)", [&] { k<<<nblk, CT, sm>>>(buf, ms, r, stride, passes); });
  }
  {
    auto k = sweep_bulk<32, 2>;
    size_t sm = 2 * 32 * r * sizeof(cplx) + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    run("bulk TR=32 NS=2 (32KB)", [&] { k<<<nblk, CT, sm>>>(buf, ms, r, stride, passes); });
  }
  return 0;
}
