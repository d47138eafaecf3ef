// K6 / K7: tensor-train contractions.
//
//  * tt_inner (tensor_train.py:143-159): per site the environment (Db x Dk)
//    is pushed through  env' = sum_s conj(B_s)^T (env K_s).  One CTA per
//    instance; env and the (env K_s) tile live in shared memory, each thread
//    owns a fixed set of env' accumulators in registers, and the s-sum runs
//    in order, so the result is bitwise reproducible.
//  * tt_evaluate_many (tensor_train.py:126-140):
//      - eval_warp_kernel: one warp per sample (public API, any index set);
//      - site_group_kernel: the convergence-check path.  The 50 000 samples
//        of tt_rand_sample_diff are fixed per (seed, shape)
//        (tensor_train.py:191-194), so they are bucketed once per site by
//        their index there; a CTA then loads the single core slice
//        G_k[:, s, :] into shared memory and streams every sample of bucket
//        s through it.  Each slice is read from HBM once per sweep instead
//        of once per sample.
#include "ttp_internal.h"
#include "dev_knobs.h"
#include "launch.h"
#include <cooperative_groups.h>
#include <cstring>
namespace cg = cooperative_groups;

namespace {

// ----------------------------------------------------------------- tt_inner
struct TTDev {
  const cplx* cores;
  long long stride;
  long long off[TTP_MAX_D + 1];
  int bonds[TTP_MAX_D + 1];
  int shape[TTP_MAX_D];
  int d;
};

TTDev tt_dev(const ttp_tt_batch& b) {
  TTDev t;
  t.cores = reinterpret_cast<const cplx*>(b.d_cores);
  t.stride = b.stride;
  t.d = b.d;
  for (int k = 0; k <= b.d; ++k) {
    t.off[k] = b.h_offsets[k];
    t.bonds[k] = b.h_bonds[k];
  }
  for (int k = 0; k < b.d; ++k) t.shape[k] = b.h_shape[k];
  return t;
}

constexpr int INNER_THREADS = 512;
constexpr int INNER_ACC = 8;  // (64*64)/512 accumulators per thread max

__global__ void __launch_bounds__(INNER_THREADS)
tt_inner_kernel(const TTDev bra, const TTDev ket, cplx* __restrict__ out) {
  extern __shared__ cplx sm[];
  const int inst = blockIdx.x;
  const int tid = threadIdx.x;
  int maxb = 1, maxk = 1;
  for (int k = 0; k <= bra.d; ++k) {
    maxb = max(maxb, bra.bonds[k]);
    maxk = max(maxk, ket.bonds[k]);
  }
  cplx* env = sm;                 // Db x Dk
  cplx* tmp = sm + maxb * maxk;   // Db x Dk'
  if (tid == 0) env[0] = mk(1.0, 0.0);
  __syncthreads();
  for (int k = 0; k < bra.d; ++k) {
    const int Db = bra.bonds[k], Db2 = bra.bonds[k + 1];
    const int Dk = ket.bonds[k], Dk2 = ket.bonds[k + 1];
    const int n = bra.shape[k];
    const cplx* B = bra.cores + inst * bra.stride + bra.off[k];
    const cplx* K = ket.cores + inst * ket.stride + ket.off[k];
    const int nacc = Db2 * Dk2;
    cplx acc[INNER_ACC];
#pragma unroll
    for (int q = 0; q < INNER_ACC; ++q) acc[q] = mk(0.0, 0.0);
    for (int s = 0; s < n; ++s) {
      // tmp[a, c] = sum_b env[a, b] * K[b, s, c]
      for (int e = tid; e < Db * Dk2; e += INNER_THREADS) {
        const int a = e / Dk2, c = e - a * Dk2;
        cplx t = mk(0.0, 0.0);
        for (int b = 0; b < Dk; ++b) t = cfma(env[a * Dk + b], K[((long long)b * n + s) * Dk2 + c], t);
        tmp[e] = t;
      }
      __syncthreads();
      // env'[a2, c] += sum_a conj(B[a, s, a2]) * tmp[a, c]
#pragma unroll
      for (int q = 0; q < INNER_ACC; ++q) {
        const int e = tid + q * INNER_THREADS;
        if (e < nacc) {
          const int a2 = e / Dk2, c = e - a2 * Dk2;
          cplx t = acc[q];
          for (int a = 0; a < Db; ++a)
            t = cfmac(B[((long long)a * n + s) * Db2 + a2], tmp[a * Dk2 + c], t);
          acc[q] = t;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < INNER_ACC; ++q) {
      const int e = tid + q * INNER_THREADS;
      if (e < nacc) env[e] = acc[q];
    }
    __syncthreads();
  }
  if (tid == 0) out[inst] = env[0];
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all_but_one() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Same contraction as tt_inner_kernel with the two core slices of every s
// staged in shared memory by cp.async (coalesced: each slice row is a
// contiguous D-vector) and double-buffered, so the slice for s+1 streams in
// while s is contracted; identical arithmetic order, hence identical bits.
__device__ __forceinline__ void stage_slice(cplx* dst, const cplx* core, int rows, int n, int s, int cols) {
  for (int e = threadIdx.x; e < rows * cols; e += INNER_THREADS) {
    const int a = e / cols, c = e - a * cols;
    cp_async16(dst + e, core + ((long long)a * n + s) * cols + c);
  }
}

__global__ void __launch_bounds__(INNER_THREADS)
tt_inner_staged_kernel(const TTDev bra, const TTDev ket, cplx* __restrict__ out, int maxb, int maxk) {
  extern __shared__ __align__(16) cplx sm[];
  const int inst = blockIdx.x;
  const int tid = threadIdx.x;
  cplx* env = sm;                        // Db x Dk
  cplx* tmp = env + maxb * maxk;         // Db x Dk'
  cplx* kst[2] = {tmp + maxb * maxk, tmp + maxb * maxk + maxk * maxk};
  cplx* bst[2] = {kst[1] + maxk * maxk, kst[1] + maxk * maxk + maxb * maxb};
  if (tid == 0) env[0] = mk(1.0, 0.0);
  __syncthreads();
  for (int k = 0; k < bra.d; ++k) {
    const int Db = bra.bonds[k], Db2 = bra.bonds[k + 1];
    const int Dk = ket.bonds[k], Dk2 = ket.bonds[k + 1];
    const int n = bra.shape[k];
    const cplx* B = bra.cores + inst * bra.stride + bra.off[k];
    const cplx* K = ket.cores + inst * ket.stride + ket.off[k];
    const int nacc = Db2 * Dk2;
    cplx acc[INNER_ACC];
#pragma unroll
    for (int q = 0; q < INNER_ACC; ++q) acc[q] = mk(0.0, 0.0);
    stage_slice(kst[0], K, Dk, n, 0, Dk2);
    stage_slice(bst[0], B, Db, n, 0, Db2);
    cp_async_commit();
    for (int s = 0; s < n; ++s) {
      const int cur = s & 1;
      if (s + 1 < n) {
        stage_slice(kst[cur ^ 1], K, Dk, n, s + 1, Dk2);
        stage_slice(bst[cur ^ 1], B, Db, n, s + 1, Db2);
      }
      cp_async_commit();
      cp_async_wait_all_but_one();
      __syncthreads();
      const cplx* Ks = kst[cur];
      const cplx* Bs = bst[cur];
      for (int e = tid; e < Db * Dk2; e += INNER_THREADS) {
        const int a = e / Dk2, c = e - a * Dk2;
        cplx t = mk(0.0, 0.0);
        for (int b = 0; b < Dk; ++b) t = cfma(env[a * Dk + b], Ks[b * Dk2 + c], t);
        tmp[e] = t;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < INNER_ACC; ++q) {
        const int e = tid + q * INNER_THREADS;
        if (e < nacc) {
          const int a2 = e / Dk2, c = e - a2 * Dk2;
          cplx t = acc[q];
          for (int a = 0; a < Db; ++a) t = cfmac(Bs[a * Db2 + a2], tmp[a * Dk2 + c], t);
          acc[q] = t;
        }
      }
      __syncthreads();
    }
    cp_async_wait_all();
#pragma unroll
    for (int q = 0; q < INNER_ACC; ++q) {
      const int e = tid + q * INNER_THREADS;
      if (e < nacc) env[e] = acc[q];
    }
    __syncthreads();
  }
  if (tid == 0) out[inst] = env[0];
}

// Bonds above 32 (cfg5, D = 64): the environment and one (env K_s) tile do
// not leave room to stage slices, and one CTA per instance leaves all but
// one SM idle for a single option.  A cluster of TS_G CTAs per instance
// splits each site's s-sum into contiguous chunks (CTA g: s in
// [g n / G, (g+1) n / G)); every CTA accumulates its partial env' in
// registers, publishes it in shared memory, and after one cluster barrier
// every CTA sums the G partials in rank order over DSMEM, so all of them
// hold the same env' bits for the next site.  Per-CTA arithmetic is that of
// tt_inner_kernel; the s-sum is grouped by chunk.
constexpr int TS_G = 16;  // CTAs per instance (non-portable cluster size)

__global__ void __launch_bounds__(INNER_THREADS, 1)
tt_inner_split_kernel(const TTDev bra, const TTDev ket, cplx* __restrict__ out, int maxb, int maxk) {
  extern __shared__ __align__(16) cplx sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks();
  const int g = (int)cl.block_rank();
  const int inst = blockIdx.x / G;
  const int tid = threadIdx.x;
  cplx* env = sm;                 // Db x Dk (full, replicated)
  cplx* tmp = env + maxb * maxk;  // Db x Dk'
  cplx* part = tmp + maxb * maxk; // Db' x Dk' partial env' of this CTA
  if (tid == 0) env[0] = mk(1.0, 0.0);
  __syncthreads();
  for (int k = 0; k < bra.d; ++k) {
    const int Db = bra.bonds[k], Db2 = bra.bonds[k + 1];
    const int Dk = ket.bonds[k], Dk2 = ket.bonds[k + 1];
    const int n = bra.shape[k];
    const cplx* B = bra.cores + inst * bra.stride + bra.off[k];
    const cplx* K = ket.cores + inst * ket.stride + ket.off[k];
    const int nacc = Db2 * Dk2;
    const int s0 = (int)((long long)g * n / G), s1 = (int)((long long)(g + 1) * n / G);
    cplx acc[INNER_ACC];
#pragma unroll
    for (int q = 0; q < INNER_ACC; ++q) acc[q] = mk(0.0, 0.0);
    for (int s = s0; s < s1; ++s) {
      for (int e = tid; e < Db * Dk2; e += INNER_THREADS) {
        const int a = e / Dk2, c = e - a * Dk2;
        cplx t = mk(0.0, 0.0);
        for (int b = 0; b < Dk; ++b) t = cfma(env[a * Dk + b], K[((long long)b * n + s) * Dk2 + c], t);
        tmp[e] = t;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < INNER_ACC; ++q) {
        const int e = tid + q * INNER_THREADS;
        if (e < nacc) {
          const int a2 = e / Dk2, c = e - a2 * Dk2;
          cplx t = acc[q];
          for (int a = 0; a < Db; ++a) t = cfmac(B[((long long)a * n + s) * Db2 + a2], tmp[a * Dk2 + c], t);
          acc[q] = t;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < INNER_ACC; ++q) {
      const int e = tid + q * INNER_THREADS;
      if (e < nacc) part[e] = acc[q];
    }
    cl.sync();  // every CTA's partial is published
#pragma unroll
    for (int q = 0; q < INNER_ACC; ++q) {
      const int e = tid + q * INNER_THREADS;
      if (e < nacc) {
        cplx t = mk(0.0, 0.0);
        for (int h = 0; h < G; ++h) t = cadd(t, cl.map_shared_rank(part, h)[e]);
        env[e] = t;
      }
    }
    cl.sync();  // no CTA rewrites its partial while a peer still reads it
  }
  if (g == 0 && tid == 0) out[inst] = env[0];
}

size_t tt_inner_split_smem(int maxb, int maxk) { return sizeof(cplx) * (size_t)(3 * maxb * maxk); }

// FP64 tensor-core variant (DMMA m8n8k4) working on chunks of IC_SC values
// of s at a time, so each of the two GEMMs per chunk is large enough to keep
// the tensor pipe busy between barriers:
//   T  = env K[:, chunk, :]                  (Db x Dk)(Dk x SC*Dk2)
//   E += sum_{a, s in chunk} conj(B[a,s,:])^T T[a,s,:]   (K dim = Db*SC)
// as real GEMMs on the interleaved layout (left operands as stored, with the
// conjugate sign for B; right operands expanded on the fly).  E lives in the
// DMMA accumulators for the whole site.  Core slices of the next chunk stream
// in by cp.async while the current one is contracted.  Bonds <= 32.
#ifndef IC_SC_DEF
#define IC_SC_DEF 2
#endif
#ifndef IC_THREADS_DEF
#define IC_THREADS_DEF 512
#endif
constexpr int IC_SC = IC_SC_DEF;            // s values per chunk
constexpr int IC_THREADS = IC_THREADS_DEF;  // 512 (one CTA per SM) or 256
constexpr int IC_MINB = IC_THREADS >= 512 ? 1 : 2;

__device__ __forceinline__ void ic_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// expanded right operand G'[k][n] of a complex matrix (rows x cols, ld ldg)
__device__ __forceinline__ double ic_gexp(const cplx* G, int ldg, int rows, int cols, int k, int n) {
  const int a = k >> 1, c = n >> 1;
  if (a >= rows || c >= cols) return 0.0;
  const cplx g = G[a * ldg + c];
  return ((k & 1) == (n & 1)) ? g.x : ((n & 1) ? g.y : -g.y);
}

__global__ void __launch_bounds__(IC_THREADS, IC_MINB)
tt_inner_chunk_kernel(const TTDev bra, const TTDev ket, cplx* __restrict__ out) {
  extern __shared__ __align__(16) cplx sm[];
  constexpr int MX = 32;
  const int inst = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  constexpr int NW = IC_THREADS / 32;
  static_assert(NW == 8 || NW == 16, "GEMM2 tiling assumes 8 or 16 warps");
  const int ldE = 2 * MX + 4;
  double* envd = reinterpret_cast<double*>(sm);                 // MX x ldE
  cplx* T = reinterpret_cast<cplx*>(envd + MX * ldE);            // MX x SC*MX
  cplx* stage = T + MX * IC_SC * MX;                             // [2] x (Kc + Bc)
  const int selems = 2 * MX * IC_SC * MX;
  for (int e = threadIdx.x; e < MX * ldE; e += IC_THREADS) envd[e] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) envd[0] = 1.0;
  __syncthreads();
  for (int k = 0; k < bra.d; ++k) {
    const int Db = bra.bonds[k], Db2 = bra.bonds[k + 1];
    const int Dk = ket.bonds[k], Dk2 = ket.bonds[k + 1];
    const int n = bra.shape[k];
    const cplx* B = bra.cores + inst * bra.stride + bra.off[k];
    const cplx* K = ket.cores + inst * ket.stride + ket.off[k];
    const int nch = (n + IC_SC - 1) / IC_SC;
    const int ldK = IC_SC * Dk2, ldB = IC_SC * Db2;
    // chunk staging: Kc[b][sl*Dk2 + c], Bc[a][sl*Db2 + a2]; missing sl zero-filled
    auto issue = [&](int ch, int buf) {
      cplx* Kc = stage + buf * selems;
      cplx* Bc = Kc + MX * IC_SC * MX;
      const int s0 = ch * IC_SC;
      for (int e = threadIdx.x; e < Dk * ldK; e += IC_THREADS) {
        const int b = e / ldK, j = e - b * ldK, sl = j / Dk2, c = j - sl * Dk2;
        const bool ok = s0 + sl < n;
        const cplx* src = K + ((long long)b * n + (ok ? s0 + sl : 0)) * Dk2 + c;
        const unsigned sa = (unsigned)__cvta_generic_to_shared(Kc + e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0));
      }
      for (int e = threadIdx.x; e < Db * ldB; e += IC_THREADS) {
        const int a = e / ldB, j = e - a * ldB, sl = j / Db2, c = j - sl * Db2;
        const bool ok = s0 + sl < n;
        const cplx* src = B + ((long long)a * n + (ok ? s0 + sl : 0)) * Db2 + c;
        const unsigned sa = (unsigned)__cvta_generic_to_shared(Bc + e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0));
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    // GEMM2 output tiles: n-tile (warp & 7) of 2*Dk2, m-tiles (warp >> 3) + MG*i of Db2
    constexpr int MG = NW / 8, MPW = 4 / MG;  // warp groups over the 4 m-tiles; m-tiles per warp
    const int ntn2 = (2 * Dk2 + 7) / 8, mtn2 = (Db2 + 7) / 8;
    const int nt2 = warp & 7, mg2 = warp >> 3;
    double acc[MPW][2];
#pragma unroll
    for (int i = 0; i < MPW; ++i) acc[i][0] = acc[i][1] = 0.0;
    issue(0, 0);
    for (int ch = 0; ch < nch; ++ch) {
      const int buf = ch & 1;
      if (ch + 1 < nch) {
        issue(ch + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      __syncthreads();
      const cplx* Kc = stage + buf * selems;
      const cplx* Bc = Kc + MX * IC_SC * MX;
      // ---- GEMM1: T = env Kc   (rows Db, real cols 2*ldK, K' = 2 Dk)
      {
        const int ntn1 = (2 * ldK + 7) / 8, mtn1 = (Db + 7) / 8, ks1 = (2 * Dk + 3) / 4;
        for (int nt = warp; nt < ntn1; nt += NW) {
          double c1[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          for (int kk = 0; kk < ks1; ++kk) {
            const int kx = 4 * kk + tig;
            const double bv = ic_gexp(Kc, ldK, Dk, ldK, kx, nt * 8 + gid);
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
              if (mt < mtn1) {
                const int row = mt * 8 + gid;
                const double av = (row < Db && kx < 2 * Dk) ? envd[row * ldE + kx] : 0.0;
                ic_dmma(c1[mt][0], c1[mt][1], av, bv);
              }
            }
          }
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const int row = mt * 8 + gid, col = (nt * 8 + 2 * tig) >> 1;
            if (mt < mtn1 && row < Db && col < ldK) T[row * ldK + col] = mk(c1[mt][0], c1[mt][1]);
          }
        }
      }
      __syncthreads();
      // ---- GEMM2: E += Bc^H T   (K dim kappa = a*SC + sl, T rows kappa)
      if (nt2 < ntn2) {
        const int kdim = Db * IC_SC, ks2 = (2 * kdim + 3) / 4;
        for (int kk = 0; kk < ks2; ++kk) {
          const int kx = 4 * kk + tig;
          const int kap = kx >> 1;
          const int a = kap / IC_SC, sl = kap - a * IC_SC;
          const double bv = ic_gexp(T, Dk2, kdim, Dk2, kx, nt2 * 8 + gid);
#pragma unroll
          for (int i = 0; i < MPW; ++i) {
            const int mt = mg2 + MG * i;
            if (mt < mtn2) {
              const int a2 = mt * 8 + gid;
              double av = 0.0;
              if (a2 < Db2 && kap < kdim) {
                const cplx bb = Bc[a * ldB + sl * Db2 + a2];
                av = (kx & 1) ? -bb.y : bb.x;
              }
              ic_dmma(acc[i][0], acc[i][1], av, bv);
            }
          }
        }
      }
      __syncthreads();  // stage buf and T are rewritten by the next chunk
    }
    // env <- E (interleaved, padded rows; entries beyond Db2 x Dk2 zero)
    for (int e = threadIdx.x; e < MX * ldE; e += IC_THREADS) envd[e] = 0.0;
    __syncthreads();
    if (nt2 < ntn2) {
#pragma unroll
      for (int i = 0; i < MPW; ++i) {
        const int mt = mg2 + MG * i;
        const int row = mt * 8 + gid, col = (nt2 * 8 + 2 * tig) >> 1;
        if (mt < mtn2 && row < Db2 && col < Dk2) {
          envd[row * ldE + 2 * col] = acc[i][0];
          envd[row * ldE + 2 * col + 1] = acc[i][1];
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[inst] = mk(envd[0], envd[1]);
}

size_t tt_inner_chunk_smem() {
  constexpr int MX = 32;
  return sizeof(double) * MX * (2 * MX + 4) + sizeof(cplx) * ((size_t)MX * IC_SC * MX + 2 * 2 * (size_t)MX * IC_SC * MX);
}

// ------------------------------------------------------- tt_evaluate_many
constexpr int EVAL_WARPS = 8;

__global__ void __launch_bounds__(EVAL_WARPS * 32)
eval_warp_kernel(const TTDev tt, const int* __restrict__ idx, long long m, cplx* __restrict__ out) {
  const int inst = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const long long j = (long long)blockIdx.x * EVAL_WARPS + (threadIdx.x >> 5);
  if (j >= m) return;
  const cplx* base = tt.cores + inst * tt.stride;
  // lane owns vec entries lane and lane+32 (bond dims <= 64)
  cplx v0 = mk(0.0, 0.0), v1 = mk(0.0, 0.0);
  {
    const int r1 = tt.bonds[1];
    const int i0 = idx[j * tt.d];
    const cplx* c0 = base + tt.off[0] + (long long)i0 * r1;
    if (lane < r1) v0 = c0[lane];
    if (lane + 32 < r1) v1 = c0[lane + 32];
  }
  for (int k = 1; k < tt.d; ++k) {
    const int ra = tt.bonds[k], rb = tt.bonds[k + 1], n = tt.shape[k];
    const int ik = idx[j * tt.d + k];
    const cplx* G = base + tt.off[k];
    cplx w0 = mk(0.0, 0.0), w1 = mk(0.0, 0.0);
    for (int a = 0; a < ra; ++a) {
      const cplx src = (a < 32) ? v0 : v1;
      cplx va;
      va.x = __shfl_sync(0xffffffffu, src.x, a & 31);
      va.y = __shfl_sync(0xffffffffu, src.y, a & 31);
      const cplx* row = G + ((long long)a * n + ik) * rb;
      if (lane < rb) w0 = cfma(va, row[lane], w0);
      if (lane + 32 < rb) w1 = cfma(va, row[lane + 32], w1);
    }
    v0 = w0;
    v1 = w1;
  }
  if (lane == 0) out[inst * m + j] = v0;
}

}  // namespace

// Site-0 gather and grouped site kernels for the convergence check (used by
// the cross driver).
__global__ void conv_site0_kernel(const cplx* __restrict__ cores, long long stride, long long off0,
                                  int r1, const int* __restrict__ idx, int d, long long m,
                                  cplx* __restrict__ V, long long vstride,
                                  const int* __restrict__ active) {
  const int inst = blockIdx.y;
  if (active && !active[inst]) return;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * r1) return;
  const long long j = e / r1;
  const int c = (int)(e - j * r1);
  V[inst * vstride + e] = cores[inst * stride + off0 + (long long)idx[j * d] * r1 + c];
}

__global__ void conv_site_kernel(const cplx* __restrict__ cores, long long stride, long long offk,
                                 int ra, int n, int rb, const int* __restrict__ perm,
                                 const int* __restrict__ goff, const cplx* __restrict__ Vin,
                                 cplx* __restrict__ Vout, long long vstride,
                                 const int* __restrict__ active) {
  extern __shared__ cplx G[];  // ra x rb slice
  const int inst = blockIdx.y;
  if (active && !active[inst]) return;
  const int s = blockIdx.x;
  const cplx* src = cores + inst * stride + offk;
  for (int e = threadIdx.x; e < ra * rb; e += blockDim.x) {
    const int a = e / rb, c = e - a * rb;
    G[e] = src[((long long)a * n + s) * rb + c];
  }
  // Register tile: a warp advances TS samples at once, lane c owns output
  // columns c and c+32.  The TS input rows are first staged in the warp's own
  // shared-memory slot with coalesced 16-byte loads (each row is contiguous),
  // then every element is a shared-memory broadcast feeding two complex FMAs,
  // and each G element feeds TS.  Accumulation order per output is
  // a = 0..ra-1, as in the reference einsum (tensor_train.py:139).
  constexpr int TS = 8;
  cplx* stage = G + ra * rb + (threadIdx.x >> 5) * TS * ra;
  __syncthreads();
  const int g0 = goff[s], g1 = goff[s + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const cplx* vin = Vin + inst * vstride;
  cplx* vout = Vout + inst * vstride;
  const bool c0 = lane < rb, c1 = lane + 32 < rb;
  for (int t0 = g0 + warp * TS; t0 < g1; t0 += nw * TS) {
    long long js[TS];
#pragma unroll
    for (int q = 0; q < TS; ++q) js[q] = perm[min(t0 + q, g1 - 1)];
#pragma unroll
    for (int q = 0; q < TS; ++q)
      for (int a = lane; a < ra; a += 32) stage[q * ra + a] = __ldg(vin + js[q] * ra + a);
    __syncwarp();
    cplx acc0[TS], acc1[TS];
#pragma unroll
    for (int q = 0; q < TS; ++q) {
      acc0[q] = mk(0.0, 0.0);
      acc1[q] = mk(0.0, 0.0);
    }
    for (int a = 0; a < ra; ++a) {
      const cplx ga = c0 ? G[a * rb + lane] : mk(0.0, 0.0);
      const cplx gb = c1 ? G[a * rb + lane + 32] : mk(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < TS; ++q) {
        const cplx x = stage[q * ra + a];
        acc0[q] = cfma(x, ga, acc0[q]);
        acc1[q] = cfma(x, gb, acc1[q]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < TS; ++q) {
      if (t0 + q < g1) {
        if (c0) vout[js[q] * rb + lane] = acc0[q];
        if (c1) vout[js[q] * rb + lane + 32] = acc1[q];
      }
    }
  }
}

size_t conv_site_smem(int ra, int rb, int threads) {
  return sizeof(cplx) * ((size_t)ra * rb + (size_t)(threads / 32) * 8 * ra);
}

// FP64 tensor-core variant (DMMA, mma.sync m8n8k4 f64: ~37 TFLOP/s on B200
// against ~18.6 for FFMA-class DFMA).  The complex product Vout = Vin G is
// the real GEMM  [Re Im](interleaved) x G'  with
//     G'[2a+p][2c+q] = Re G[a][c]  (p == q),  Im G[a][c] (p=0,q=1),  -Im G[a][c] (p=1,q=0)
// so the interleaved complex128 rows of V are the A operand as stored and
// each accumulator pair (c0, c1) is one complex output.  Block: 8 warps as
// 2 warp rows x 4 warp columns, 64 samples per tile (CD_MT = 4 m-tiles of 8
// rows per warp), N' = 2 rb split over the 4 warp columns (NT 8-wide n-tiles
// each); tiles of gathered rows double-buffered by cp.async.  Summation
// order differs from the scalar kernel by rounding only.
constexpr int CD_ROWS = 64;
constexpr int CD_THREADS = 256;
constexpr int CD_MT = 4;  // m-tiles (8 rows) per warp
static_assert(CD_THREADS % CD_ROWS == 0, "gather: whole threads per row");

__host__ __device__ inline int cd_kp(int ra) { return ((2 * ra + 3) & ~3) + 4; }  // padded row stride (doubles)

// B' fragment of lane (gid, tig) for k-step k0 and n-tile column n0.
__device__ __forceinline__ double cd_bfrag(const cplx* G, int ra, int rb, int k0, int n0, int gid, int tig) {
  const int k = k0 + tig, ncol = n0 + gid;
  const int a = k >> 1, p = k & 1, c = ncol >> 1, q = ncol & 1;
  if (a >= ra || c >= rb) return 0.0;
  const cplx g = G[a * rb + c];
  // -Im by a sign-bit flip (integer pipe; the FP64 pipe feeds the DMMA)
  const double im = (q ? g.y : __longlong_as_double(__double_as_longlong(g.y) ^ (long long)0x8000000000000000ULL));
  return (p == q) ? g.x : im;
}

// KS > 0: all KS x NT B' fragments of the warp live in registers (formed
// once per CTA); KS == 0: formed per k-step from the complex slice.
// Gather modes of the site kernel:
//   CD_PLAIN  row j of Vin (the previous site's sample vectors)
//   CD_G0     site 1: row i_0(j) of the first core (site-0 vectors are core rows)
//   CD_TAB1   site 1 as a table: every first-core row t of the bucket s, output
//             row s * n0 + t of Vout (one product per (i_1, i_0) pair instead
//             of one per sample; used when n0 * n1 <= the sample count)
//   CD_TAB2   site 2 from that table: row i_1(j) * n0 + i_0(j) of Vin
constexpr int CD_PLAIN = 0, CD_G0 = 1, CD_TAB1 = 2, CD_TAB2 = 3;

// WC: warp columns (4, 2 or 1) of the 8 warps; 8 / WC warp rows of
// CD_ROWS / (8 * 8 / WC) m-tiles each.  N' = 2 rb is covered by WC * NT
// 8-wide n-tiles: 4 x {1, 2, 4} wastes up to 37% of the MMAs on bonds that
// are not multiples of 16 (rb = 20: 64 columns for 40), so rb = 17..24
// takes 2 x 3 (48 columns; configs 2/3: conv site 4.16 -> 3.68 ms per
// launch).  Every output entry keeps its k order, so the variants are
// bitwise equal.
template <int NT, int KS, int MODE, int WC>
__global__ void __launch_bounds__(CD_THREADS, 2) conv_site_dmma_kernel(
    const cplx* __restrict__ cores, long long stride, long long offk, int ra, int n, int rb,
    const int* __restrict__ perm, const int* __restrict__ goff, const cplx* __restrict__ Vin,
    cplx* __restrict__ Vout, long long vstride, const int* __restrict__ active,
    long long off0, const int* __restrict__ idx0, int idx_d, int n0) {
  extern __shared__ __align__(16) double cd_smem[];
  const int inst = blockIdx.y;
  if (active && !active[inst]) return;
  const int s = blockIdx.x;
  const int g0 = MODE == CD_TAB1 ? 0 : goff[s], g1 = MODE == CD_TAB1 ? n0 : goff[s + 1];
  if (g0 >= g1) return;
  const int KP = cd_kp(ra);
  const int K2 = 2 * ra;
  const int Kpad = (K2 + 3) & ~3;
  cplx* G = reinterpret_cast<cplx*>(cd_smem);  // ra x rb
  double* stage0 = cd_smem + 2 * ((ra * rb + 1) & ~1);
  double* stage1 = stage0 + CD_ROWS * KP;
  int* rowj = reinterpret_cast<int*>(stage1 + CD_ROWS * KP);  // [2][CD_ROWS]
  const cplx* vin = Vin + inst * vstride;
  cplx* vout = Vout + inst * vstride;
  // site 1 (idx0 set): a sample's input row is row i_0 of the first core,
  // gathered straight from it (no materialised site-0 rows)
  const cplx* core0 = cores + inst * stride + off0;
  const int ntile = (g1 - g0 + CD_ROWS - 1) / CD_ROWS;
  // gather of one tile: CD_THREADS / CD_ROWS threads per row, each loading
  // the row's sample index once and copying every TPR-th 16-byte chunk
  // (the sample index of a row is loaded one tile ahead: sample_j)
  constexpr int TPR = CD_THREADS / CD_ROWS;
  const int grow = threadIdx.x / TPR, gcg = threadIdx.x - grow * TPR;
  auto sample_j = [&](int tile) {
    if constexpr (MODE == CD_TAB1) return min(tile * CD_ROWS + grow, g1 - 1);
    return tile < ntile ? perm[min(g0 + tile * CD_ROWS + grow, g1 - 1)] : 0;
  };
  // source row index of sample j (CD_G0: its i_0; CD_TAB2: i_1 n0 + i_0)
  auto src_index = [&](int j) {
    if constexpr (MODE == CD_G0) return (long long)idx0[(long long)j * idx_d];
    if constexpr (MODE == CD_TAB2)
      return (long long)idx0[(long long)j * idx_d + 1] * n0 + idx0[(long long)j * idx_d];
    return (long long)j;
  };
  // i0 >= 0: the sample's source row, already loaded (gather modes)
  auto issue = [&](int tile, int buf, int j, long long i0) {
    double* st = buf ? stage1 : stage0;
    int* rj = rowj + buf * CD_ROWS;
    const int t0 = g0 + tile * CD_ROWS;
    const int row = grow, cg = gcg;
    if (cg == 0) rj[row] = (t0 + row < g1) ? (MODE == CD_TAB1 ? s * n0 + j : j) : -1;
    const cplx* srow;
    if constexpr (MODE == CD_G0 || MODE == CD_TAB2) {
      if (i0 < 0) i0 = src_index(j);
      srow = (MODE == CD_G0 ? core0 : vin) + i0 * ra;
    } else if constexpr (MODE == CD_TAB1) {
      srow = core0 + (long long)j * ra;
    } else {
      srow = vin + (long long)j * ra;
    }
    const unsigned dst = (unsigned)__cvta_generic_to_shared(st + row * KP);
    for (int ch = cg; ch < ra; ch += TPR)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * ch), "l"(srow + ch));
    cp_async_commit();
  };
  issue(0, 0, sample_j(0), -1);  // first gather overlaps the slice load below
  int jnext = sample_j(1);
  long long inext = -1;
  const cplx* src = cores + inst * stride + offk;
  for (int e = threadIdx.x; e < ra * rb; e += CD_THREADS) {
    const int a = e / rb, c = e - a * rb;
    G[e] = src[((long long)a * n + s) * rb + c];
  }
  // zero the K padding columns once (never written by cp.async)
  for (int e = threadIdx.x; e < 2 * CD_ROWS; e += CD_THREADS) {
    double* st = (e < CD_ROWS) ? stage0 : stage1;
    const int row = e % CD_ROWS;
    for (int k = K2; k < Kpad; ++k) st[row * KP + k] = 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  constexpr int WR = 8 / WC, MT = CD_ROWS / (8 * WR);
  static_assert(WC == 1 || WC == 2 || WC == 4, "8 warps as WR x WC");
  const int wr = warp % WR, wc = warp / WR;
  const int ncol0 = wc * NT * 8;  // first real column (of N') of this warp
  double breg[KS > 0 ? KS : 1][NT];
  if constexpr (KS > 0) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) breg[ks][nt] = cd_bfrag(G, ra, rb, 4 * ks, ncol0 + nt * 8, gid, tig);
  }
  for (int tile = 0; tile < ntile; ++tile) {
    const int buf = tile & 1;
    if (tile + 1 < ntile) {
      issue(tile + 1, buf ^ 1, jnext, inext);
      jnext = sample_j(tile + 2);
      inext = -1;
      cp_async_wait_all_but_one();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    const double* st = buf ? stage1 : stage0;
    const int* rj = rowj + buf * CD_ROWS;
    double acc[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    const double* arow = st + (wr * 8 * MT + gid) * KP + tig;
    // the table's buckets are n0 = N+1 rows (odd): warps whose rows of the
    // last tile are all past it skip their MMAs (table mode only)
    bool skip_mma = false;
    if constexpr (MODE == CD_TAB1) skip_mma = g0 + tile * CD_ROWS + wr * 8 * MT >= g1;
    if constexpr (KS > 0) {
      if (!skip_mma)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        if (4 * ks >= Kpad) break;  // KS rounds the k-steps up; columns past Kpad are not staged
        double av[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) av[mt] = arow[mt * 8 * KP + 4 * ks];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1]) : "d"(av[mt]), "d"(breg[ks][nt]));
      }
    } else {
      for (int k0 = 0; k0 < Kpad; k0 += 4) {
        double av[MT], bv[NT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) av[mt] = arow[mt * 8 * KP + k0];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bv[nt] = cd_bfrag(G, ra, rb, k0, ncol0 + nt * 8, gid, tig);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1]) : "d"(av[mt]), "d"(bv[nt]));
      }
    }
    if constexpr (MODE == CD_G0 || MODE == CD_TAB2) {
      if (tile + 2 < ntile) inext = src_index(jnext);  // jnext has landed by now
    }
    // c0, c1 = C'[row][2 tig], C'[row][2 tig + 1] = one complex output
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int j = rj[wr * 8 * MT + mt * 8 + gid];
      if (j < 0) continue;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = (ncol0 + nt * 8 + 2 * tig) >> 1;
        if (c < rb) vout[(long long)j * rb + c] = mk(acc[mt][nt][0], acc[mt][nt][1]);
      }
    }
    __syncthreads();  // stage buf is refilled two tiles later
  }
}

size_t conv_site_dmma_smem(int ra, int rb) {
  return sizeof(double) * (2 * (size_t)((ra * rb + 1) & ~1) + 2 * (size_t)CD_ROWS * cd_kp(ra)) +
         sizeof(int) * 2 * CD_ROWS;
}

// n-tiles per warp for N' = 2 rb split over 4 warp columns: 1, 2 or 4
int conv_site_dmma_nt(int rb) {
  const int need = (2 * rb + 31) / 32;
  return need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : 0;
}

cudaError_t launch_conv_site_dmma(const cplx* cores, long long stride, long long offk, int ra, int n,
                                  int rb, const int* perm, const int* goff, const cplx* vin, cplx* vout,
                                  long long vstride, const int* active, int n_inst, cudaStream_t s,
                                  long long off0, const int* idx0, int idx_d, int mode, int n0) {
  const size_t smem = conv_site_dmma_smem(ra, rb);
  dim3 grid((unsigned)n, (unsigned)n_inst);
  // warp layout: the fewest 8-wide n-tiles that cover N' = 2 rb
  const int tiles = (2 * rb + 7) / 8;
  int wc = 4, nt = conv_site_dmma_nt(rb);
  if (tiles == 5 || tiles == 6) { wc = 2; nt = 3; }  // rb = 17..24 (1 x 3 for rb = 9..12 measured no gain)
  // register-resident B' when its KS x NT fragments fit in 32 registers
  const int ks_need = ((2 * ra + 3) & ~3) / 4;
  int ks = ks_need <= 4 ? 4 : ks_need <= 8 ? 8 : (ks_need <= 10 && wc == 2) ? 10 : ks_need <= 16 ? 16 : 0;
  if (ks * nt > 32) ks = 0;
  const int code = wc * 10000 + nt * 100 + ks;
#define CD_LAUNCH(NT, KS, MODE, WC)                                                              \
  {                                                                                              \
    cudaError_t e = ensure_max_smem((const void*)conv_site_dmma_kernel<NT, KS, MODE, WC>);       \
    if (e != cudaSuccess) return e;                                                              \
    conv_site_dmma_kernel<NT, KS, MODE, WC><<<grid, CD_THREADS, smem, s>>>(                      \
        cores, stride, offk, ra, n, rb, perm, goff, vin, vout, vstride, active, off0, idx0, idx_d, n0); \
  }
#define CD_CASE(WC, NT, KS)                                                                      \
  case WC * 10000 + NT * 100 + KS:                                                               \
    if (mode == CD_G0) CD_LAUNCH(NT, KS, CD_G0, WC)                                              \
    else if (mode == CD_TAB1) CD_LAUNCH(NT, KS, CD_TAB1, WC)                                     \
    else if (mode == CD_TAB2) CD_LAUNCH(NT, KS, CD_TAB2, WC)                                     \
    else CD_LAUNCH(NT, KS, CD_PLAIN, WC)                                                         \
    break;
  switch (code) {
    CD_CASE(4, 1, 0) CD_CASE(4, 1, 4) CD_CASE(4, 1, 8) CD_CASE(4, 1, 16)
    CD_CASE(4, 2, 0) CD_CASE(4, 2, 4) CD_CASE(4, 2, 8) CD_CASE(4, 2, 16)
    CD_CASE(4, 4, 0) CD_CASE(4, 4, 4) CD_CASE(4, 4, 8)
    CD_CASE(2, 3, 0) CD_CASE(2, 3, 4) CD_CASE(2, 3, 8) CD_CASE(2, 3, 10)
    default:
      return cudaErrorInvalidValue;
  }
#undef CD_CASE
#undef CD_LAUNCH
  return cudaGetLastError();
}

// Fixed-order per-instance sums of |exact - approx| and |exact|.
__global__ void sample_diff_kernel(const cplx* __restrict__ exact, const cplx* __restrict__ approx,
                                   long long m, long long estride, long long astride,
                                   double* __restrict__ out, const int* __restrict__ active) {
  const int inst = blockIdx.x;
  if (active && !active[inst]) return;
  __shared__ double sn[32], sd[32];
  double num = 0.0, den = 0.0;
  const cplx* ex = exact + inst * estride;
  const cplx* ap = approx + inst * astride;
  for (long long j = threadIdx.x; j < m; j += blockDim.x) {
    const cplx e = ex[j];
    num += cabsh(csub(e, ap[j]));
    den += cabsh(e);
  }
  num = warp_sum(num);
  den = warp_sum(den);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sn[w] = num;
    sd[w] = den;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    num = lane < nw ? sn[lane] : 0.0;
    den = lane < nw ? sd[lane] : 0.0;
    num = warp_sum(num);
    den = warp_sum(den);
    if (lane == 0) {
      out[2 * inst] = num;
      out[2 * inst + 1] = den;
    }
  }
}

// ----------------------------------------------------------------- C ABI
static bool tt_shape_ok(const ttp_tt_batch* t) {
  if (!t || t->d < 1 || t->d > TTP_MAX_D || t->n_inst < 0) return false;
  for (int k = 0; k <= t->d; ++k)
    if (t->h_bonds[k] < 1 || t->h_bonds[k] > 64) return false;
  return t->h_bonds[0] == 1 && t->h_bonds[t->d] == 1;
}

extern "C" int ttp_tt_inner(const ttp_tt_batch* bra, const ttp_tt_batch* ket, double* d_out,
                            void* stream) {
  if (!tt_shape_ok(bra) || !tt_shape_ok(ket) || bra->d != ket->d || bra->n_inst != ket->n_inst)
    return ttp_fail(TTP_ERR_INVALID, "tt_inner: bad train batch");
  for (int k = 0; k < bra->d; ++k)
    if (bra->h_shape[k] != ket->h_shape[k])
      return ttp_fail(TTP_ERR_INVALID, "tt_inner: physical shape mismatch");
  if (bra->n_inst == 0) return TTP_OK;
  TTDev b = tt_dev(*bra), k = tt_dev(*ket);
  int maxb = 1, maxk = 1;
  for (int q = 0; q <= bra->d; ++q) {
    maxb = max(maxb, bra->h_bonds[q]);
    maxk = max(maxk, ket->h_bonds[q]);
  }
  const size_t smem = sizeof(cplx) * (size_t)(2 * maxb * maxk);
  const size_t smem_staged = smem + sizeof(cplx) * (size_t)(2 * maxk * maxk + 2 * maxb * maxb);
  int dev = 0, lim = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  static const bool dmma = [] {
    const char* e = ttp_dev_env("TTP_INNER");
    return !(e && strcmp(e, "scalar") == 0);
  }();
  if (dmma && maxb <= 32 && maxk <= 32 && tt_inner_chunk_smem() <= (size_t)lim) {
    TTP_CUDA_CHECK(ensure_max_smem((const void*)tt_inner_chunk_kernel));
    LaunchScope _ls(KC_TT_INNER, (cudaStream_t)stream);
    tt_inner_chunk_kernel<<<bra->n_inst, IC_THREADS, tt_inner_chunk_smem(), (cudaStream_t)stream>>>(
        b, k, reinterpret_cast<cplx*>(d_out));
  } else if (maxb > 32 || maxk > 32) {
    // large bonds: the s-sum of each site split over a 16-CTA cluster
    const size_t ssm = tt_inner_split_smem(maxb, maxk);
    if (ssm > (size_t)lim) return ttp_fail(TTP_ERR_CAPACITY, "tt_inner: bonds too large for shared memory");
    TTP_CUDA_CHECK(ensure_max_smem((const void*)tt_inner_split_kernel));
    TTP_CUDA_CHECK(cudaFuncSetAttribute(tt_inner_split_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(bra->n_inst * TS_G));
    cfg.blockDim = dim3(INNER_THREADS);
    cfg.dynamicSmemBytes = ssm;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = TS_G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LaunchScope _ls(KC_TT_INNER, (cudaStream_t)stream);
    TTP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tt_inner_split_kernel, b, k, reinterpret_cast<cplx*>(d_out), maxb, maxk));
  } else if (smem_staged <= (size_t)lim) {
    TTP_CUDA_CHECK(ensure_max_smem((const void*)tt_inner_staged_kernel));
    LaunchScope _ls(KC_TT_INNER, (cudaStream_t)stream);
    tt_inner_staged_kernel<<<bra->n_inst, INNER_THREADS, smem_staged, (cudaStream_t)stream>>>(
        b, k, reinterpret_cast<cplx*>(d_out), maxb, maxk);
  } else {
    TTP_CUDA_CHECK(ensure_max_smem((const void*)tt_inner_kernel));
    LaunchScope _ls(KC_TT_INNER, (cudaStream_t)stream);
    tt_inner_kernel<<<bra->n_inst, INNER_THREADS, smem, (cudaStream_t)stream>>>(
        b, k, reinterpret_cast<cplx*>(d_out));
  }
  TTP_CUDA_CHECK(cudaGetLastError());
  return TTP_OK;
}

extern "C" size_t ttp_tt_eval_workspace(const ttp_tt_batch*, int64_t) { return 0; }

extern "C" int ttp_tt_eval(const ttp_tt_batch* tt, const int32_t* d_idx, int64_t m, double* d_out,
                           void*, size_t, void* stream) {
  if (!tt_shape_ok(tt) || m < 0) return ttp_fail(TTP_ERR_INVALID, "tt_eval: bad train batch");
  if (m == 0 || tt->n_inst == 0) return TTP_OK;
  TTDev t = tt_dev(*tt);
  dim3 grid((unsigned)((m + EVAL_WARPS - 1) / EVAL_WARPS), (unsigned)tt->n_inst);
  {
    LaunchScope _ls(KC_TT_EVAL, (cudaStream_t)stream);
    eval_warp_kernel<<<grid, EVAL_WARPS * 32, 0, (cudaStream_t)stream>>>(
        t, d_idx, m, reinterpret_cast<cplx*>(d_out));
  }
  TTP_CUDA_CHECK(cudaGetLastError());
  return TTP_OK;
}

extern "C" int ttp_sample_diff(int32_t n_inst, int64_t m, const double* d_exact,
                               const double* d_approx, double* h_out, void* d_ws, size_t ws_bytes,
                               void* stream) {
  if (n_inst < 0 || m < 1) return ttp_fail(TTP_ERR_INVALID, "sample count must be >= 1");
  if (ws_bytes < sizeof(double) * 2 * (size_t)n_inst)
    return ttp_fail(TTP_ERR_WORKSPACE, "sample_diff: workspace too small");
  if (n_inst == 0) return TTP_OK;
  double* sums = reinterpret_cast<double*>(d_ws);
  {
    LaunchScope _ls(KC_SAMPLE_DIFF, (cudaStream_t)stream);
    sample_diff_kernel<<<n_inst, 1024, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const cplx*>(d_exact), reinterpret_cast<const cplx*>(d_approx), m, m, m,
        sums, nullptr);
  }
  TTP_CUDA_CHECK(cudaGetLastError());
  std::string err;
  double* host = new double[2 * (size_t)n_inst];
  cudaError_t e = cudaMemcpyAsync(host, sums, sizeof(double) * 2 * n_inst, cudaMemcpyDeviceToHost,
                                  (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    delete[] host;
    return ttp_record_cuda_error(e);
  }
  for (int i = 0; i < n_inst; ++i) {
    const double num = host[2 * i], den = host[2 * i + 1];
    h_out[i] = (den == 0.0) ? (num == 0.0 ? 0.0 : INFINITY) : num / den;
  }
  delete[] host;
  return TTP_OK;
}
