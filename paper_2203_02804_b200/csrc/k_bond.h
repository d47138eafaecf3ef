// Bond kernel job description (internal).
#pragma once

#include <cuda_runtime.h>
#include "ttp_common.cuh"
#include "ttp_internal.h"

// one-CTA kernel: blocks of at most this many bytes run the 128-thread shape
#ifndef V0_SMALL_BYTES
#define V0_SMALL_BYTES (64 << 10)
#endif

struct BondJob {
  int m, r;               // tall block rows / cols (m >= r)
  long long mat_stride;   // complex elements per instance for A, W, B
  cplx* A;                // sampled block (col-major, ld m); overwritten by Q
  cplx* W;                // working copy
  cplx* B;                // maxvol matrix
  int* iwork;             // 2m ints per instance
  long long iw_stride;
  double* dwork;          // 2m doubles per instance
  long long dw_stride;
  const int* active;      // optional per-instance mask
  int* status;            // per-instance ttp_status (skips instances != OK)
  int* err_bond;          // optional: bond index recorded with an error
  int bond;               // bond number of this launch (SingularMatrixError.bond)
  double rank_tol;        // 0 on the cross path (cross.py:343), 1e-12 for maxvol()
  long long max_iters;    // < 0: None  (10 * m)
  double slack;
  int pairwise;           // allow _pairwise_refine (m <= 96, r <= 8)
  int* sel_out;           // optional: sorted selection per instance
  long long sel_stride;
  // factor output (write_mode 0: none, 1: left-to-right core, 2: right-to-left core)
  int write_mode;
  cplx* core_out;         // core base (already offset to this site)
  long long core_stride;  // complex elements per instance
  // nested index-set update
  int* set_out;           // destination set base (all instances)
  const int* set_in;      // parent set base
  long long set_stride;   // ints per instance
  long long set_out_off, set_in_off;
  int set_d;              // row stride of the packed sets (= d)
  int klen;               // tuple length of the new set
  int na;                 // axis size (left-to-right decode)
  int rr;                 // right count (right-to-left decode)
};

size_t bond_smem_bytes(int m, int r);
cudaError_t launch_bond(const BondJob& job, int n_inst, cudaStream_t s);

// Cluster variant (k_cluster.cu): one thread-block cluster per instance, the
// block resident in distributed shared memory.
// Two instantiations (k_cluster_impl.cuh): ck_lat (512 threads, one CTA
// per SM; latency: single options, shared-memory clusters) and ck_tp (256
// threads, two CTAs per SM; throughput batches of global-slice clusters,
// where two instances per SM hide each other's barrier and latency stalls).

struct ClusterJob {
  BondJob b;              // shared fields (A/W/B/iwork/dwork unused)
  int cl;                 // CTAs per cluster (1, 2, 4, 8, 16)
  int src_mode;           // 0: evaluate fibers from `oracle`/`fiber`; 1: numpy row-major `src`
  int fiber_fast;         // src_mode 0: separable evaluation allowed (fiber_fast.cuh)
  int q_wy;               // form Q in compact-WY form (else zung2r rounds)
  int fused_starts;       // both dominant-row starts in one read-only pass sequence
  int fused_qr;           // column basis: each update pass also forms the next step's partials
  int basis_only;         // stop after the column basis (ttp_column_basis)
  int tsqr;               // global-slice mode: column basis by TSQR + zlaqp2 on the triangle (k_tsqr.cuh)
  int big;                // bit 0: per-row arrays, bit 1: B[sel,:] in global memory (set by the launcher)
  cplx* Sg;               // global-slice mode: B buffer (holds B[sel,:] in big mode), stride wg_stride
  OracleDev oracle;
  FiberJob fiber;         // index-set views and geometry (out/ld unused)
  const cplx* src;
  long long src_stride;   // complex elements per instance (src_mode 1)
  cplx* Qg;               // global Q buffer, m x r column-major per instance
  long long q_stride;
  // Global-slice mode: when Wg != nullptr each CTA's row slice lives in
  // global memory (L2-resident for a bounded number of concurrent clusters)
  // at Wg + inst*wg_stride + rank*ms*r, and only the small state uses shared
  // memory, so smaller clusters (more instances in flight) are possible.
  cplx* Wg;
  long long wg_stride;
};

#ifdef TTP_DEV
#define TTP_DEV_CLUSTER_API int debug_phase_clocks(int enable, int64_t* out, int32_t n); int debug_inst_times(int64_t* out, int32_t n);
#else
#define TTP_DEV_CLUSTER_API
#endif
#define TTP_CLUSTER_API                                                                     \
  size_t cluster_smem_bytes(int m, int r, int C, bool global_slice = false, int big = 0);   \
  int pick_cluster_size(int m, int r, size_t smem_limit); /* 0 if no cluster fits */        \
  int max_active_clusters(const ClusterJob& job);                                           \
  cudaError_t launch_cluster_bond(const ClusterJob& job, int n_inst, cudaStream_t s);       \
  TTP_DEV_CLUSTER_API
namespace ck_lat { TTP_CLUSTER_API }
namespace ck_tp { TTP_CLUSTER_API }
