/* ttpricer_b200.h -- C ABI of the B200-native TT-Fourier pricer hot path.
 *
 * The reference (`ttpricer`, pure Python) has no FFI: its seam is the Python
 * pricing API.  Each entry point below replaces one reference function; the
 * citation names the file:line of the interface it stands in for (paths are
 * relative to the reference's pkg/src/ttpricer/).  The Python package
 * `paper_2203_02804_b200` binds these through ctypes and keeps the reference's
 * Python signatures on top.
 *
 * Conventions
 *  - Every buffer argument named d_* is a DEVICE pointer owned by the caller
 *    (torch tensors in the Python host).  h_* arguments are host pointers.
 *  - complex128 values are interleaved (re, im) doubles, numpy's layout.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Return value is a ttp_status; on error ttp_last_error() holds a
 *    message.  Status codes map 1:1 onto the reference exception classes
 *    (errors.py:4-33).
 *  - All reductions run in a fixed order: results are bitwise reproducible
 *    run to run for a fixed batch layout.
 *  - No entry point calls back into the host and none has a CPU fallback:
 *    without a CUDA device every compute call returns TTP_ERR_CUDA.
 */
#ifndef TTPRICER_B200_H
#define TTPRICER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTP_ABI_VERSION 1

enum ttp_status {
  TTP_OK = 0,
  TTP_ERR_INVALID = 1,     /* ValueError / IndexError                      */
  TTP_ERR_CUDA = 2,        /* CUDA runtime failure or no device            */
  TTP_ERR_SINGULAR = 3,    /* SingularMatrixError   (cross.py:114,346-354) */
  TTP_ERR_MAXVOL_ITER = 4, /* MaxvolIterationError  (cross.py:139,169)     */
  TTP_ERR_BUDGET = 5,      /* OracleBudgetError     (cross.py:286-288)     */
  TTP_ERR_CAPACITY = 6,    /* CapacityError         (pricers.py:209-212)   */
  TTP_ERR_WORKSPACE = 7,   /* caller workspace too small                   */
  TTP_ERR_RESIDUE = 8      /* ResidueError          (pricers.py:221-225)   */
};

enum ttp_oracle_kind {
  TTP_ORACLE_PHI_GBM = 1,   /* phi_grid_oracle     pricers.py:234-240      */
  TTP_ORACLE_VHAT_MIN = 2,  /* payoff_grid_oracle  pricers.py:243-253      */
  TTP_ORACLE_SEPARABLE = 3, /* prod_k w_k[i_k]   (test oracle)             */
  TTP_ORACLE_TT = 4,        /* tt_evaluate_many of a target train (test)   */
  TTP_ORACLE_TABLE = 5      /* dense C-order table lookup (test)           */
};

/* Device oracle descriptor.  Replaces the reference oracle callable
 * convention `(m, d) int64 -> (m,) complex128` (tensor_train.py:11-13) for a
 * batch of n_inst instances that share kind and shape.
 *   PHI_GBM   params per instance: [eta, alpha, n/2, mu[d], C[d*d]]
 *   VHAT_MIN  params per instance: [eta, alpha, n/2, K, conj_flag]
 *   SEPARABLE table per instance: concatenated axis weights; table_offsets[k]
 *   TT        table per instance: packed cores; table_offsets[k], tt_bonds[d+1]
 *   TABLE     table per instance: dense tensor, C order                      */
typedef struct ttp_oracle {
  int32_t kind;
  int32_t d;
  int64_t param_stride;         /* doubles per instance                       */
  const double* params;         /* device                                     */
  int64_t table_stride;         /* complex entries per instance               */
  const double* table;          /* device, interleaved complex                */
  const int64_t* table_offsets; /* device, d+1 entries (complex elements)     */
  const int32_t* tt_bonds;      /* device, d+1 entries                        */
} ttp_oracle;

/* A batch of tensor trains with identical shape and bond dimensions.
 * Core k of instance i starts at d_cores + 2*(i*stride + h_offsets[k]) doubles
 * and has shape (bonds[k], shape[k], bonds[k+1]), row-major complex --
 * the TensorTrain core layout (tensor_train.py:40-75).                      */
typedef struct ttp_tt_batch {
  int32_t d;
  int32_t n_inst;
  const int32_t* h_shape;   /* host, d      */
  const int32_t* h_bonds;   /* host, d+1    */
  const int64_t* h_offsets; /* host, d+1    */
  int64_t stride;           /* complex elements per instance */
  double* d_cores;          /* device       */
} ttp_tt_batch;

/* TT-cross controls; mirrors CrossConfig (cross.py:40-70). */
typedef struct ttp_cross_cfg {
  int32_t bond_dim;
  int32_t max_sweeps;
  double eps_tol;
  int64_t n_conv_samples;
  double maxvol_slack;
  int64_t oracle_call_budget; /* < 0 means None */
} ttp_cross_cfg;

/* One batched TT-cross problem: n_inst instances of the same shape and cfg,
 * each with its own oracle parameters.  Index sets and convergence samples
 * are drawn on the host with numpy's Generator (bit-exact with the reference:
 * cross.py:296-307,402-403 and tensor_train.py:191-194) and passed in.      */
typedef struct ttp_cross_problem {
  int32_t d;
  int32_t n_inst;
  const int32_t* h_shape;      /* host, d                                    */
  const int32_t* d_shape;      /* device, d                                  */
  ttp_oracle oracle;           /* device-resident parameters                 */
  ttp_cross_cfg cfg;
  const int32_t* d_right_init; /* device: initial right sets, packed as
                                  [k=0..d][r_k][d-k] (ttp_cross_layout)      */
  const int32_t* d_conv_idx;   /* device: [M][d] convergence samples        */
  const int32_t* d_conv_perm;  /* device: [d][M] stable argsort per site     */
  const int32_t* d_conv_off;   /* device: per site k, n_k+1 group offsets,
                                  packed at sum_{j<k}(n_j+1)                 */
} ttp_cross_problem;

/* Sizes of the packed per-instance buffers of a cross problem. */
typedef struct ttp_cross_layout {
  int32_t ranks[65];            /* r_0..r_d (d <= 64)                       */
  int64_t core_offsets[65];     /* complex elements, d+1 entries            */
  int64_t core_stride;          /* complex elements per instance            */
  int64_t set_offsets[65];      /* int32 elements, k=0..d, r_k*d each       */
  int64_t set_stride;           /* int32 per instance (left or right)       */
  int64_t max_rows;             /* largest unfolding row count              */
  int32_t max_rank;
} ttp_cross_layout;

/* Per-instance outcome; mirrors CrossReport (cross.py:73-100).  The pivot
 * sets themselves are in d_left / d_right (same packing as d_right_init:
 * left[k][t][0..k-1], right[k][t][0..d-k-1], row stride d).               */
typedef struct ttp_cross_out {
  double* d_cores;           /* device, n_inst * core_stride complex          */
  int32_t* d_left;           /* device, n_inst * set_stride                   */
  int32_t* d_right;          /* device, n_inst * set_stride                   */
  int32_t* h_status;         /* host, n_inst: ttp_status per instance         */
  int32_t* h_error_bond;     /* host, n_inst: bond of a SINGULAR error or -1  */
  int32_t* h_converged;      /* host, n_inst                                  */
  int32_t* h_sweeps;         /* host, n_inst                                  */
  int32_t* h_left_valid;     /* host, n_inst*(d+1): left[k] assigned?         */
  int64_t* h_oracle_calls;   /* host, n_inst                                  */
  int64_t* h_conv_calls;     /* host, n_inst                                  */
  double* h_final_diff;      /* host, n_inst                                  */
} ttp_cross_out;

/* Per-kernel-class launch statistics (diagnostics; see ttp_profile_read). */
typedef struct ttp_kernel_stat {
  char name[32];
  int64_t launches;        /* kernels launched since the last reset          */
  int64_t timed_launches;  /* of which bracketed by CUDA events              */
  double total_ms;         /* summed device time of the timed launches       */
} ttp_kernel_stat;

int ttp_abi_version(void);
const char* ttp_last_error(void);
int ttp_device_count(void);

/* Diagnostics: total kernel launches issued by this library (monotone), and
 * optional CUDA-event timing of every launch on its own stream.  Reading
 * synchronises on the recorded events; enabling adds two event records per
 * launch and no host synchronisation.                                       */
int64_t ttp_launch_count(void);
void ttp_profile_enable(int on);
void ttp_profile_reset(void);
int ttp_profile_read(ttp_kernel_stat* out, int32_t max_entries);

/* K1/K2 fiber evaluators at explicit multi-indices (shared by all
 * instances): d_out[i*m + j] = oracle_i(d_idx[j, :]).
 * Replaces phi_grid_oracle / payoff_grid_oracle calls (pricers.py:234-253). */
int ttp_oracle_eval(const ttp_oracle* oracle, const int32_t* d_shape, int32_t n_inst,
                    const int32_t* d_idx, int64_t m, double* d_out, void* stream);

/* K1/K2 at one sampled unfolding block per instance -- the reference's
 * _block (cross.py:310-332) plus its single oracle call, evaluated by the
 * SAME separable device code the bond kernels use to fill their blocks
 * (fiber_fast.cuh: the v0 path's fiber kernel and the cluster kernels'
 * load_block share phi_part / vhat_part / *_combine, op for op).
 * The sampled axis sits at position `axis` of the multi-index: left tuples
 * have `axis` entries (d_left: n_left x axis int32, row-major), right tuples
 * d - axis - 1 (d_right: n_right x (d - axis - 1)); both are shared by all
 * instances.  Entry (a, s, b) = oracle_i(left[a] ++ (s) ++ right[b]).
 *   layout 0 (left-to-right sweep, cross.py:412-423): the tall matrix has
 *            rows a*n + s and columns b   ((n_left*n) x n_right);
 *   layout 1 (right-to-left sweep, cross.py:424-435): rows s*n_right + b
 *            and columns a                ((n*n_right) x n_left), i.e. the
 *            transpose of _block(..., axis_first=True) that _interp_core
 *            receives (cross.py:428).
 * d_out[i*out_stride + col*rows + row]: each instance's tall matrix,
 * column-major (the bond kernels' layout).                                */
int ttp_eval_fibers(const ttp_oracle* oracle, const int32_t* d_shape, int32_t n_inst, int32_t layout,
                    int32_t axis, int32_t axis_size, const int32_t* d_left, int32_t n_left,
                    const int32_t* d_right, int32_t n_right, double* d_out, int64_t out_stride,
                    void* stream);

/* K7: batched tt_inner(bra, ket) = sum conj(bra[idx]) ket[idx]
 * (tensor_train.py:143-159); d_out holds n_inst complex values.            */
int ttp_tt_inner(const ttp_tt_batch* bra, const ttp_tt_batch* ket, double* d_out,
                 void* stream);

/* K6: tt_evaluate_many at shared indices (tensor_train.py:126-140);
 * d_out[i*m + j].  Workspace: ttp_tt_eval_workspace().                     */
size_t ttp_tt_eval_workspace(const ttp_tt_batch* tt, int64_t m);
int ttp_tt_eval(const ttp_tt_batch* tt, const int32_t* d_idx, int64_t m, double* d_out,
                void* d_ws, size_t ws_bytes, void* stream);

/* Sampled one-norm difference sum|exact-approx| / sum|exact| per instance
 * (tensor_train.py:199-203); h_out[i].                                     */
int ttp_sample_diff(int32_t n_inst, int64_t m, const double* d_exact, const double* d_approx,
                    double* h_out, void* d_ws, size_t ws_bytes, void* stream);

/* K8: dense contour sum  sum_grid phi(-z) vhat(z)  (pricers.py:185-196)
 * for n_inst instances on the grid d_shape (n_terms = prod shape);
 * phi is a PHI_GBM oracle, vhat a VHAT_MIN oracle with conj_flag 0.
 * h_out: n_inst complex sums.                                             */
size_t ttp_dense_workspace(int32_t n_inst, int64_t n_terms);
int ttp_dense_sum(const ttp_oracle* phi, const ttp_oracle* vhat, const int32_t* h_shape,
                  const int32_t* d_shape, int32_t n_inst, double* h_out, void* d_ws,
                  size_t ws_bytes, void* stream);
/* Same sum over the flat C-order term range [first, first + count) (count < 0:
 * to the end) -- the per-rank share of a dense cross-check sharded by flat
 * index range across GPUs; partials combine in rank order. */
int ttp_dense_sum_range(const ttp_oracle* phi, const ttp_oracle* vhat, const int32_t* h_shape,
                        const int32_t* d_shape, int32_t n_inst, int64_t first, int64_t count,
                        double* h_out, void* d_ws, size_t ws_bytes, void* stream);

/* K3-K6 batched TT-cross (cross.py:358-453). */
int ttp_cross_layout_of(int32_t d, const int32_t* h_shape, int32_t bond_dim,
                        ttp_cross_layout* out);
size_t ttp_cross_workspace(const ttp_cross_problem* prob);
int ttp_cross_run(const ttp_cross_problem* prob, ttp_cross_out* out, void* d_ws,
                  size_t ws_bytes, void* stream);

/* maxvol on n_mat independent (rows x cols) complex matrices, row-major
 * like numpy (cross.py:208-230, including _pairwise_refine for rows <= 96,
 * cols <= 8).  max_iters < 0 means None.  h_sel: n_mat*cols sorted rows.  */
size_t ttp_maxvol_workspace(int32_t n_mat, int64_t rows, int32_t cols);
int ttp_maxvol(int32_t n_mat, int64_t rows, int32_t cols, const double* d_mats, double slack,
               int64_t max_iters, double rank_tol, int64_t* h_sel, int32_t* h_status,
               void* d_ws, size_t ws_bytes, void* stream);

/* _column_basis (cross.py:103-119: scipy.linalg.qr(pivoting=True), the rank
 * check of lines 110-118) on n_mat (rows x cols) complex matrices, row-major
 * like numpy, exactly as the bond kernel's global-slice path computes it
 * (TSQR + zlaqp2 on the triangle for 17 <= cols <= 32).  d_q receives n_mat
 * column-major (rows x cols) orthonormal bases, columns in pivot order
 * (the reference's Q up to unimodular column phases).  The shapes that path
 * serves: rows >= 2 cols, cols <= 64, rows * cols * 16 >= 1 MiB. */
size_t ttp_column_basis_workspace(int32_t n_mat, int64_t rows, int32_t cols);
int ttp_column_basis(int32_t n_mat, int64_t rows, int32_t cols, const double* d_mats,
                     double rank_tol, double* d_q, int32_t* h_status, void* d_ws,
                     size_t ws_bytes, void* stream);

/* One-call batch pricing (price_fourier_tt, pricers.py:256-294, for n_inst
 * options sharing grid and configs): the phi cross (PHI_GBM oracle), the
 * vhat cross (VHAT_MIN oracle, conj_flag 1), the bra-conjugated inner
 * product and the prefactor, all on `stream`.  h_prefactor[i] =
 * e^{-r_i (T_i - t)} eta^d / (2 pi)^d.  Outputs: h_price / h_imag (real and
 * imaginary part of the priced contour sum) per instance, and both crosses'
 * cores / index sets / reports through out_phi / out_v exactly as
 * ttp_cross_run.  Instances whose cross failed keep their status in the
 * out structs and get NaN prices.  The seeded host draws (initial right sets,
 * convergence samples) come in the two problems, as for ttp_cross_run.      */
typedef struct ttp_price_problem {
  ttp_cross_problem phi;
  ttp_cross_problem vhat;
  const double* h_prefactor;
} ttp_price_problem;
size_t ttp_price_tt_workspace(const ttp_price_problem* prob);
int ttp_price_tt_batch(const ttp_price_problem* prob, ttp_cross_out* out_phi, ttp_cross_out* out_v,
                       double* h_price, double* h_imag, void* d_ws, size_t ws_bytes, void* stream);

/* K9: Monte Carlo estimate of the discounted min-option payoff
 * (price_monte_carlo, pricers.py:297-350) for n_inst instances of dimension
 * d, n_samples paths each.  Parameters per instance (doubles, stride
 * param_stride >= ttp_mc_param_count(d)):
 *   [s0 d][drift d][vol d][rates d][sigma d][chol d*d (row-major, lower)]
 *   [strike][disc][dt]
 * with drift = (rates - sigma^2/2) T, vol = sigma sqrt(T), disc =
 * exp(-r (T - t)), dt = T / n_steps (pricers.py:313-330).
 * scheme 0 = terminal_exact, 1 = euler_path (n_steps Euler steps).
 * Normals: Philox4x32-10 (Random123) keyed by h_seeds[inst], counter =
 * (sample lo, sample hi, draw, 0x4D43), two 53-bit uniforms per call and
 * Box-Muller.  The stream is a function of (seed, sample) only, so results
 * do not depend on chunking or grid shape; partial sums reduce in a fixed
 * order.  h_out: n_inst x 2 doubles = (sum, sum of squares) of the
 * discounted payoffs.                                                      */
int32_t ttp_mc_param_count(int32_t d);
size_t ttp_mc_workspace(int32_t n_inst, int64_t n_samples);
int ttp_mc_price(const double* d_params, int64_t param_stride, int32_t d, int32_t n_inst,
                 int64_t n_samples, const uint64_t* h_seeds, int32_t scheme, int32_t n_steps,
                 double* h_out, void* d_ws, size_t ws_bytes, void* stream);
/* Philox4x32-10 block for known-answer tests: h_ctr[4], h_key[2] -> h_out[4]. */
int ttp_philox4x32(const uint32_t* h_ctr, const uint32_t* h_key, uint32_t* h_out);

#ifdef __cplusplus
}
#endif

#endif /* TTPRICER_B200_H */
