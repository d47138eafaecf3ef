// Column basis by tall-skinny QR (global-slice mode of cluster_bond_kernel).
//
// The reference's _column_basis is scipy's pivoted QR, zgeqp3 on the m x r
// block (cross.py:103-119).  Restated step by step on the device (the
// zlaqp2 path in column_basis above), each of its r steps streams the whole
// m x r block through HBM: ~35 of the ~95 block passes a bond makes.  The
// pivot choices of zgeqp3 depend on the block only through its Gram matrix
// A^H A, which the triangular factor of an UNPIVOTED QR carries exactly
// (A = Q1 R1  =>  A^H A = R1^H R1).  So:
//
//   1. TSQR: every warp factors its own contiguous rows independently -- a
//      dense Householder QR of its first r rows, then 16-row chunks each
//      stacked under the running triangle (structured Householder QR of
//      [R; X], flat tree).  Lane k owns column k: the chunk lives in the
//      lane's registers and the r x r triangle in the warp's slice of tensor
//      memory (TMEM, tcgen05.ld/st; 32 lanes x 128 columns per warp), so a
//      step needs no shuffles and no block barrier -- only the reflector's
//      owner lane publishing it through shared memory.  The block is read
//      once and the reflectors written once.
//   2. The warps' triangles merge by a binary tree (structured QR of
//      [R_a; R_b]), then across the cluster into CTA 0, which runs zlaqp2 --
//      the reference's pivot rule, partial-norm downdates and recompute test
//      -- on the final r x r triangle: pivots P, Q_p, R_p.
//   3. Q = Q_tsqr Q_p by one reverse pass over the stored reflectors (tree
//      first, then every warp's own rows): A P = Q R_p with orthonormal Q,
//      the reference's Q up to unimodular column phases when the pivots agree
//      (exactly so in exact arithmetic), and every later decision -- maxvol
//      starts, swaps, slogdet, the core Q Q[sel]^-1 -- is invariant under
//      those phases.
//
// Both Householder QRs are backward stable, so Q differs from the
// restatement's only at rounding level -- the level at which the reference
// differs from itself across BLAS builds.  Every reduction
// runs in a fixed order, so results are bitwise reproducible and do not
// depend on the batch.
//
// Applies to r <= 32 (lane = column); wider blocks keep the restated zlaqp2.

#ifndef TW_LC_DEF
#define TW_LC_DEF 8
#endif
constexpr int TW_LC = TW_LC_DEF;           // structured chunk rows (registers per lane)
constexpr int TW_COLS = 128;               // TMEM columns per warp: 32 rows x 4 words
constexpr int TW_NCOLS = TW_COLS * CW / 4;  // TMEM columns per CTA (4 warps share a column range)
constexpr int TW_LEVELS = (CW >= 16) ? 4 : (CW >= 8) ? 3 : (CW >= 4) ? 2 : 1;
constexpr int TW_TC = (32 + TW_LC - 1) / TW_LC;  // chunks per merged triangle (r <= 32)

// ---- tensor memory: row j of the warp's r x r matrix at columns 4j..4j+3
__device__ __forceinline__ uint32_t tw_region(uint32_t tbase) {
  const int w = threadIdx.x >> 5;
  return tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * TW_COLS);
}
__device__ __forceinline__ cplx tm_ld(uint32_t a, int row) {
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a + 4u * row));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return mk(__hiloint2double((int)r1, (int)r0), __hiloint2double((int)r3, (int)r2));
}
__device__ __forceinline__ void tm_st(uint32_t a, int row, cplx v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + 4u * row),
               "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y)));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// four consecutive rows
__device__ __forceinline__ void tm_ld4(uint32_t a, int row0, cplx (&v)[4]) {
  uint32_t q[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
        "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
      : "r"(a + 4u * row0));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i)
    v[i] = mk(__hiloint2double((int)q[4 * i + 1], (int)q[4 * i]), __hiloint2double((int)q[4 * i + 3], (int)q[4 * i + 2]));
}
__device__ __forceinline__ void tm_st4(uint32_t a, int row0, const cplx (&v)[4]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(a + 4u * row0),
      "r"(__double2loint(v[0].x)), "r"(__double2hiint(v[0].x)), "r"(__double2loint(v[0].y)), "r"(__double2hiint(v[0].y)),
      "r"(__double2loint(v[1].x)), "r"(__double2hiint(v[1].x)), "r"(__double2loint(v[1].y)), "r"(__double2hiint(v[1].y)),
      "r"(__double2loint(v[2].x)), "r"(__double2hiint(v[2].x)), "r"(__double2loint(v[2].y)), "r"(__double2hiint(v[2].y)),
      "r"(__double2loint(v[3].x)), "r"(__double2hiint(v[3].x)), "r"(__double2loint(v[3].y)), "r"(__double2hiint(v[3].y)));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Asynchronous forms: the load's registers are handed through the wait as
// in/out operands, so no use can be scheduled before the data has landed.
struct TmRow {
  uint32_t q0, q1, q2, q3;
};
__device__ __forceinline__ void tm_ld_async(uint32_t a, int row, TmRow& t) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(t.q0), "=r"(t.q1), "=r"(t.q2), "=r"(t.q3) : "r"(a + 4u * row));
}
__device__ __forceinline__ cplx tm_wait_row(TmRow& t) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(t.q0), "+r"(t.q1), "+r"(t.q2), "+r"(t.q3) :: "memory");
  return mk(__hiloint2double((int)t.q1, (int)t.q0), __hiloint2double((int)t.q3, (int)t.q2));
}
__device__ __forceinline__ void tm_st_async(uint32_t a, int row, cplx v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + 4u * row),
               "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y))
               : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// zlarfg from the squared norm (fast form in the safe range, else the
// scaled LAPACK form over the values themselves, supplied by ssq)
__device__ __forceinline__ Reflector tw_zlarfg(cplx alpha, double s2, double mx, Ssq ss) {
  if (mx > 1e-140 && mx < 1e140) return zlarfg_fast(alpha, s2);
  return zlarfg_core(alpha, ssq_norm(ss));
}

// ---- one structured chunk step sequence (forward): [R; X] -> [R'; 0] with
// R in TMEM (lane = column), X[i] = chunk row i of this lane's column.  On
// return X holds the chunk's reflector vectors (column j = reflector j);
// taus to tau_g[j].  vb: this warp's 2 x (TW_LC + 2) broadcast slots.
// Steps j < j0 are skipped: the caller guarantees the chunk is zero in
// columns < j0 (rows of a triangle), where every reflector is the identity
// (tau = 0 exactly), so skipping them changes no bit.  Per step, the next
// triangle row is loaded from TMEM while this one is used, and rows are
// stored back without waiting (one wait at the end).
__device__ __forceinline__ void tw_chunk_fwd(uint32_t ta, cplx (&X)[TW_LC], int r, cplx* vb, cplx* tau_g,
                                             int j0 = 0) {
  const int lane = threadIdx.x & 31;
  // The owner lane publishes its raw column x and the reflector's scale
  // (v = scal x); the others fold scal into their two scalars, and the owner
  // scales its own column once at the end, so a step costs the owner a norm
  // and zlarfg only.
  cplx myscal = mk(1.0, 0.0);
  TmRow nx;
  if (j0 < r) tm_ld_async(ta, j0, nx);
  for (int j = j0; j < r; ++j) {
    cplx Rj = tm_wait_row(nx);
    if (j + 1 < r) tm_ld_async(ta, j + 1, nx);
    cplx* b = vb + (j & 1) * (TW_LC + 2);
    if (lane == j) {
      double p[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < TW_LC; ++i) {
        p[i & 3] = fma(X[i].x, X[i].x, fma(X[i].y, X[i].y, p[i & 3]));
        b[i] = X[i];
      }
      const double s2 = (p[0] + p[1]) + (p[2] + p[3]);
      Reflector h;
      if (s2 > 1e-280 && s2 < 1e280) {
        h = zlarfg_fast(Rj, s2);
      } else {  // tiny or huge column: the scaled LAPACK form
        Ssq ss = ssq_init();
#pragma unroll
        for (int i = 0; i < TW_LC; ++i) ssq_addc(ss, X[i]);
        h = zlarfg_core(Rj, ssq_norm(ss));
      }
      myscal = reflector_scale(h);
      b[TW_LC] = h.tau;
      b[TW_LC + 1] = myscal;
      Rj = mk(h.beta, 0.0);
      tau_g[j] = h.tau;
    }
    __syncwarp();
    if (lane > j && lane < r) {
      // w = R(j,k) + v^H x_k = R(j,k) + conj(scal) (x^H x_k);  x_k -= (conj(tau) w scal) x
      const cplx ct = cconj(b[TW_LC]), sc = b[TW_LC + 1];
      cplx w0 = mk(0.0, 0.0), w1 = mk(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < TW_LC; i += 2) {
        w0 = cfmac(b[i], X[i], w0);
        w1 = cfmac(b[i + 1], X[i + 1], w1);
      }
      const cplx w = cfmac(sc, cadd(w0, w1), Rj);
      const cplx tw = cmul(ct, w);
      Rj = csub(Rj, tw);
      const cplx tws = cmul(tw, sc);
#pragma unroll
      for (int i = 0; i < TW_LC; ++i) X[i] = csub(X[i], cmul(tws, b[i]));
    }
    __syncwarp();
    tm_st_async(ta, j, Rj);
  }
  if (lane >= j0 && lane < r)
#pragma unroll
    for (int i = 0; i < TW_LC; ++i) X[i] = cmul(X[i], myscal);
  tm_wait_st();
}

// ---- reverse of one structured chunk: [Z; W] <- H_j0 ... H_{r-1} [Z; W]
// (reflectors applied from the last), Z in TMEM, W[i] chunk row i of this
// lane's column.  Reflector j's chunk part at V[j * ldv + i] (i < nrow),
// tau at tau_g[j]; every lane reads the same values (L1 broadcast), one step
// ahead.  Steps j < j0 are identities (see tw_chunk_fwd) and skipped.
__device__ __forceinline__ void tw_chunk_rev(uint32_t ta, cplx (&W)[TW_LC], int r, const cplx* V, long long ldv,
                                             int nrow, const cplx* tau_g, int j0 = 0) {
  const int lane = threadIdx.x & 31;
  // the next reflector's values are loaded one step ahead (L1 hits)
  cplx vn[TW_LC];
  cplx tn;
  auto loadv = [&](int j) {
#pragma unroll
    for (int i = 0; i < TW_LC; ++i) vn[i] = i < nrow ? V[(long long)j * ldv + i] : mk(0.0, 0.0);
    tn = tau_g[j];
  };
  TmRow nz;
  if (j0 < r) {
    loadv(r - 1);
    tm_ld_async(ta, r - 1, nz);
  }
  for (int j = r - 1; j >= j0; --j) {
    cplx v[TW_LC];
#pragma unroll
    for (int i = 0; i < TW_LC; ++i) v[i] = vn[i];
    const cplx tau = tn;
    cplx Zj = tm_wait_row(nz);
    if (j > j0) {
      loadv(j - 1);
      tm_ld_async(ta, j - 1, nz);
    }
    if (lane < r) {
      cplx w0 = Zj, w1 = mk(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < TW_LC; i += 2) {
        w0 = cfmac(v[i], W[i], w0);
        w1 = cfmac(v[i + 1], W[i + 1], w1);
      }
      const cplx tw = cmul(tau, cadd(w0, w1));
      Zj = csub(Zj, tw);
#pragma unroll
      for (int i = 0; i < TW_LC; ++i) W[i] = csub(W[i], cmul(tw, v[i]));
    }
    __syncwarp();
    tm_st_async(ta, j, Zj);
  }
  tm_wait_st();
}

// ---- dense Householder QR of the r x r block in TMEM (rows padded to a
// multiple of 4 with zeros).  Reflector j's part below row j goes to
// V[j * ldv + row] (global, in place of the block) and its tau to tau_g[j];
// afterwards TMEM holds R on and above the diagonal.
__device__ void tw_dense_fwd(uint32_t ta, int r, cplx* vb, cplx* V, long long ldv, cplx* tau_g) {
  const int lane = threadIdx.x & 31;
  const int r4 = (r + 3) & ~3;
  for (int j = 0; j < r; ++j) {
    const int b0 = j & ~3;
    // norm of column j below the diagonal (every lane for its own column;
    // lane j's is the one used)
    double s2 = 0.0, mx = 0.0;
    cplx alpha = mk(0.0, 0.0);
    for (int rb = b0; rb < r4; rb += 4) {
      cplx v[4];
      tm_ld4(ta, rb, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = rb + i;
        if (row == j) alpha = v[i];
        if (row > j && row < r) {
          s2 = fma(v[i].x, v[i].x, fma(v[i].y, v[i].y, s2));
          mx = fmax(mx, fmax(fabs(v[i].x), fabs(v[i].y)));
        }
      }
    }
    const double mxw = __shfl_sync(0xffffffffu, mx, j);
    Ssq ss = ssq_init();
    if (!(mxw > 1e-140 && mxw < 1e140)) {  // out of the safe range: scaled sum of squares
      for (int rb = b0; rb < r4; rb += 4) {
        cplx v[4];
        tm_ld4(ta, rb, v);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (rb + i > j && rb + i < r) ssq_addc(ss, v[i]);
      }
    }
    cplx scal = mk(0.0, 0.0);
    double beta = 0.0;
    if (lane == j) {
      const Reflector h = tw_zlarfg(alpha, s2, mx, ss);
      scal = reflector_scale(h);
      beta = h.beta;
      vb[r] = h.tau;
      tau_g[j] = h.tau;
    }
    __syncwarp();
    // scale column j below the diagonal into v (lane j), publish v
    for (int rb = b0; rb < r4; rb += 4) {
      cplx v[4];
      tm_ld4(ta, rb, v);
      if (lane == j) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = rb + i;
          if (row == j) v[i] = mk(beta, 0.0);
          if (row > j && row < r) {
            v[i] = cmul(v[i], scal);
            vb[row] = v[i];
            V[(long long)j * ldv + row] = v[i];
          }
        }
      }
      __syncwarp();
      tm_st4(ta, rb, v);
    }
    if (lane == j) vb[j] = mk(1.0, 0.0);
    __syncwarp();
    const cplx ct = cconj(vb[r]);
    // w = v^H R(j:, k) for lanes k > j, then R(j:, k) -= conj(tau) w v
    cplx w = mk(0.0, 0.0);
    for (int rb = b0; rb < r4; rb += 4) {
      cplx v[4];
      tm_ld4(ta, rb, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = rb + i;
        if (row >= j && row < r) w = cfmac(vb[row], v[i], w);
      }
    }
    const cplx tw = cmul(ct, w);
    for (int rb = b0; rb < r4; rb += 4) {
      cplx v[4];
      tm_ld4(ta, rb, v);
      if (lane > j && lane < r) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = rb + i;
          if (row >= j && row < r) v[i] = csub(v[i], cmul(tw, vb[row]));
        }
      }
      __syncwarp();
      tm_st4(ta, rb, v);
    }
    __syncwarp();
  }
}

// ---- reverse of the dense block: TMEM Z <- H_0 ... H_{r-1} Z (the block's
// Q rows when Z is the triangle's Q factor)
__device__ void tw_dense_rev(uint32_t ta, int r, cplx* vb, const cplx* V, long long ldv, const cplx* tau_g) {
  const int lane = threadIdx.x & 31;
  const int r4 = (r + 3) & ~3;
  for (int j = r - 1; j >= 0; --j) {
    const int b0 = j & ~3;
    for (int row = j + 1 + lane; row < r; row += 32) vb[row] = V[(long long)j * ldv + row];
    if (lane == 0) vb[j] = mk(1.0, 0.0);
    __syncwarp();
    const cplx tau = tau_g[j];
    cplx w = mk(0.0, 0.0);
    for (int rb = b0; rb < r4; rb += 4) {
      cplx v[4];
      tm_ld4(ta, rb, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = rb + i;
        if (row >= j && row < r) w = cfmac(vb[row], v[i], w);
      }
    }
    const cplx tw = cmul(tau, w);
    for (int rb = b0; rb < r4; rb += 4) {
      cplx v[4];
      tm_ld4(ta, rb, v);
      if (lane < r) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = rb + i;
          if (row >= j && row < r) v[i] = csub(v[i], cmul(tw, vb[row]));
        }
      }
      __syncwarp();
      tm_st4(ta, rb, v);
    }
    __syncwarp();
  }
}

// Sixteen per-lane values summed over the warp (transposed butterfly):
// afterwards lane L holds the sum of value (L >> 1) & 15.  Fixed order.
template <class Op>
__device__ __forceinline__ double tw_tsum16(const double (&v)[16], Op op) {
  const int lane = threadIdx.x & 31;
  double k8[8], k4[4], k2[2];
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int j = 0; j < 8; ++j) k8[j] = op(b4 ? v[j + 8] : v[j], __shfl_xor_sync(0xffffffffu, b4 ? v[j] : v[j + 8], 16));
#pragma unroll
  for (int j = 0; j < 4; ++j) k4[j] = op(b3 ? k8[j + 4] : k8[j], __shfl_xor_sync(0xffffffffu, b3 ? k8[j] : k8[j + 4], 8));
#pragma unroll
  for (int j = 0; j < 2; ++j) k2[j] = op(b2 ? k4[j + 2] : k4[j], __shfl_xor_sync(0xffffffffu, b2 ? k4[j] : k4[j + 2], 4));
  const double k1 = op(b1 ? k2[1] : k2[0], __shfl_xor_sync(0xffffffffu, b1 ? k2[0] : k2[1], 2));
  return op(k1, __shfl_xor_sync(0xffffffffu, k1, 1));
}

// zlaqp2 + zung2r on the final r x r triangle (r <= 32), all warps of the
// CTA: lane = row, warp w owns columns j = w (mod CW).  Every warp derives
// the pivot (first maximum of the squared partial norms) and the reflector
// itself from shared memory, identically, so a step needs two block
// barriers.  The reference's rules (zgeqp3 -> zlaqp2): partial-norm downdate with the
// tol3z recompute test on squared norms as in column_basis, the rank
// check of _column_basis (cross.py:110-118).
__device__ void ts_qrcp_block(CC& c, cplx* R, cplx* Z, double rank_tol, int* singular) {
  const int r = c.r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < r; j += CW) {
    Ssq sq = ssq_init();
    if (lane < r) ssq_addc(sq, R[(long long)j * r + lane]);
    sq = warp_ssq(sq);
    if (lane == 0) {
      const double n2 = ssq_norm2(sq);
      c.cn1[j] = n2;
      c.cn2[j] = n2;
      c.colmap[j] = j;
    }
  }
  __syncthreads();
  for (int i = 0; i < r; ++i) {
    ArgMax am{-1.0, LLONG_MAX};
    if (i + lane < r) am = ArgMax{c.cn1[i + lane], i + lane};
    am = warp_argmax(am);
    const int p = (int)am.key;
    __syncthreads();  // every warp has read cn1
    if (p != i) {
      if ((int)threadIdx.x < r) {
        const int t = threadIdx.x;
        const cplx a = R[(long long)p * r + t];
        R[(long long)p * r + t] = R[(long long)i * r + t];
        R[(long long)i * r + t] = a;
      }
      if (threadIdx.x == 0) {
        const int t = c.colmap[p];
        c.colmap[p] = c.colmap[i];
        c.colmap[i] = t;
        c.cn1[p] = c.cn1[i];
        c.cn2[p] = c.cn2[i];
      }
      __syncthreads();
    }
    // reflector of column i (every warp, identically)
    const cplx x = (lane < r) ? R[(long long)i * r + lane] : mk(0.0, 0.0);
    const bool below = lane > i && lane < r;
    double s2 = below ? cabs2(x) : 0.0, mx = below ? fmax(fabs(x.x), fabs(x.y)) : 0.0;
    s2 = warp_sum(s2);
    mx = warp_max(mx);
    const cplx alpha = mk(__shfl_sync(0xffffffffu, x.x, i), __shfl_sync(0xffffffffu, x.y, i));
    Reflector h;
    if (mx > 1e-140 && mx < 1e140) {
      h = zlarfg_fast(alpha, s2);
    } else {
      Ssq sq = ssq_init();
      if (below) ssq_addc(sq, x);
      h = zlarfg_core(alpha, ssq_norm(warp_ssq(sq)));
    }
    const cplx scal = reflector_scale(h);
    const cplx v = below ? cmul(x, scal) : mk(lane == i ? 1.0 : 0.0, 0.0);
    const cplx ct = cconj(h.tau);
    for (int j = i + 1 + ((warp - (i + 1)) % CW + CW) % CW; j < r; j += CW) {
      cplx a = (lane < r) ? R[(long long)j * r + lane] : mk(0.0, 0.0);
      const cplx w = warp_sum(lane >= i ? cmulc(v, a) : mk(0.0, 0.0));
      if (lane >= i && lane < r) {
        a = csub(a, cmul(cmul(ct, w), v));
        R[(long long)j * r + lane] = a;
      }
      const cplx rij = mk(__shfl_sync(0xffffffffu, a.x, i), __shfl_sync(0xffffffffu, a.y, i));
      const double s1 = c.cn1[j];
      if (s1 != 0.0) {
        const double s1n = fmax(s1 - cabs2(rij), 0.0);
        if (s1n <= TOL3Z * c.cn2[j]) {
          Ssq sq = ssq_init();
          if (lane > i && lane < r) ssq_addc(sq, a);
          const double n2 = (i < r - 1) ? ssq_norm2(warp_ssq(sq)) : 0.0;
          if (lane == 0) {
            c.cn1[j] = n2;
            c.cn2[j] = n2;
          }
        } else if (lane == 0) {
          c.cn1[j] = s1n;
        }
      }
    }
    if (warp == i % CW) {
      if (below) R[(long long)i * r + lane] = v;
      if (lane == i) R[(long long)i * r + i] = mk(h.beta, 0.0);
      if (lane == 0) {
        c.tau[i] = h.tau;
        c.betas[i] = fabs(h.beta);
      }
    }
    __syncthreads();
  }
  double lead = 0.0, mn = INFINITY;
  for (int t = 0; t < r; ++t) {
    lead = fmax(lead, c.betas[t]);
    mn = fmin(mn, c.betas[t]);
  }
  if (threadIdx.x == 0) *singular = (lead == 0.0 || mn < rank_tol * lead) ? 1 : 0;
  // Z = H_0 ... H_{r-1} [I] (zung2r), columns over the warps
  for (int j = warp; j < r; j += CW)
    if (lane < r) Z[(long long)j * r + lane] = mk(lane == j ? 1.0 : 0.0, 0.0);
  __syncthreads();
  for (int i = r - 1; i >= 0; --i) {
    const cplx v = (lane > i && lane < r) ? R[(long long)i * r + lane] : mk(lane == i ? 1.0 : 0.0, 0.0);
    const cplx ti = c.tau[i];
    for (int j = i + ((warp - i) % CW + CW) % CW; j < r; j += CW) {
      cplx z = (lane < r) ? Z[(long long)j * r + lane] : mk(0.0, 0.0);
      const cplx w = warp_sum(lane >= i ? cmulc(v, z) : mk(0.0, 0.0));
      if (lane >= i && lane < r) Z[(long long)j * r + lane] = csub(z, cmul(cmul(ti, w), v));
    }
    __syncthreads();
  }
}

// ---- global scratch of one CTA (complex elements, after the C r^2 of B[sel,:])
struct TwScratch {
  cplx *taus, *ttree, *tx, *Rx, *Zx, *PV, *XV;
};
__device__ __forceinline__ int tw_nch(int rows, int r) { return rows > r ? (rows - r + TW_LC - 1) / TW_LC : 0; }
__device__ __forceinline__ long long tw_tstride(int ms, int r, int C) {
  const int nch = tw_nch((ms + CW - 1) / CW, r);
  const long long rr = (long long)r * r;
  return (long long)CW * (1 + nch) * r + (long long)CW * TW_LEVELS * TW_TC * r + (long long)C * TW_TC * r +
         2LL * CW * rr + (long long)CW * TW_LEVELS * TW_TC * TW_LC * r + (long long)C * TW_TC * TW_LC * r;
}
__device__ __forceinline__ TwScratch tw_scratch(cplx* base, int ms, int r, int C) {
  const int nch = tw_nch((ms + CW - 1) / CW, r);
  const long long rr = (long long)r * r;
  TwScratch s;
  s.taus = base;                                        // [CW][1 + nch][r]  dense block, chunks
  s.ttree = s.taus + (long long)CW * (1 + nch) * r;       // [CW][TW_LEVELS][TW_TC][r]
  s.tx = s.ttree + (long long)CW * TW_LEVELS * TW_TC * r;  // [C][TW_TC][r]  cross-CTA merges (CTA 0)
  s.Rx = s.tx + (long long)C * TW_TC * r;                  // [CW][r][r] exported triangles (column-major)
  s.Zx = s.Rx + CW * rr;                                   // [CW][r][r] handed-down Z factors
  s.PV = s.Zx + CW * rr;                                   // [CW][TW_LEVELS][TW_TC][r][TW_LC] tree reflectors
  s.XV = s.PV + (long long)CW * TW_LEVELS * TW_TC * TW_LC * r;  // [C][TW_TC][r][TW_LC] cross-CTA reflectors
  return s;
}

// Whether the TSQR column basis applies to this launch (cluster-uniform).
__device__ __forceinline__ bool tsqr_usable(const CC& c, const ClusterJob& J) {
  // r <= 32: lane = column; the per-warp broadcast slots (2r complex of
  // wrow) must hold 2 x (TW_LC + 2) entries and the dense block's r + 1
  if (!c.ns_global || !J.Sg || !J.tsqr || c.r > 32 || 2 * c.r < 2 * (TW_LC + 2)) return false;
  const int ms = c.ldw, last = c.m - (c.C - 1) * ms;
  // every warp's rows start with a dense r x r block
  const int rpw0 = (ms + CW - 1) / CW, rpw1 = (last + CW - 1) / CW;
  if (last < 1 || ms - (CW - 1) * rpw0 < c.r || last - (CW - 1) * rpw1 < c.r) return false;
  return (long long)c.C * c.r * c.r + c.C * tw_tstride(ms, c.r, c.C) <= J.wg_stride;
}

__device__ __forceinline__ void tw_export(uint32_t ta, int r, cplx* dst) {  // triangle -> dst (column-major)
  const int lane = threadIdx.x & 31;
  for (int row = 0; row < r; ++row) {
    const cplx v = tm_ld(ta, row);
    if (lane < r) dst[(long long)lane * r + row] = row <= lane ? v : mk(0.0, 0.0);
  }
}
__device__ __forceinline__ void tw_import(uint32_t ta, int r, const cplx* src) {  // dst (column-major) -> TMEM
  const int lane = threadIdx.x & 31;
  for (int row = 0; row < r; ++row) {
    const cplx v = lane < r ? src[(long long)lane * r + row] : mk(0.0, 0.0);
    __syncwarp();
    tm_st(ta, row, v);
  }
}
// rows [c0, c0 + TW_LC) of a column-major r x r triangle as a chunk
__device__ __forceinline__ void tw_tri_chunk(const cplx* R, int r, int c0, cplx (&X)[TW_LC]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < TW_LC; ++i) X[i] = (lane < r && c0 + i < r) ? R[(long long)lane * r + c0 + i] : mk(0.0, 0.0);
}
// chunk reflectors X (lane = reflector index) -> V[j * TW_LC + i]
__device__ __forceinline__ void tw_store_v(const cplx (&X)[TW_LC], int r, cplx* V) {
  const int lane = threadIdx.x & 31;
  if (lane < r)
#pragma unroll
    for (int i = 0; i < TW_LC; ++i) V[(long long)lane * TW_LC + i] = X[i];
}

// Q rows (this lane's column) of TW_LC consecutive local rows l0.. (nrow
// valid) to global memory, with their squared norms for the fused starts.
__device__ __forceinline__ void tw_emit_q(CC& c, const cplx (&W)[TW_LC], int l0, int nrow, bool norms) {
  const int lane = threadIdx.x & 31;
  const int r = c.r, m = c.m;
  static_assert(TW_LC <= 16, "row norms reduce up to 16 rows at once");
  double d2[16], dm[16];
#pragma unroll
  for (int i = TW_LC; i < 16; ++i) d2[i] = dm[i] = 0.0;
#pragma unroll
  for (int i = 0; i < TW_LC; ++i) {
    const bool on = lane < r && i < nrow;
    if (on) c.Qg[(long long)lane * m + c.row0 + l0 + i] = W[i];
    d2[i] = on ? fma(W[i].x, W[i].x, W[i].y * W[i].y) : 0.0;
    dm[i] = on ? fmax(fabs(W[i].x), fabs(W[i].y)) : 0.0;
  }
  if (!norms) return;
  __syncwarp();  // the rows just written are readable by the whole warp
  double n2 = tw_tsum16(d2, [](double a, double b) { return a + b; });
  const double nmx = tw_tsum16(dm, [](double a, double b) { return fmax(a, b); });
  const int i = (lane >> 1) & 15;
  if ((lane & 1) == 0 && i < nrow) {
    const int l = l0 + i, g = c.row0 + l;
    if (!(nmx == 0.0 || (nmx > 1e-140 && nmx < 1e140))) n2 = ssq_norm2(ssq_of(Qrow(c, g), m, r));
    c.vn1[l] = n2;
    c.vn2[l] = n2;
    c.rpos[l] = g;
    c.rpos2[l] = g;
  }
}

// The column basis by TSQR + zlaqp2 on the triangle (see the file comment).
// Same contract as column_basis: Q (logical column order) in c.Qg, row norms
// and initial positions in vn1/vn2/rpos/rpos2 when norms_in_q; false
// (cluster-uniform) when the block is zero or rank deficient by rank_tol.
__device__ bool tsqr_basis(cg::cluster_group& cl, CC& c, const ClusterJob& J, int inst, double rank_tol,
                           bool norms_in_q) {
  const int r = c.r, C = c.C, crank = c.crank;
  const int nl = c.nrows, ms = c.ldw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rpw = (nl + CW - 1) / CW;
  const int rb = warp * rpw, re = min(nl, rb + rpw);  // this warp's local rows
  const int nch = tw_nch(re - rb, r);
  const int ntc = (r + TW_LC - 1) / TW_LC;  // chunks per triangle
  cplx* sbase = J.Sg + inst * J.wg_stride + (long long)C * r * r;
  const long long tstride = tw_tstride(ms, r, C);
  const TwScratch S = tw_scratch(sbase + crank * tstride, ms, r, C);
  const long long rr = (long long)r * r;
  cplx* taus_w = S.taus + (long long)warp * (1 + tw_nch((ms + CW - 1) / CW, r)) * r;
  cplx* vb = c.wrow + warp * 2 * r;
  int* flag = c.ibc + 8;
  uint32_t* holder = reinterpret_cast<uint32_t*>(c.ibc + 12);
  // ---- tensor memory: one 32-lane x 128-column region per warp
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(holder)),
                 "n"(TW_NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ta = tw_region(*holder);
  auto release_tmem = [&]() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*holder), "n"(TW_NCOLS));
  };
  SP_BEGIN(spq);
  // ---- 1. every warp: dense r x r block, then TW_LC-row chunks
  {
    const int r4 = (r + 3) & ~3;
    for (int b4 = 0; b4 < r4; b4 += 4) {
      cplx v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        v[i] = (lane < r && b4 + i < r) ? c.Ws[(long long)lane * ms + rb + b4 + i] : mk(0.0, 0.0);
      tm_st4(ta, b4, v);
    }
    tw_dense_fwd(ta, r, vb, c.Ws + rb, ms, taus_w);
    for (int ch = 0; ch < nch; ++ch) {
      const int row0 = rb + r + ch * TW_LC, nrow = min(TW_LC, re - row0);
      cplx X[TW_LC];
#pragma unroll
      for (int i = 0; i < TW_LC; ++i)
        X[i] = (lane < r && i < nrow) ? c.Ws[(long long)lane * ms + row0 + i] : mk(0.0, 0.0);
      if (ch + 1 < nch && lane < r) {  // next chunk of this column: 256 bytes
        const cplx* nx = c.Ws + (long long)lane * ms + row0 + TW_LC;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(nx));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(nx + 8));
      }
      tw_chunk_fwd(ta, X, r, vb, taus_w + (long long)(1 + ch) * r);
      if (lane < r)
#pragma unroll
        for (int i = 0; i < TW_LC; ++i)
          if (i < nrow) c.Ws[(long long)lane * ms + row0 + i] = X[i];
    }
    tw_export(ta, r, S.Rx + warp * rr);
  }
  SP(spq, 0);
  // ---- 2. binary tree over the warps: warp a absorbs warp a + s
  __syncthreads();
  for (int lvl = 0, s = 1; s < CW; s *= 2, ++lvl) {
    if (warp % (2 * s) == 0 && warp + s < CW) {
      const cplx* Rb = S.Rx + (warp + s) * rr;
      for (int k = 0; k < ntc; ++k) {
        cplx X[TW_LC];
        tw_tri_chunk(Rb, r, k * TW_LC, X);
        tw_chunk_fwd(ta, X, r, vb, S.ttree + ((long long)(warp * TW_LEVELS + lvl) * TW_TC + k) * r, k * TW_LC);
        tw_store_v(X, r, S.PV + ((long long)(warp * TW_LEVELS + lvl) * TW_TC + k) * TW_LC * r);
      }
      tw_export(ta, r, S.Rx + warp * rr);
    }
    __syncthreads();
  }
  SP(spq, 1);
  // ---- 3. across the cluster into CTA 0, zlaqp2 on the final triangle, and
  //         back down to every CTA's warp 0
  cl.sync();
  if (crank == 0) {
  if (warp == 0) {
    for (int p = 1; p < C; ++p) {
      const TwScratch Sp = tw_scratch(sbase + p * tstride, ms, r, C);
      for (int k = 0; k < ntc; ++k) {
        cplx X[TW_LC];
        tw_tri_chunk(Sp.Rx, r, k * TW_LC, X);
        tw_chunk_fwd(ta, X, r, vb, S.tx + ((long long)p * TW_TC + k) * r, k * TW_LC);
        tw_store_v(X, r, S.XV + ((long long)p * TW_TC + k) * TW_LC * r);
      }
    }
    tw_export(ta, r, c.aug);
  }
  __syncthreads();
  SP_BEGIN(spx);
  cplx* Rs = c.aug;
  cplx* Zs = c.aug + rr;
  ts_qrcp_block(c, Rs, Zs, rank_tol, flag);
  SP(spx, 5);
  if (warp == 0) {
    tw_import(ta, r, Zs);
    for (int p = C - 1; p >= 1; --p) {
      const TwScratch Sp = tw_scratch(sbase + p * tstride, ms, r, C);
      for (int k = ntc - 1; k >= 0; --k) {
        cplx W[TW_LC];
#pragma unroll
        for (int i = 0; i < TW_LC; ++i) W[i] = mk(0.0, 0.0);
        const int nrow = min(TW_LC, r - k * TW_LC);
        tw_chunk_rev(ta, W, r, S.XV + ((long long)p * TW_TC + k) * TW_LC * r, TW_LC, nrow, S.tx + ((long long)p * TW_TC + k) * r,
                     k * TW_LC);
        if (lane < r)
#pragma unroll
          for (int i = 0; i < TW_LC; ++i)
            if (i < nrow) Sp.Zx[(long long)lane * r + k * TW_LC + i] = W[i];
      }
    }
  }
  }
  cl.sync();
  SP(spq, 2);
  if (*cl.map_shared_rank(flag, 0)) {
    release_tmem();
    return false;
  }
  if (crank != 0 && warp == 0) tw_import(ta, r, S.Zx);
  // ---- 4. down the warp tree
  for (int lvl = TW_LEVELS - 1; lvl >= 0; --lvl) {
    const int s = 1 << lvl;
    if (s >= CW) continue;
    if (warp % (2 * s) == 0 && warp + s < CW) {
      cplx* Zb = S.Zx + (warp + s) * rr;
      for (int k = ntc - 1; k >= 0; --k) {
        cplx W[TW_LC];
#pragma unroll
        for (int i = 0; i < TW_LC; ++i) W[i] = mk(0.0, 0.0);
        const int nrow = min(TW_LC, r - k * TW_LC);
        const long long slot = (long long)(warp * TW_LEVELS + lvl) * TW_TC + k;
        tw_chunk_rev(ta, W, r, S.PV + slot * TW_LC * r, TW_LC, nrow, S.ttree + slot * r, k * TW_LC);
        if (lane < r)
#pragma unroll
          for (int i = 0; i < TW_LC; ++i)
            if (i < nrow) Zb[(long long)lane * r + k * TW_LC + i] = W[i];
      }
    }
    __syncthreads();
    if (warp % (2 * s) == s) tw_import(ta, r, S.Zx + warp * rr);
  }
  SP(spq, 3);
  // ---- 5. every warp's own rows, last chunk first, then the dense block
  for (int ch = nch - 1; ch >= 0; --ch) {
    const int row0 = rb + r + ch * TW_LC, nrow = min(TW_LC, re - row0);
    cplx W[TW_LC];
#pragma unroll
    for (int i = 0; i < TW_LC; ++i) W[i] = mk(0.0, 0.0);
    tw_chunk_rev(ta, W, r, c.Ws + row0, ms, nrow, taus_w + (long long)(1 + ch) * r);
    tw_emit_q(c, W, row0, nrow, norms_in_q);
  }
  tw_dense_rev(ta, r, vb, c.Ws + rb, ms, taus_w);
  for (int h0 = 0; h0 < r; h0 += TW_LC) {
    cplx W[TW_LC];
#pragma unroll
    for (int i = 0; i < TW_LC; ++i) W[i] = (h0 + i < r) ? tm_ld(ta, h0 + i) : mk(0.0, 0.0);
    tw_emit_q(c, W, rb + h0, min(TW_LC, r - h0), norms_in_q);
  }
  SP(spq, 4);
  release_tmem();
  __threadfence();
  __syncthreads();
  return true;
}
