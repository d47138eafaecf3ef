"""CPU ORACLE -- test infrastructure only, never on the product path.

A numpy/scipy restatement of the reference's hot path (arXiv 2203.02804's
``ttpricer`` package, pure Python):

  evaluators      market.py:204-219 (phi), market.py:237-262 (vhat_min),
                  pricers.py:83-86 (contour), pricers.py:234-253 (grid oracles)
  contractions    tensor_train.py:126-140 (evaluate_many),
                  tensor_train.py:143-159 (inner), tensor_train.py:181-203 (sample diff)
  cross           cross.py:103-119 (column basis), :122-139 (swaps),
                  :147-169 (pairwise refine), :172-205 (dominant rows),
                  :296-307 (initial right sets), :310-332 (blocks),
                  :335-355 (interpolation factor), :358-453 (tt_cross)
  pricers         pricers.py:185-231 (dense sum), :256-294 (TT price)

It issues the same numpy/scipy calls in the same order as the reference, so
with one BLAS thread its outputs are bitwise equal to the reference's (that
is how it is pinned: tests/test_oracle_cpu.py checks it against the golden
fixtures generated from the reference itself, tests/golden/make_golden.py).
Index sets are kept as integer arrays instead of tuple lists; the sampled
index arrays, and hence every oracle call, are identical.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  The GPU package never does.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg

COND_LIMIT = 1e12
CHUNK = 1 << 20


class OracleError(RuntimeError):
    """Raised for the reference's numerical failure modes (kind in .kind)."""

    def __init__(self, kind, msg, bond=None):
        super().__init__(msg)
        self.kind = kind
        self.bond = bond


# ----------------------------------------------------------------- inputs
def model_arrays(sigma, corr, T, s0, rates):
    """(mu, C) of correlated GBM (market.py:114-121)."""
    sigma = np.asarray(sigma, float)
    corr = np.asarray(corr, float)
    mu = np.log(np.asarray(s0, float)) + np.asarray(rates, float) * T - 0.5 * sigma ** 2 * np.diag(corr) * T
    cov = np.outer(sigma, sigma) * corr * T
    return mu, cov


def contour(idx, n, eta, alpha):
    return eta * (np.asarray(idx, dtype=np.int64) - n // 2) + 1j * alpha


def phi_values(mu, cov, z):
    z = np.atleast_2d(np.asarray(z, dtype=np.complex128))
    lin = z @ mu
    quad = np.einsum("mj,jk,mk->m", z, cov, z)
    return np.exp(1j * lin - 0.5 * quad)


def vhat_min_values(z, strike):
    z = np.atleast_2d(np.asarray(z, dtype=np.complex128))
    d = z.shape[-1]
    w = z.sum(axis=-1)
    return ((-1.0) ** (d - 1) * np.exp((1.0 + 1j * w) * np.log(strike))
            / ((1.0 + 1j * w) * np.prod(1j * z, axis=-1)))


class GridModel:
    """Everything the two grid oracles need for one option."""

    def __init__(self, r, sigma, T, s0, strike, corr, n, eta, alpha, rates=None):
        d = np.asarray(corr).shape[0]
        self.d, self.r, self.T, self.strike = d, float(r), float(T), float(strike)
        sig = np.broadcast_to(np.asarray(sigma, float), (d,)).copy()
        s0v = np.broadcast_to(np.asarray(s0, float), (d,)).copy()
        rt = np.full(d, self.r) if rates is None else np.broadcast_to(np.asarray(rates, float), (d,)).copy()
        self.mu, self.cov = model_arrays(sig, corr, self.T, s0v, rt)
        self.n, self.eta, self.alpha = int(n), float(eta), float(alpha)

    @property
    def shape(self):
        return (self.n + 1,) * self.d

    def phi_oracle(self):
        return lambda idx: phi_values(self.mu, self.cov, -contour(idx, self.n, self.eta, self.alpha))

    def vhat_oracle(self):
        return lambda idx: np.conj(vhat_min_values(contour(idx, self.n, self.eta, self.alpha), self.strike))

    def prefactor(self, t=0.0):
        return np.exp(-self.r * (self.T - t)) * self.eta ** self.d / (2.0 * np.pi) ** self.d


# ------------------------------------------------------------ contractions
def tt_eval(cores, idx):
    idx = np.asarray(idx, dtype=np.int64)
    acc = cores[0][0, idx[:, 0], :]
    for k in range(1, len(cores)):
        acc = np.einsum("mi,imj->mj", acc, cores[k][:, idx[:, k], :])
    return acc[:, 0]


def tt_inner(bra, ket):
    env = np.ones((1, 1), dtype=np.complex128)
    for b, k in zip(bra, ket):
        env = np.tensordot(b.conj(), np.tensordot(env, k, axes=(1, 0)), axes=([0, 1], [0, 1]))
    return complex(env[0, 0])


def draw_samples(phys, m, seed):
    gen = np.random.default_rng(seed)
    out = np.empty((m, len(phys)), dtype=np.int64)
    for k, n in enumerate(phys):
        out[:, k] = gen.integers(0, n, size=m)
    return out


def sample_diff(cores, oracle, m, seed):
    phys = tuple(c.shape[1] for c in cores)
    idx = draw_samples(phys, m, seed)
    approx = tt_eval(cores, idx)
    exact = np.asarray(oracle(idx), dtype=np.complex128)
    num = float(np.sum(np.abs(exact - approx)))
    den = float(np.sum(np.abs(exact)))
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / den


# ------------------------------------------------------------------ maxvol
def column_basis(mat, rank_tol):
    q, r, _ = scipy.linalg.qr(mat, mode="economic", pivoting=True)
    dg = np.abs(np.diag(r))
    top = dg.max(initial=0.0)
    if top == 0.0 or dg.min() < rank_tol * top:
        raise OracleError("singular", f"block {mat.shape} is rank deficient")
    return q


def swaps(q, start, slack, max_iters):
    rows = np.asarray(start, dtype=np.int64).copy()
    b = np.linalg.solve(q[rows].T, q.T).T
    budget = max_iters if max_iters is not None else 10 * q.shape[0]
    for it in range(budget):
        i, j = np.unravel_index(np.argmax(np.abs(b)), b.shape)
        piv = b[i, j]
        if abs(piv) <= 1.0 + slack:
            return np.sort(rows)
        b += np.outer(b[:, j], b[rows[j], :] - b[i, :]) / piv
        rows[j] = i
        if (it + 1) % 64 == 0:
            b = np.linalg.solve(q[rows].T, q.T).T
    raise OracleError("maxvol_iter", f"no dominance within {budget} swaps")


def pair_refine(q, rows, slack, max_iters):
    budget = max_iters if max_iters is not None else 10 * q.shape[0]
    for _ in range(budget):
        rows = swaps(q, rows, slack, max_iters)
        b = np.linalg.solve(q[rows].T, q.T).T
        minors = np.abs(np.einsum("ij,kl->ikjl", b, b) - np.einsum("il,kj->ikjl", b, b))
        i1, i2, j1, j2 = np.unravel_index(np.argmax(minors), minors.shape)
        if minors[i1, i2, j1, j2] <= 1.0 + 1e-9:
            return rows
        rows = rows.copy()
        rows[j1], rows[j2] = i1, i2
    raise OracleError("maxvol_iter", "pairwise refinement did not settle")


def dominant_rows(q, slack, max_iters):
    n, r = q.shape
    if n == r:
        return np.arange(r, dtype=np.int64)
    piv = scipy.linalg.qr(q.conj().T, mode="economic", pivoting=True)[2]
    candidates = [np.sort(piv[:r].astype(np.int64))]
    perm = scipy.linalg.lu(q, p_indices=True)[0]
    lu_rows = np.sort(np.argsort(perm)[:r].astype(np.int64))
    if not np.array_equal(lu_rows, candidates[0]):
        candidates.append(lu_rows)
    best, best_vol, last_err = None, -math.inf, None
    for cand in candidates:
        try:
            rows = swaps(q, cand, slack, max_iters)
        except OracleError as exc:
            last_err = exc
            continue
        vol = np.linalg.slogdet(q[rows])[1]
        if vol > best_vol:
            best, best_vol = rows, vol
    if best is None:
        raise last_err
    if n <= 96 and r <= 8:
        best = pair_refine(q, best, slack, max_iters)
    return best


def maxvol(mat, slack=0.01, max_iters=None, rank_tol=1e-12):
    mat = np.asarray(mat, dtype=np.complex128)
    return dominant_rows(column_basis(mat, rank_tol), slack, max_iters)


# ------------------------------------------------------------------- cross
def rank_profile(shape, bond):
    d = len(shape)
    return [min(bond, math.prod(shape[:k]), math.prod(shape[k:])) for k in range(d + 1)]


def initial_right(shape, ranks, seed):
    d = len(shape)
    gen = np.random.default_rng(seed)
    right = [None] * (d + 1)
    right[d] = np.zeros((1, 0), dtype=np.int64)
    for k in range(d - 1, 0, -1):
        tail = right[k + 1]
        total = shape[k] * len(tail)
        chosen = np.sort(gen.choice(total, size=min(ranks[k], total), replace=False))
        s, b = np.divmod(chosen, len(tail))
        right[k] = np.column_stack([s, tail[b]]).astype(np.int64)
    return right


def sample_block(oracle, left, n_axis, right, axis_first):
    """Unfolding block; rows/cols as integer tuple arrays (cross.py:310-332)."""
    if axis_first:
        rows = left
        cols = np.column_stack([np.repeat(np.arange(n_axis), len(right)), np.tile(right, (n_axis, 1))])
    else:
        rows = np.column_stack([np.repeat(left, n_axis, axis=0), np.tile(np.arange(n_axis), len(left))])
        cols = right
    idx = np.concatenate([np.repeat(rows, len(cols), axis=0), np.tile(cols, (len(rows), 1))], axis=1)
    vals = np.asarray(oracle(idx.astype(np.int64)), dtype=np.complex128)
    return vals.reshape(len(rows), len(cols)), rows, cols


def interp_factor(block, slack, bond):
    try:
        q = column_basis(block, 0.0)
        rows = dominant_rows(q, slack, None)
    except OracleError as exc:
        raise OracleError(exc.kind, f"bond {bond}: {exc}", bond=bond) from exc
    sub = q[rows]
    if np.linalg.cond(sub) > COND_LIMIT:
        raise OracleError("singular", f"pivot block at bond {bond} is ill conditioned", bond=bond)
    return rows, np.linalg.solve(sub.T, q.T).T


def tt_cross(oracle, shape, bond_dim, eps_tol=0.005, max_sweeps=4, n_conv=50_000, seed=0,
             slack=0.01, budget=None):
    """Returns (cores, report dict).  report has the CrossReport fields plus
    'left'/'right' index-set arrays."""
    shape = tuple(int(n) for n in shape)
    d = len(shape)
    used = {"construction": 0, "convergence": 0}

    def call(idx, kind="construction"):
        total = used["construction"] + used["convergence"] + len(idx)
        if budget is not None and total > budget:
            raise OracleError("budget", f"oracle budget {budget} exceeded")
        used[kind] += len(idx)
        return np.asarray(oracle(idx), dtype=np.complex128)

    def conv_check(cores):
        return sample_diff(cores, lambda ix: call(ix, "convergence"), n_conv, seed)

    if d == 1:
        vec = call(np.arange(shape[0], dtype=np.int64)[:, None])
        cores = [vec.reshape(1, shape[0], 1)]
        diff = conv_check(cores)
        return cores, dict(converged=diff <= eps_tol, sweeps_used=1,
                           oracle_calls=used["construction"], conv_check_calls=used["convergence"],
                           final_diff=diff, compression_ratio=used["construction"] / shape[0],
                           left=[np.zeros((1, 0), np.int64), None], right=[None, np.zeros((1, 0), np.int64)])
    ranks = rank_profile(shape, bond_dim)
    right = initial_right(shape, ranks, seed)
    left = [None] * (d + 1)
    left[0] = np.zeros((1, 0), dtype=np.int64)
    cores = [None] * d
    diff, sweeps, converged = math.inf, 0, False
    while sweeps < max_sweeps and not converged:
        if sweeps % 2 == 0:
            for k in range(1, d):
                blk, rows, _ = sample_block(call, left[k - 1], shape[k - 1], right[k], False)
                sel, fac = interp_factor(blk, slack, k)
                left[k] = rows[sel]
                cores[k - 1] = fac.reshape(len(left[k - 1]), shape[k - 1], len(right[k]))
            blk, _, _ = sample_block(call, left[d - 1], shape[d - 1], right[d], False)
            cores[d - 1] = blk.reshape(len(left[d - 1]), shape[d - 1], 1)
        else:
            for k in range(d - 1, 0, -1):
                blk, _, cols = sample_block(call, left[k], shape[k], right[k + 1], True)
                sel, fac = interp_factor(blk.T, slack, k)
                right[k] = cols[sel]
                cores[k] = fac.T.reshape(len(left[k]), shape[k], len(right[k + 1]))
            blk, _, _ = sample_block(call, left[0], shape[0], right[1], True)
            cores[0] = blk.reshape(1, shape[0], len(right[1]))
        sweeps += 1
        diff = conv_check(cores)
        converged = diff <= eps_tol
    return cores, dict(converged=converged, sweeps_used=sweeps, oracle_calls=used["construction"],
                       conv_check_calls=used["convergence"], final_diff=diff,
                       compression_ratio=used["construction"] / math.prod(shape),
                       left=left, right=right)


# ----------------------------------------------------------------- pricers
def dense_sum(gm):
    shape = gm.shape
    total = math.prod(shape)
    acc = 0.0 + 0.0j
    phi, vh = gm.phi_oracle(), None
    for lo in range(0, total, CHUNK):
        flat = np.arange(lo, min(lo + CHUNK, total), dtype=np.int64)
        idx = np.stack(np.unravel_index(flat, shape), axis=1)
        z = contour(idx, gm.n, gm.eta, gm.alpha)
        acc += np.sum(phi_values(gm.mu, gm.cov, -z) * vhat_min_values(z, gm.strike))
    del phi, vh
    return acc


def price_dense(gm, t=0.0):
    return float((gm.prefactor(t) * dense_sum(gm)).real)


def price_tt(gm, bond_phi, bond_v, seed_phi, seed_v, t=0.0, **cross_kw):
    phi_cores, rep_phi = tt_cross(gm.phi_oracle(), gm.shape, bond_phi, seed=seed_phi, **cross_kw)
    v_cores, rep_v = tt_cross(gm.vhat_oracle(), gm.shape, bond_v, seed=seed_v, **cross_kw)
    raw = tt_inner(v_cores, phi_cores)
    value = gm.prefactor(t) * raw
    return float(value.real), {"raw": raw, "cross_phi": rep_phi, "cross_v": rep_v,
                               "phi_cores": phi_cores, "v_cores": v_cores}
