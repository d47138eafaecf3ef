"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the device Monte Carlo
sampler (csrc/k_mc.cu) for the GPU tests; never imported by the product.

Philox4x32-10 follows the published algorithm (Salmon, Moraes, Dror, Shaw,
"Parallel random numbers: as easy as 1, 2, 3", SC'11; Random123): 10 rounds
of the (0xD2511F53, 0xCD9E8D57) multiply-xorshift with the key bumped by the
Weyl constants (0x9E3779B9, 0xBB67AE85).  It is pinned by the Random123
known-answer vectors in tests/test_mc_cpu.py.  The path estimator mirrors
the reference's price_monte_carlo (pricers.py:297-350) with these normals.
"""
import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
TAG = 0x4D43
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint32 arrays; returns four uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32).copy() for x in (c0, c1, c2, c3))
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for _ in range(10):
        p0 = M0 * c0.astype(np.uint64)
        p1 = M1 * c2.astype(np.uint64)
        hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & MASK).astype(np.uint32)
        hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & MASK).astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint32(k0), lo1, hi0 ^ c3 ^ np.uint32(k1), lo0
        k0 = (k0 + 0x9E3779B9) & 0xFFFFFFFF
        k1 = (k1 + 0xBB67AE85) & 0xFFFFFFFF
    return c0, c1, c2, c3


def _u53(lo, hi):
    v = (hi.astype(np.uint64) << np.uint64(32)) | lo.astype(np.uint64)
    return ((v >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53


def normals(paths, step, d, seed):
    """(len(paths), d) normals of draw step `step` for the given path indices."""
    paths = np.asarray(paths, dtype=np.uint64)
    k0, k1 = seed & 0xFFFFFFFF, seed >> 32
    np_ = (d + 1) // 2
    out = np.empty((len(paths), 2 * np_))
    lo = (paths & MASK).astype(np.uint32)
    hi = (paths >> np.uint64(32)).astype(np.uint32)
    for p in range(np_):
        g = np.full(len(paths), step * np_ + p, dtype=np.uint32)
        o0, o1, o2, o3 = philox4x32_10(lo, hi, g, np.full(len(paths), TAG, np.uint32), k0, k1)
        u1, u2 = _u53(o0, o1), _u53(o2, o3)
        rad = np.sqrt(-2.0 * np.log(u1))
        out[:, 2 * p] = rad * np.cos(2.0 * np.pi * u2)
        out[:, 2 * p + 1] = rad * np.sin(2.0 * np.pi * u2)
    return out[:, :d]


def mc_sums(model, n_samples, seed, scheme="terminal_exact", n_steps=64, t=0.0):
    """(sum, sum of squares) of the discounted payoff over paths 0..n-1."""
    paths = np.arange(n_samples, dtype=np.uint64)
    disc = np.exp(-model.r * (model.T - t))
    if scheme == "terminal_exact":
        drift = (model.rates - 0.5 * model.sigma ** 2) * model.T
        vol = model.sigma * np.sqrt(model.T)
        shocks = normals(paths, 0, model.d, seed) @ model.chol.T
        s_t = model.s0 * np.exp(drift + vol * shocks)
    else:
        dt = model.T / n_steps
        s_t = np.broadcast_to(model.s0, (n_samples, model.d)).copy()
        for t_ in range(n_steps):
            dw = normals(paths, t_, model.d, seed) @ model.chol.T * np.sqrt(dt)
            s_t *= 1.0 + model.rates * dt + model.sigma * dw
        s_t = np.maximum(s_t, 0.0)
    pay = disc * np.maximum(s_t.min(axis=1) - model.strike, 0.0)
    return float(pay.sum()), float((pay * pay).sum())
