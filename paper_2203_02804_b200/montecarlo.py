"""GPU Monte Carlo pricer for the min-option.

Drop-in for the reference's ``price_monte_carlo`` (pricers.py:297-350):
same signature, same validation, same estimator (mean of the discounted
payoff, sample standard error from the sum of squares, pricers.py:339-342)
and the same two schemes -- ``terminal_exact`` (exact lognormal terminal
law, pricers.py:324-326) and ``euler_path`` (``n_steps`` Euler increments,
pricers.py:327-333).

What differs by design: the normals.  The reference spawns one numpy PCG64
stream per chunk from ``SeedSequence(seed)``; here each path draws from a
counter-based Philox4x32-10 stream keyed by the seed and indexed by the
path number (csrc/k_mc.cu), so a path's shocks do not depend on chunking or
on the launch geometry.  ``chunk_size`` is accepted for signature
compatibility; like the reference's, results do not depend on it.  Parity
with the reference is statistical (same law, independent streams).
"""
import ctypes
import math
import time

import numpy as np

from . import _lib
from .pricers import PricingResult

SCHEMES = ("terminal_exact", "euler_path")


def _check(n_samples, scheme, n_steps, seed):
    if n_samples < 2:
        raise ValueError("n_samples must be >= 2")
    if scheme not in SCHEMES:
        raise ValueError(f"unknown scheme {scheme!r}")
    if scheme == "euler_path" and n_steps < 1:
        raise ValueError("n_steps must be >= 1")
    seed = int(seed)
    if seed < 0 or seed >= 1 << 64:
        raise ValueError("seed must be a non-negative 64-bit integer")
    return seed


def mc_params(model, scheme="terminal_exact", n_steps=64, t=0.0):
    """Packed per-instance parameters of ttp_mc_price (include/ttpricer_b200.h)."""
    d = model.d
    drift = (model.rates - 0.5 * model.sigma ** 2) * model.T      # pricers.py:319
    vol = model.sigma * np.sqrt(model.T)                            # pricers.py:320
    disc = np.exp(-model.r * (model.T - t))                         # pricers.py:313
    dt = model.T / n_steps if scheme == "euler_path" else 0.0       # pricers.py:328
    return np.concatenate([model.s0, drift, vol, model.rates, model.sigma,
                           np.asarray(model.chol, float).reshape(-1),
                           [model.strike, disc, dt]]).astype(np.float64)


def price_monte_carlo_batch(models, n_samples, seeds, scheme="terminal_exact", n_steps=64, t=0.0):
    """Monte Carlo estimates for several models of one dimension in one
    launch -> list of PricingResult (``seeds``: one per model)."""
    models = list(models)
    seeds = [_check(n_samples, scheme, n_steps, s) for s in seeds]
    if len(seeds) != len(models):
        raise ValueError("one seed per model")
    if not models:
        return []
    d = models[0].d
    if any(m.d != d for m in models):
        raise ValueError("all models of a batch must share d")
    torch = _lib.require_device()
    lib = _lib.load_library()
    start = time.perf_counter()
    prm = np.stack([mc_params(m, scheme, n_steps, t) for m in models])
    d_prm = torch.from_numpy(prm).to("cuda")
    n = len(models)
    ws_bytes = lib.ttp_mc_workspace(n, n_samples)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    h_seeds = (ctypes.c_uint64 * n)(*seeds)
    out = (ctypes.c_double * (2 * n))()
    st = lib.ttp_mc_price(ctypes.c_void_p(d_prm.data_ptr()), prm.shape[1], d, n, int(n_samples), h_seeds,
                          SCHEMES.index(scheme), int(n_steps), out, ctypes.c_void_p(ws.data_ptr()),
                          ws_bytes, _lib.stream_handle())
    _lib.raise_for(st, "monte carlo")
    wall = time.perf_counter() - start
    res = []
    for i in range(n):
        total, total_sq = out[2 * i], out[2 * i + 1]
        mean = total / n_samples                                        # pricers.py:339-341
        var = max(total_sq - n_samples * mean * mean, 0.0) / (n_samples - 1)
        res.append(PricingResult(mean, "monte_carlo", wall / n,
                                 {"n_samples": int(n_samples), "std_error": math.sqrt(var / n_samples),
                                  "scheme": scheme, "seed": seeds[i], "rng": "philox4x32-10"}))
    return res


def price_monte_carlo(model, n_samples, seed, scheme="terminal_exact", n_steps=64, t=0.0,
                      chunk_size=1_000_000):
    """Monte Carlo estimate of the discounted min-option payoff on the GPU
    (pricers.py:297-350).  ``chunk_size`` is accepted for compatibility;
    per-path counter-based streams make the result independent of it."""
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    return price_monte_carlo_batch([model], n_samples, [seed], scheme=scheme, n_steps=n_steps, t=t)[0]
