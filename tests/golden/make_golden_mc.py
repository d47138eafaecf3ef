"""Reference Monte Carlo / closed-form / dense values for the GPU Monte Carlo
tests (statistical parity).  Runs the UNMODIFIED reference
from /root/reference (read-only) in this container; writes mc_ref.json.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_mc.py
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from ttpricer import (GridSpec, MarketModel, black_scholes_price, price_fourier_dense,  # noqa: E402
                      price_monte_carlo, table1_hyperparams)

BENCH = dict(r=0.3, sigma=0.5, T=1.0, s0=100.0, strike=100.0)


def single():
    return MarketModel(d=1, **BENCH)


def plus(d, beta=0.5):
    return MarketModel.with_plus_correlation(d=d, beta=beta, **BENCH)


def grid(d, n=50):
    if d == 1:
        return GridSpec(n=n, eta=0.5, alpha=3.0, d=1)
    return GridSpec(n=n, eta=table1_hyperparams(d)[0], alpha=5.0 / d, d=d)


def mc(model, n, seed, **kw):
    r = price_monte_carlo(model, n, seed=seed, **kw)
    return {"price": r.price, "std_error": r.diagnostics["std_error"], "n": n, "seed": seed, **kw}


out = {
    "black_scholes_d1": black_scholes_price(single()),
    "mc_d1_1e6_seed2024": mc(single(), 1_000_000, 2024),
    "mc_d1_euler_2e5_seed3": mc(single(), 200_000, 3, scheme="euler_path", n_steps=128),
    "mc_d2_plus05_2e6_seed42": mc(plus(2), 2_000_000, 42),
    "dense_d2_plus05_n50": price_fourier_dense(plus(2), grid(2)).price,
    "dense_d3_plus05_n50": price_fourier_dense(plus(3), grid(3)).price,
    "mc_d5_plus05_1e6_seed777": mc(plus(5), 1_000_000, 777),
    "mc_d6_plus05_1e6_seed777": mc(plus(6), 1_000_000, 777),
}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mc_ref.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
