"""Seeded synthetic instances of the five BASELINE.json configurations.

The reference measures only on synthetic model parameters (paper section V);
these generators follow SURVEY.md 8(d): parameter draws use
``np.random.default_rng([config_id, instance_id])`` in the listed order, the
grid is ``GridSpec(n=N, eta=table1_hyperparams(d)[0], alpha=5/d)`` and the
cross seed is ``1234 + d`` (the reference's bench.py:342 convention).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .market import MarketModel, corr_matrix_plus
from .pricers import GridSpec, table1_hyperparams


def sampled_corr(rng, d):
    """Normalised covariance of 20 standard-normal draws per asset, made SPD."""
    x = rng.standard_normal((20, d))
    s = np.cov(x, rowvar=False)
    scale = 1.0 / np.sqrt(np.diag(s))
    c = s * np.outer(scale, scale)
    c = 0.5 * (c + c.T)
    np.fill_diagonal(c, 1.0)
    return c


def uniform_corr(d, rho):
    c = np.full((d, d), rho)
    np.fill_diagonal(c, 1.0)
    return c


def block_corr(n_blocks, block, intra, inter):
    d = n_blocks * block
    c = np.full((d, d), inter)
    for b in range(n_blocks):
        sl = slice(b * block, (b + 1) * block)
        c[sl, sl] = intra
    np.fill_diagonal(c, 1.0)
    return c


@dataclass(frozen=True)
class ConfigSpec:
    cid: int
    d: int
    n: int          # GridSpec.n (points per axis = n + 1)
    bond_dim: int
    n_instances: int
    label: str

    @property
    def grid(self):
        eta = table1_hyperparams(self.d)[0] if self.d >= 2 else 0.5
        return GridSpec(n=self.n, eta=eta, alpha=5.0 / self.d, d=self.d)

    @property
    def cross_seed(self):
        return 1234 + self.d


CONFIGS = {
    1: ConfigSpec(1, 3, 32, 10, 1, "d=3 call-on-min, N=32, D=10"),
    2: ConfigSpec(2, 5, 64, 20, 1, "d=5 call-on-min, N=64, D=20"),
    3: ConfigSpec(3, 5, 64, 20, 4096, "4096 x d=5 call-on-min, N=64, D=20"),
    4: ConfigSpec(4, 10, 128, 32, 1, "d=10 call-on-min, N=128, D=32"),
    5: ConfigSpec(5, 20, 256, 64, 1024, "1024 x d=20 call-on-min, N=256, D=64"),
}


def make_model(cid, instance=0):
    """MarketModel of instance ``instance`` of BASELINE config ``cid``."""
    rng = np.random.default_rng([cid, instance])
    if cid == 1:
        return MarketModel(r=0.05, sigma=0.2, T=1.0, s0=100.0, strike=100.0,
                           corr=corr_matrix_plus(3, 1.0), d=3)
    if cid == 2:
        sigma = rng.uniform(0.15, 0.35, size=5)
        corr = sampled_corr(rng, 5)
        return MarketModel(r=0.03, sigma=sigma, T=1.0, s0=100.0, strike=100.0, corr=corr)
    if cid == 3:
        strike = rng.uniform(80.0, 120.0)
        T = rng.uniform(0.25, 2.0)
        r = rng.uniform(0.0, 0.05)
        sigma = rng.uniform(0.15, 0.35, size=5)
        corr = sampled_corr(rng, 5)
        return MarketModel(r=r, sigma=sigma, T=T, s0=100.0, strike=strike, corr=corr)
    if cid == 4:
        sigma = rng.uniform(0.1, 0.4, size=10)
        return MarketModel(r=0.05, sigma=sigma, T=1.0, s0=100.0, strike=100.0,
                           corr=uniform_corr(10, 0.3))
    if cid == 5:
        s0 = rng.uniform(90.0, 110.0, size=20)
        strike = rng.uniform(90.0, 110.0)
        sigma = rng.uniform(0.1, 0.4, size=20)
        return MarketModel(r=0.04, sigma=sigma, T=1.0, s0=s0, strike=strike,
                           corr=block_corr(4, 5, 0.6, 0.2))
    raise ValueError(f"unknown config {cid}")


def model_kwargs(model):
    """Plain-dict constructor arguments (to rebuild the model in another package)."""
    return dict(r=model.r, sigma=np.array(model.sigma), T=model.T, s0=np.array(model.s0),
                strike=model.strike, corr=np.array(model.corr))
