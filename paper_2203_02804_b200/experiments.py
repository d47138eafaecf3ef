"""Batched experiment runners on the device path.

Row-for-row equivalents of the reference's ``run_table1``
(bench.py:318-363), ``run_bond_dim_sweep`` (bench.py:366-423) and
``run_strike_sweep`` (bench.py:478-510): same configuration fields and
defaults (ExperimentConfig, bench.py:74-240), same row keys.  CSV/manifest
emission and the CLI stay out of scope; the rows are returned.

The device path batches where the experiment is batchable:
  * bond sweep: the payoff train of each seed is built once (as the
    reference's v cache), the dense prices of all betas in one launch, and
    for each (seed, D_phi) the phi crosses of all betas in one batch;
  * strike sweep: price_strike_ladder (one phi train for the ladder),
    Monte Carlo and dense prices of all strikes in one launch each.
"""
import math
from dataclasses import dataclass, replace

import numpy as np

from .cross import CrossConfig, tt_cross, tt_cross_batch
from .errors import NumericsError
from .market import MarketModel, black_scholes_price
from .montecarlo import price_monte_carlo, price_monte_carlo_batch
from .oracles import OracleBatch, PhiGridOracle
from .pricers import (GridSpec, PricingResult, payoff_grid_oracle, price_fourier_dense,
                      price_fourier_dense_batch, price_fourier_tt, price_strike_ladder,
                      table1_hyperparams)
from .tensor_train import tt_inner

_EPS_FLOOR = 1e-16  # bench.py:70


@dataclass
class ExperimentConfig:
    """The experiment fields of the reference's ExperimentConfig (bench.py:74-110)."""
    r: float = 0.3
    sigma: float = 0.5
    T: float = 1.0
    s0: float = 100.0
    strike: float = 100.0
    beta: float = 0.5
    d: int = 1
    d_list: tuple = (2, 3, 4, 5, 6, 7, 8, 9, 10, 15)
    n_grid: int = 50
    eta: float = None
    alpha: float = None
    bond_v: int = None
    bond_phi: int = None
    eps_tol: float = 0.005
    max_sweeps: int = 4
    n_conv_samples: int = 50_000
    seed: int = 1234
    n_repeats: int = 20
    bond_phi_list: tuple = (2, 4, 6, 8, 10, 12)
    beta_list: tuple = (0.2, 0.5, 1.0)
    mc_samples: int = 50_000_000
    mc_seed: int = 99
    method: str = "bs_exact"

    def model_for(self, d, beta=None):  # bench.py:217-221
        return MarketModel.with_plus_correlation(
            d=d, beta=self.beta if beta is None else beta,
            r=self.r, sigma=self.sigma, T=self.T, s0=self.s0, strike=self.strike)

    def grid_for(self, d):  # bench.py:223-230
        if d == 1:
            eta = 0.5 if self.eta is None else self.eta
            alpha = 3.0 if self.alpha is None else self.alpha
        else:
            eta = table1_hyperparams(d)[0] if self.eta is None else self.eta
            alpha = 5.0 / d if self.alpha is None else self.alpha
        return GridSpec(n=self.n_grid, eta=eta, alpha=alpha, d=d)

    def bonds_for(self, d):  # bench.py:232-240
        if d == 1:
            table_v = table_phi = 1
        else:
            _, table_v, table_phi = table1_hyperparams(d)
        return (table_v if self.bond_v is None else self.bond_v,
                table_phi if self.bond_phi is None else self.bond_phi)

    def cross(self, bond_dim, seed):
        return CrossConfig(bond_dim=bond_dim, eps_tol=self.eps_tol, max_sweeps=self.max_sweeps,
                           n_conv_samples=self.n_conv_samples, seed=seed)


def run_table1(cfg):
    """Rows of bench.py:318-363 (t_rel against the device Monte Carlo time at
    d=2, extrapolated linearly in d, as the reference does with its own)."""
    t_mc2 = None
    if cfg.mc_samples > 0:
        t_mc2 = price_monte_carlo(cfg.model_for(2), cfg.mc_samples, cfg.mc_seed).wall_time_s
    rows = []
    for d in [int(x) for x in cfg.d_list]:
        bond_v, bond_phi = cfg.bonds_for(d)
        grid = cfg.grid_for(d)
        row = {"d": d, "D_v": bond_v, "D_phi": bond_phi, "eta": grid.eta, "t_wall": None,
               "t_rel": None, "r_comp": None, "eps_trunc": None, "price": None,
               "converged": None, "error": ""}
        try:
            res = price_fourier_tt(cfg.model_for(d), grid, cfg_phi=cfg.cross(bond_phi, cfg.seed + d),
                                   cfg_v=cfg.cross(bond_v, cfg.seed + d))
        except NumericsError as exc:
            row["error"] = str(exc)
            rows.append(row)
            continue
        diag = res.diagnostics
        row["price"] = res.price
        row["t_wall"] = res.wall_time_s
        row["r_comp"] = diag["oracle_calls_total"] / grid.n_terms
        row["eps_trunc"] = diag.get("eps_trunc")
        row["converged"] = diag["cross_phi"].converged and diag["cross_v"].converged
        if t_mc2 is not None:
            row["t_rel"] = res.wall_time_s / (t_mc2 * d / 2.0)
        rows.append(row)
    return rows


def run_bond_dim_sweep(cfg):
    """Rows of bench.py:366-423: mean log10 truncation error vs D_phi per beta."""
    d = cfg.d if cfg.d > 1 else 3
    grid = cfg.grid_for(d)
    bond_v = 30 if cfg.bond_v is None else cfg.bond_v
    shape = (grid.points_per_axis,) * d
    seeds = [cfg.seed + i for i in range(cfg.n_repeats)]
    prefactor = grid.eta ** d / (2.0 * np.pi) ** d
    v_model = cfg.model_for(d, beta=0.0)
    v_cache = {s: tt_cross(payoff_grid_oracle(v_model, grid), shape, cfg.cross(bond_v, s))[0]
               for s in seeds}
    betas = list(cfg.beta_list)
    models = [cfg.model_for(d, beta=b) for b in betas]
    dense = [r.price for r in price_fourier_dense_batch(models, grid)]
    logs = {(b, int(bp)): [] for b in range(len(betas)) for bp in cfg.bond_phi_list}
    conv = {k: 0 for k in logs}
    for bp in [int(x) for x in cfg.bond_phi_list]:
        for s in seeds:
            res = tt_cross_batch(OracleBatch([PhiGridOracle(m, grid) for m in models]), shape,
                                 cfg.cross(bp, s))
            trains = res.trains.to_trains()
            for b, m in enumerate(models):
                err = res.error_for(b)
                if err is not None:
                    raise err
                disc = np.exp(-m.r * m.T)
                price = disc * prefactor * tt_inner(v_cache[s], trains[b]).real
                eps = abs(price - dense[b]) / abs(dense[b])
                logs[(b, bp)].append(math.log10(max(eps, _EPS_FLOOR)))
                conv[(b, bp)] += res.reports[b].converged
    rows = []
    for b, beta in enumerate(betas):
        for bp in [int(x) for x in cfg.bond_phi_list]:
            rows.append({"beta": beta, "D_phi": bp,
                         "mean_log_eps_trunc": float(np.mean(logs[(b, bp)])),
                         "n_repeats": cfg.n_repeats,
                         "converged_fraction": conv[(b, bp)] / cfg.n_repeats})
    return rows


def _err_estimate(result):  # bench.py:449-461
    diag = result.diagnostics
    if result.method == "bs_exact":
        return 0.0
    if result.method == "fourier_dense":
        return diag["imag_residue"]
    if result.method == "fourier_tt":
        if "eps_trunc" in diag:
            return diag["eps_trunc"]
        return max(diag["cross_phi"].final_diff, diag["cross_v"].final_diff)
    if result.method == "monte_carlo":
        return diag["std_error"]
    return None


def _evaluation_count(result):  # bench.py:464-475
    diag = result.diagnostics
    return {"bs_exact": 0, "fourier_dense": diag.get("n_terms"),
            "fourier_tt": diag.get("oracle_calls_total"),
            "monte_carlo": diag.get("n_samples")}[result.method]


def run_strike_sweep(cfg, strikes, methods=None):
    """Rows of bench.py:478-510 for the device methods (bs_exact, fourier_dense,
    fourier_tt, monte_carlo); the d=1 direct-grid validator is out of scope."""
    methods = [cfg.method] if methods is None else list(methods)
    strikes = [float(k) for k in strikes]
    rows = []
    for method in methods:
        subs = [replace(cfg, method=method, strike=k) for k in strikes]
        d = cfg.d
        models = [s.model_for(d) if d > 1 else
                  MarketModel(r=s.r, sigma=s.sigma, T=s.T, s0=s.s0, strike=s.strike, d=1) for s in subs]
        if method == "bs_exact":
            results = [PricingResult(black_scholes_price(m), "bs_exact", 0.0, {}) for m in models]
        elif method == "fourier_dense":
            results = price_fourier_dense_batch(models, cfg.grid_for(d))
        elif method == "fourier_tt":
            bond_v, bond_phi = cfg.bonds_for(d)
            # price_fourier_tt's default dense_reference="auto" (pricers.py:256-294)
            results = price_strike_ladder(models[0], cfg.grid_for(d), strikes,
                                          cfg.cross(bond_phi, cfg.seed), cfg.cross(bond_v, cfg.seed),
                                          dense_reference="auto")
        elif method == "monte_carlo":
            results = price_monte_carlo_batch(models, cfg.mc_samples, [cfg.mc_seed] * len(models))
        else:
            raise ValueError(f"method: unknown or out-of-scope pricing method {method!r}")
        for s, res in zip(subs, results):
            rows.append({"method": method, "d": s.d, "beta": s.beta, "K": s.strike, "price": res.price,
                         "err_estimate": _err_estimate(res), "wall_time_s": res.wall_time_s,
                         "oracle_calls": _evaluation_count(res)})
    return rows
