"""Market inputs of the pricer (host side).

Only the quantities the device evaluators consume are derived here: the
log-price drift mu and the log-price covariance C of correlated GBM
(reference market.py:73-124, formulas at :114-121).  Validation follows the
reference's rules and messages so callers see the same errors.
"""

from __future__ import annotations

import numpy as np


def corr_matrix_plus(d, beta):
    """Correlation with beta/(1+beta) off the diagonal (reference market.py:32-45)."""
    if d < 1:
        raise ValueError("d must be >= 1")
    if not 0.0 <= beta <= 1.0:
        raise ValueError(f"beta must lie in [0, 1], got {beta}")
    out = np.eye(d)
    out[~np.eye(d, dtype=bool)] = beta / (1.0 + beta)
    return out


def _as_vector(value, d):
    return np.array(np.broadcast_to(np.asarray(value, dtype=float), (d,)))


def _infer_d(d, sigma, s0, rates, corr):
    if d is not None:
        return int(d)
    for candidate in (sigma, s0, rates):
        if candidate is not None and np.ndim(candidate) > 0:
            return len(candidate)
    return corr.shape[0] if corr is not None else 1


class MarketModel:
    """Correlated multi-asset GBM with a common strike.

    Same constructor as the reference (market.py:73): ``r, sigma, T, s0,
    strike, corr=None, rates=None, d=None``.  Arrays are frozen after
    construction.
    """

    def __init__(self, r, sigma, T, s0, strike, corr=None, rates=None, d=None):
        d = _infer_d(d, sigma, s0, rates, corr)
        self.d = d
        self.r = float(r)
        self.T = float(T)
        self.strike = float(strike)
        self.sigma = _as_vector(sigma, d)
        self.s0 = _as_vector(s0, d)
        self.rates = np.full(d, self.r) if rates is None else _as_vector(rates, d)
        corr = np.eye(d) if corr is None else np.asarray(corr, dtype=float)
        if corr.shape != (d, d):
            raise ValueError(f"corr must be {d}x{d}, got {corr.shape}")
        if not np.allclose(corr, corr.T, atol=1e-12):
            raise ValueError("corr must be symmetric")
        if np.max(np.abs(np.diag(corr) - 1.0)) > 1e-12:
            raise ValueError("corr must have a unit diagonal")
        try:
            self.chol = np.linalg.cholesky(corr)
        except np.linalg.LinAlgError as exc:
            raise ValueError("corr must be positive definite") from exc
        self.corr = corr
        if self.T <= 0:
            raise ValueError("T must be > 0")
        if self.strike <= 0:
            raise ValueError("strike must be > 0")
        if np.any(self.sigma <= 0):
            raise ValueError("sigma must be > 0")
        if np.any(self.s0 <= 0):
            raise ValueError("s0 must be > 0")
        # mu_j = ln S0_j + r_j T - sigma_j^2 Sigma_jj T / 2      (market.py:115-119)
        var_t = self.sigma ** 2 * np.diag(self.corr) * self.T
        self.log_drift = np.log(self.s0) + self.rates * self.T - 0.5 * var_t
        # C_jk = sigma_j sigma_k Sigma_jk T                      (market.py:121)
        self.log_cov = np.outer(self.sigma, self.sigma) * self.corr * self.T
        for arr in (self.sigma, self.s0, self.rates, self.corr, self.chol,
                    self.log_drift, self.log_cov):
            arr.flags.writeable = False

    @classmethod
    def with_plus_correlation(cls, d, beta, r=0.3, sigma=0.5, T=1.0, s0=100.0,
                              strike=100.0):
        return cls(r=r, sigma=sigma, T=T, s0=s0, strike=strike,
                   corr=corr_matrix_plus(d, beta), d=d)

    def __repr__(self):
        return (f"MarketModel(d={self.d}, r={self.r}, sigma={self.sigma.tolist()}, "
                f"T={self.T}, s0={self.s0.tolist()}, strike={self.strike})")


def black_scholes_price(model, t=0.0):
    """Closed-form European call for one asset (market.py:173-190):
    ``S0 Phi(d1) - K e^{-r(T-t)} Phi(d2)`` with scipy's ndtr."""
    from scipy.special import ndtr
    if model.d != 1:
        raise ValueError(f"closed form needs d=1, model has d={model.d}")
    if t >= model.T:
        raise ValueError(f"valuation time {t} must precede maturity {model.T}")
    s0, k, sig = model.s0[0], model.strike, model.sigma[0]
    tau = model.T - t
    vol = sig * np.sqrt(tau)
    d1 = (np.log(s0 / k) + (model.r + 0.5 * sig ** 2) * tau) / vol
    d2 = d1 - vol
    return float(s0 * ndtr(d1) - k * np.exp(-model.r * tau) * ndtr(d2))
