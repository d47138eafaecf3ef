"""Golden fixture generator (test infrastructure): the reference's own
reproducibility band on cfg4 instance 0 -> tests/golden/cfg4_noise_band.json.

The pinned CPU restatement (which reproduces the reference's outputs bit
for bit) is rerun with each oracle value perturbed by independent relative
noise of 1e-15 (SURVEY.md 8(c)'s noise-floor probe, here with several noise
seeds), and the spread of the resulting prices around the unperturbed one
is reported.  Runs on the host; OPENBLAS_NUM_THREADS=1 recommended.
"""
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from oracle import ttp_oracle as O  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

CID = 4


def run(noise_seed):
    m = configs.make_model(CID, 0)
    spec = configs.CONFIGS[CID]
    g = spec.grid
    gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, g.n, g.eta, g.alpha)
    if noise_seed >= 0:
        rng = np.random.default_rng(noise_seed)
        phi0, v0 = gm.phi_oracle(), gm.vhat_oracle()

        def noisy(f):
            def g_(idx):
                v = f(idx)
                return v * (1 + 1e-15 * (rng.standard_normal(v.shape) + 1j * rng.standard_normal(v.shape)))
            return g_
        gm.phi_oracle = lambda: noisy(phi0)
        gm.vhat_oracle = lambda: noisy(v0)
    price, _ = O.price_tt(gm, spec.bond_dim, spec.bond_dim, spec.cross_seed, spec.cross_seed)
    return noise_seed, price


if __name__ == "__main__":
    seeds = [-1] + list(range(int(sys.argv[1]) if len(sys.argv) > 1 else 12))
    with ProcessPoolExecutor(max_workers=min(len(seeds), 16)) as ex:
        out = dict(ex.map(run, seeds))
    base = out.pop(-1)
    rel = sorted(abs(p - base) / abs(base) for p in out.values())
    print(json.dumps({"config": CID, "instance": 0, "unperturbed": base, "perturbed": out,
                      "rel_dev_sorted": rel, "max": max(rel), "median": float(np.median(rel))}, indent=1))
