"""Golden fixture generator (test infrastructure): the reference's own
reproducibility band per (config, instance) -> tests/golden/noise_bands.json.

The pinned CPU restatement (oracle/ttp_oracle.py, bitwise equal to the
reference's outputs with one BLAS thread) is rerun with every oracle value
perturbed by independent relative noise of 1e-15 (SURVEY.md 8(c)'s noise-floor
probe, several noise seeds per instance).  The spread of the perturbed prices
around the unperturbed one is how far the reference's own TT price moves under
rounding-level changes of its inputs -- the yardstick for an independent
implementation's end-to-end price.

Usage: OPENBLAS_NUM_THREADS=1 python tests/golden/make_noise_band.py CID N_INST N_SEEDS [FIRST]
(instances FIRST .. N_INST-1, default FIRST = 0; merges into noise_bands.json).
"""
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import ttp_oracle as O  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

OUT = os.path.join(HERE, "noise_bands.json")


def run(job):
    cid, inst, noise_seed = job
    m = configs.make_model(cid, inst)
    spec = configs.CONFIGS[cid]
    g = spec.grid
    gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, g.n, g.eta, g.alpha)
    if noise_seed >= 0:
        rng = np.random.default_rng([noise_seed, cid, inst])
        phi0, v0 = gm.phi_oracle(), gm.vhat_oracle()

        def noisy(f):
            def g_(idx):
                v = f(idx)
                return v * (1 + 1e-15 * (rng.standard_normal(v.shape) + 1j * rng.standard_normal(v.shape)))
            return g_
        gm.phi_oracle = lambda: noisy(phi0)
        gm.vhat_oracle = lambda: noisy(v0)
    price, info = O.price_tt(gm, spec.bond_dim, spec.bond_dim, spec.cross_seed, spec.cross_seed)
    return job, (price, {k: {"sweeps_used": int(info[k]["sweeps_used"]), "final_diff": float(info[k]["final_diff"])}
                         for k in ("cross_phi", "cross_v")})


if __name__ == "__main__":
    cid, n_inst, n_seeds = (int(a) for a in sys.argv[1:4])
    first = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    jobs = [(cid, i, s) for i in range(first, n_inst) for s in [-1] + list(range(n_seeds))]
    with ProcessPoolExecutor(max_workers=int(os.environ.get('BAND_WORKERS', os.cpu_count()))) as ex:
        res = dict(ex.map(run, jobs))
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for i in range(first, n_inst):
        base = res[(cid, i, -1)][0]
        rel = sorted(abs(res[(cid, i, s)][0] - base) / abs(base) for s in range(n_seeds))
        data[f"cfg{cid}_i{i}"] = {"unperturbed": base, "rel_dev_sorted": rel, "max": max(rel),
                                  "median": float(np.median(rel)), "n_seeds": n_seeds,
                                  "reports": [res[(cid, i, s)][1] for s in [-1] + list(range(n_seeds))]}
        print(f"cfg{cid} i{i}: price {base!r} noise max {max(rel):.2e} median {np.median(rel):.2e}")
    data["generator"] = ("tests/golden/make_noise_band.py CID N_INST N_SEEDS (OPENBLAS_NUM_THREADS=1): "
                         "the pinned restatement with 1e-15 relative oracle noise")
    with open(OUT, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
