"""Reference rows of the batched experiment runners
on small configurations.  Runs the UNMODIFIED reference from /root/reference
(read-only) in this container; writes experiments_ref.json.

    python tests/golden/make_golden_experiments.py
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from ttpricer.bench import ExperimentConfig, run_bond_dim_sweep, run_strike_sweep, run_table1  # noqa: E402

SWEEP = dict(experiment="bond_dim_sweep", model={"d": 2},
             grid={"N": 20}, cross={"D_v": 8, "n_repeats": 3, "D_phi_list": [2, 3, 5],
                                    "beta_list": [0.2, 0.8], "n_conv_samples": 4000, "seed": 11})
TABLE = dict(experiment="table1", model={"d_list": [2, 3]}, grid={"N": 20},
             cross={"n_conv_samples": 4000}, mc={"n_samples": 0})
STRIKE = dict(experiment="price_once", model={"d": 2}, grid={"N": 20},
              cross={"D_v": 6, "D_phi": 6, "n_conv_samples": 4000}, mc={"n_samples": 200_000, "seed": 5})
STRIKES = [90.0, 100.0, 115.0]


def clean(rows):
    return [{k: v for k, v in r.items() if k not in ("t_wall", "t_rel", "wall_time_s")} for r in rows]


out = {
    "sweep_cfg": SWEEP, "sweep": clean(run_bond_dim_sweep(ExperimentConfig.from_dict(SWEEP))),
    "table_cfg": TABLE, "table": clean(run_table1(ExperimentConfig.from_dict(TABLE))),
    "strike_cfg": STRIKE, "strikes": STRIKES,
    "strike": clean(run_strike_sweep(ExperimentConfig.from_dict(STRIKE), STRIKES,
                                     methods=["fourier_dense", "fourier_tt", "monte_carlo"])),
}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "experiments_ref.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
