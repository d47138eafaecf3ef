"""Dev probe: cfg5 instance 0, both crosses, per-sweep final_diff and price
(run under the dev library to A/B bond paths: TTP_DEV_LIBRARY=1 TTP_BOND_PATH=...)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

spec = configs.CONFIGS[5]
m = configs.make_model(5, int(os.environ.get("INST", "0")))
shape = (spec.grid.points_per_axis,) * spec.d
out = {"path": os.environ.get("TTP_BOND_PATH", "default")}
for sweeps in (1, 2, 3, 4):
    cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed, max_sweeps=sweeps, eps_tol=1e-300)
    t0 = time.time()
    _, rv = P.tt_cross(P.PayoffGridOracle(m, spec.grid, conj=True), shape, cfg)
    _, rp = P.tt_cross(P.PhiGridOracle(m, spec.grid), shape, cfg)
    out[sweeps] = {"v_diff": rv.final_diff, "phi_diff": rp.final_diff, "s": round(time.time() - t0, 2)}
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
out["price"] = P.price_fourier_tt(m, spec.grid, cfg, cfg, dense_reference="never").price
print(json.dumps(out))
