"""Reference TT price for config-5 instance 0 (d=20, 257 points, D=64).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_cfg5.py

About 10 minutes on one core.  Writes cfg5_ref.json with the
price, the cross reports (sweeps, calls, final_diff) and the wall time.
"""
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

import ttpricer as ref  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

spec = configs.CONFIGS[5]
g = spec.grid
grid = ref.GridSpec(n=g.n, eta=g.eta, alpha=g.alpha, d=g.d)
cfg = ref.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
m = ref.MarketModel(**configs.model_kwargs(configs.make_model(5, 0)))
t0 = time.time()
res = ref.price_fourier_tt(m, grid, cfg, cfg, dense_reference="never")
out = {"instance": 0, "price": res.price, "wall_s": time.time() - t0,
       "cross_phi": res.diagnostics["cross_phi"].to_dict(),
       "cross_v": res.diagnostics["cross_v"].to_dict()}
json.dump(out, open(os.path.join(HERE, "cfg5_ref.json"), "w"), indent=1)
print(out)
