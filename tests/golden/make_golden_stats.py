"""Reference TT prices for many cfg3 instances (statistical P4 yardstick).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_stats.py

Writes tests/golden/cfg3_ref_prices.json: the reference's price_fourier_tt
(dense_reference='never') for config-3 instances 0..N-1.  Dense prices are
not stored: the GPU dense sum (validated against the reference's own dense
sums in golden.json, including the 65^5 cfg2 sum) provides them in the test.
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

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
spec = configs.CONFIGS[3]
g = spec.grid
grid = ref.GridSpec(n=g.n, eta=g.eta, alpha=g.alpha, d=g.d)
cfg = ref.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
out = {"config": 3, "instances": [], "reference": "ttpricer " + ref.__version__}
t0 = time.time()
for i in range(N):
    m = ref.MarketModel(**configs.model_kwargs(configs.make_model(3, i)))
    res = ref.price_fourier_tt(m, grid, cfg, cfg, dense_reference="never")
    out["instances"].append({"i": i, "price": res.price,
                             "sweeps": [res.diagnostics["cross_phi"].sweeps_used,
                                        res.diagnostics["cross_v"].sweeps_used]})
out["wall_s"] = time.time() - t0
json.dump(out, open(os.path.join(HERE, "cfg3_ref_prices.json"), "w"), indent=1)
print("done", out["wall_s"])
