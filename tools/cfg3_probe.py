"""Config-3 instances 0..N-1: device TT price, device dense sum, and the
reference's TT price (tests/golden), side by side (dev tool for the bench's
parity bands).  Usage: python tools/cfg3_probe.py [N]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ref = json.load(open(os.path.join(root, "tests", "golden", "cfg3_ref_prices.json")))["instances"]
bands = json.load(open(os.path.join(root, "tests", "golden", "noise_bands.json")))
spec = configs.CONFIGS[3]
models = [configs.make_model(3, i) for i in range(n)]
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
res = P.price_fourier_tt_batch(models, spec.grid, cfg, cfg)
dense = P.price_fourier_dense_batch(models, spec.grid, term_cap=2_000_000_000)
for i in range(n):
    g, d, r = res[i].price, dense[i].price, ref[i]["price"]
    b = bands.get(f"cfg3_i{i}", {}).get("max", float("nan"))
    print(f"i{i:2d} K={models[i].strike:7.2f} T={models[i].T:.2f} dense {d:.9g} gpu {g:.9g} ref {r:.9g}  "
          f"|gpu-dense|/dense {abs(g - d) / abs(d):.2e} |ref-dense|/dense {abs(r - d) / abs(d):.2e} "
          f"|gpu-ref|/ref {abs(g - r) / abs(r):.2e} band {b:.2e} "
          f"diff_phi {res[i].diagnostics['cross_phi'].final_diff:.2e} diff_v {res[i].diagnostics['cross_v'].final_diff:.2e}", flush=True)
