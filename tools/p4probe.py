import sys, json
sys.path.insert(0, ".")
import numpy as np
import paper_2203_02804_b200 as P
from paper_2203_02804_b200 import configs
spec = configs.CONFIGS[4]
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
ref = json.load(open("tests/golden/golden.json"))["prices"]["cfg4_i0"]["price"]
for n in (1, 3, 17, 40):
    res = P.price_fourier_tt_batch([configs.make_model(4, i) for i in range(n)], spec.grid, cfg, cfg)
    r = res[0]
    print(n, r.price, f"rel {abs(r.price-ref)/ref:.2e}", r.diagnostics["cross_phi"].final_diff, r.diagnostics["cross_v"].final_diff)
