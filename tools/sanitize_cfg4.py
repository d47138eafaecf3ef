"""compute-sanitizer target: one cfg4 batch of 17 options through the public
batch API (global-slice throughput path: TSQR column basis, fused starts,
filtered deferred swaps, DMMA convergence check, tt_inner)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

n = int(os.environ.get("N_OPT", "17"))
spec = configs.CONFIGS[4]
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed, max_sweeps=int(os.environ.get("SWEEPS", "1")))
res = P.price_fourier_tt_batch([configs.make_model(4, i) for i in range(n)], spec.grid, cfg, cfg)
print("prices", [round(r.price, 10) for r in res[:4]], "...", flush=True)
