"""Run one config-4 TT-cross (phi) for a single instance twice (profiling target)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = configs.CONFIGS[cid]
models = [configs.make_model(cid, i) for i in range(nb)]
shape = (spec.grid.points_per_axis,) * spec.d
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed, max_sweeps=1)
ob = P.OracleBatch([P.PhiGridOracle(m, spec.grid) for m in models])
for _ in range(2):
    P.tt_cross_batch(ob, shape, cfg, with_reports=False)
torch.cuda.synchronize()
print("ok")
