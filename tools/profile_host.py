"""cProfile of the public batch API's host side at the bench batch (dev tool)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

sp = configs.CONFIGS[4]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 592
models = [configs.make_model(4, i) for i in range(n)]
cfg = P.CrossConfig(bond_dim=sp.bond_dim, seed=sp.cross_seed)
P.price_fourier_tt_batch(models, sp.grid, cfg, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
P.price_fourier_tt_batch(models, sp.grid, cfg, cfg)
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
