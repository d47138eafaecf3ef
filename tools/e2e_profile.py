"""cProfile of one public-API batch call (host-side overhead of the e2e path;
dev tool).  Usage: python tools/e2e_profile.py [CID] [N]"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

CID = int(sys.argv[1]) if len(sys.argv) > 1 else 3
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
sp = configs.CONFIGS[CID]
cfg = P.CrossConfig(bond_dim=sp.bond_dim, seed=sp.cross_seed)
models = [configs.make_model(CID, i) for i in range(NB)]
for _ in range(2):
    P.price_fourier_tt_batch(models, sp.grid, cfg, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
P.price_fourier_tt_batch(models, sp.grid, cfg, cfg)
torch.cuda.synchronize()
print(f"one call: {1e3 * (time.perf_counter() - t0):.1f} ms")
pr = cProfile.Profile()
pr.enable()
P.price_fourier_tt_batch(models, sp.grid, cfg, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(28)
