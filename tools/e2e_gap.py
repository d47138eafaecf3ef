"""Where the e2e (public API, host inputs) step spends time beyond the
device-resident step (dev tool)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402
from paper_2203_02804_b200.pricers import price_fourier_tt_batch_capi, run_cross_pair  # noqa: E402

sp = configs.CONFIGS[4]
grid = sp.grid
shape = (grid.points_per_axis,) * grid.d
cfg = P.CrossConfig(bond_dim=sp.bond_dim, seed=sp.cross_seed)
models = [configs.make_model(4, i) for i in range(592)]
phi_b = P.OracleBatch([P.PhiGridOracle(m, grid) for m in models])
v_b = P.OracleBatch([P.PayoffGridOracle(m, grid, conj=True) for m in models])


def timed(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name:40s} {1e3 * min(ts):8.1f} ms (min of {reps}), {1e3 * np.median(ts):8.1f} median", flush=True)


timed("device step, no reports", lambda: P.tt_inner_batch(*[r.trains for r in run_cross_pair(phi_b, v_b, shape, cfg, cfg, with_reports=False)][::-1]))
timed("device step, reports", lambda: P.tt_inner_batch(*[r.trains for r in run_cross_pair(phi_b, v_b, shape, cfg, cfg, with_reports=True)][::-1]))
timed("oracle batches from models", lambda: (P.OracleBatch([P.PhiGridOracle(m, grid) for m in models]),
                                              P.OracleBatch([P.PayoffGridOracle(m, grid, conj=True) for m in models])))
timed("price_fourier_tt_batch", lambda: P.price_fourier_tt_batch(models, grid, cfg, cfg, dense_reference="never"))
timed("price_fourier_tt_batch_capi", lambda: price_fourier_tt_batch_capi(models, grid, cfg, cfg))
