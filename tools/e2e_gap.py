"""Where the e2e (public API, host inputs) step spends time beyond the
device-resident step (dev tool).  Usage: python tools/e2e_gap.py [CID] [N]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402
from paper_2203_02804_b200.pricers import price_fourier_tt_batch_capi, run_cross_pair  # noqa: E402

CID = int(sys.argv[1]) if len(sys.argv) > 1 else 4
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 592
sp = configs.CONFIGS[CID]
grid = sp.grid
shape = (grid.points_per_axis,) * grid.d
cfg = P.CrossConfig(bond_dim=sp.bond_dim, seed=sp.cross_seed)
models = [configs.make_model(CID, i) for i in range(NB)]
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

# segment timing of one public call
import paper_2203_02804_b200.pricers as PR  # noqa: E402
t0 = time.perf_counter()
ob = (P.OracleBatch([P.PhiGridOracle(m, grid) for m in models]), P.OracleBatch([P.PayoffGridOracle(m, grid, conj=True) for m in models]))
t1 = time.perf_counter()
rp, rv = run_cross_pair(ob[0], ob[1], shape, cfg, cfg)
torch.cuda.synchronize()
t2 = time.perf_counter()
raw = P.tt_inner_batch(rv.trains, rp.trains)
t3 = time.perf_counter()
res = []
for i, m in enumerate(models):
    err = rp.error_for(i) or rv.error_for(i)
    value = PR._prefactor(m, grid, 0.0) * raw[i]
    diag = {"cross_phi": rp.reports[i], "cross_v": rv.reports[i], "imag_part": float(value.imag),
            "oracle_calls_total": rp.reports[i].oracle_calls + rv.reports[i].oracle_calls}
    res.append(PR.PricingResult(float(value.real), "fourier_tt", 0.0, diag))
t4 = time.perf_counter()
print(f"oracles {1e3*(t1-t0):.1f} ms, crosses {1e3*(t2-t1):.1f} ms, inner {1e3*(t3-t2):.1f} ms, results {1e3*(t4-t3):.1f} ms")
