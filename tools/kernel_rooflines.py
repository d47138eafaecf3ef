"""Drive each secondary kernel once at a representative size (dev tool; the
ncu captures of tools/kernel_rooflines.sh wrap it).

usage: python tools/kernel_rooflines.py dense|fiber|mc
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

what = sys.argv[1]
t0 = time.perf_counter()
if what == "dense":
    # cfg2 full grid: 65^5 = 1.16e9 terms of phi(-z) * vhat(z)
    spec = configs.CONFIGS[2]
    m = configs.make_model(2, 0)
    P.price_fourier_dense(m, spec.grid, term_cap=10**10)  # context, library, first launch
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = P.price_fourier_dense(m, spec.grid, term_cap=10**10)
    dt = time.perf_counter() - t1
    print("dense price", r.price, "terms", spec.grid.n_terms, f"second call {dt * 1e3:.1f} ms",
          f"{spec.grid.n_terms / dt / 1e9:.2f} G terms/s")
elif what == "fiber":
    # cfg2 batch of 1024: one-CTA bond kernel with the separable fiber evaluator
    spec = configs.CONFIGS[2]
    models = [configs.make_model(2, i) for i in range(1024)]
    cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
    shape = (spec.grid.points_per_axis,) * spec.d
    b = P.tt_cross_batch([P.PhiGridOracle(m, spec.grid) for m in models], shape, cfg, with_reports=False)
    print("fiber ok", int((b.status == 0).sum()))
elif what == "inner64":
    # D = 64 trains (cfg5-like): the cluster-split inner product
    rng = np.random.default_rng(5)
    phys, bonds = [257] * 6, [1, 64, 64, 64, 64, 64, 1]
    def rnd():
        return P.TensorTrain([rng.standard_normal((bonds[k], phys[k], bonds[k + 1])) + 0j for k in range(6)])
    a, b = rnd(), rnd()
    P.tt_inner(a, b)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    v = P.tt_inner(a, b)
    print("inner64", v, f"{(time.perf_counter() - t1) * 1e3:.1f} ms")
elif what == "mc":
    models = [configs.make_model(4, i) for i in range(8)]
    res = P.price_monte_carlo_batch(models, 1 << 22, seeds=list(range(8)))
    print("mc", [round(x.price, 6) for x in res[:2]])
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0)
