"""Monte Carlo throughput (paths/s) on the GPU vs the reference's numpy MC (dev tool).

usage: python tools/bench_mc.py [d] [n_paths]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2203_02804_b200 as P  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000
BENCH = dict(r=0.3, sigma=0.5, T=1.0, s0=100.0, strike=100.0)
m = P.MarketModel.with_plus_correlation(d=d, beta=0.5, **BENCH)
out = {"d": d, "paths": n}
for scheme, steps in (("terminal_exact", 64), ("euler_path", 64)):
    nn = n if scheme == "terminal_exact" else n // 64
    P.price_monte_carlo(m, 1000, seed=1, scheme=scheme, n_steps=steps)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.price_monte_carlo(m, nn, seed=1, scheme=scheme, n_steps=steps)
    dt = time.perf_counter() - t0
    out[scheme] = {"paths": nn, "s": dt, "paths_per_s": nn / dt, "price": r.price,
                   "std_error": r.diagnostics["std_error"]}
print(json.dumps(out))
