"""Per-instance parity probe (dev tool): GPU TT price of instances 0..N-1 of a
BASELINE config against the reference's own unperturbed price and noise band
(tests/golden/noise_bands.json) and against the dense full-grid sum where it
is feasible (d <= 5).  Usage: python tools/cfg_probe.py CID N"""
import json
import sys

sys.path.insert(0, ".")
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

cid, n = int(sys.argv[1]), int(sys.argv[2])
spec = configs.CONFIGS[cid]
bands = json.load(open("tests/golden/noise_bands.json"))
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
models = [configs.make_model(cid, i) for i in range(n)]
res = P.price_fourier_tt_batch(models, spec.grid, cfg, cfg)
for i, r in enumerate(res):
    b = bands.get(f"cfg{cid}_i{i}")
    dense = P.price_fourier_dense(models[i], spec.grid, term_cap=2_000_000_000).price if spec.d <= 5 else float("nan")
    ref = b["unperturbed"] if b else float("nan")
    rel = abs(r.price - ref) / abs(ref) if b else float("nan")
    band = b["max"] if b else float("nan")
    print(f"i{i}: gpu {r.price:.12g} ref {ref:.12g} dense {dense:.12g} rel {rel:.2e} band {band:.2e} "
          f"ratio {rel / band:.2f} ref-dense {abs(ref - dense) / abs(dense):.2e} gpu-dense {abs(r.price - dense) / abs(dense):.2e} "
          f"sweeps {r.diagnostics['cross_phi'].sweeps_used}/{r.diagnostics['cross_v'].sweeps_used}")
