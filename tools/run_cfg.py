"""Price n instances of a BASELINE config on the GPU and report timing (dev tool)."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import _lib, configs  # noqa: E402

cid = int(sys.argv[1])
n = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
spec = configs.CONFIGS[cid]
models = [configs.make_model(cid, i) for i in range(n)]
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
for rep in range(reps):
    _lib.profile_reset()
    _lib.profile_enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.price_fourier_tt_batch(models, spec.grid, cfg, cfg, raise_errors=False)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    _lib.profile_enable(False)
    st = _lib.profile_read()
    out = {"cfg": cid, "n": n, "wall_s": wall, "options_per_s": n / wall,
           "prices": [r.price if not isinstance(r, Exception) else repr(r) for r in res[:4]],
           "sweeps": [[r.diagnostics["cross_phi"].sweeps_used, r.diagnostics["cross_v"].sweeps_used]
                      for r in res[:4] if not isinstance(r, Exception)],
           "diffs": [[r.diagnostics["cross_phi"].final_diff, r.diagnostics["cross_v"].final_diff]
                     for r in res[:4] if not isinstance(r, Exception)],
           "kernels_ms": {k: round(v[2], 2) for k, v in st.items() if v[0]}}
    print(json.dumps(out), flush=True)
