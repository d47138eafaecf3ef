"""Dev tool: per-instance duration spread of the last cluster bond launch of a
cfg4 sweep (dev library: globaltimer marks of cluster rank 0)."""
import ctypes
import os
import sys

os.environ["TTP_DEV_LIBRARY"] = "1"
import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import _lib, configs  # noqa: E402

lib = _lib.load_library()
lib.ttp_dev_inst_times.restype = ctypes.c_int32
lib.ttp_dev_inst_times.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]
nb = int(os.environ.get("NB", "148"))
spec = configs.CONFIGS[4]
models = [configs.make_model(4, i) for i in range(nb)]
shape = (spec.grid.points_per_axis,) * spec.d
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed, max_sweeps=1)
ob = P.OracleBatch([P.PhiGridOracle(m, spec.grid) for m in models])
P.tt_cross_batch(ob, shape, cfg, with_reports=False)
torch.cuda.synchronize()
lib.ttp_dev_phase_clocks(1, None, 0)
P.tt_cross_batch(ob, shape, cfg, with_reports=False)
torch.cuda.synchronize()
out = (ctypes.c_int64 * (3 * nb))()
rc = lib.ttp_dev_inst_times(out, nb)
clk = (ctypes.c_int64 * 32)()
rc2 = lib.ttp_dev_phase_clocks(0, clk, 32)
print('rc', rc, rc2, list(clk)[:9])
a = np.frombuffer(out, dtype=np.int64).reshape(3, nb)
t0 = a[0].min()
st, en, sm = (a[0] - t0) / 1e3, (a[1] - t0) / 1e3, a[2]
dur = en - st
q = np.percentile(dur, [0, 10, 50, 90, 100])
print(f"batch {nb}: launch span {en.max():.0f} us; instance duration us min/p10/p50/p90/max "
      + "/".join(f"{x:.0f}" for x in q) + f"; start spread {st.max():.0f} us; distinct SMs {len(set(sm.tolist()))}")
order = np.argsort(-dur)[:8]
print("slowest:", ", ".join(f"i{i} sm{sm[i]} start {st[i]:.0f} dur {dur[i]:.0f}" for i in order))
print("fastest:", ", ".join(f"i{i} sm{sm[i]} start {st[i]:.0f} dur {dur[i]:.0f}" for i in np.argsort(dur)[:5]))
