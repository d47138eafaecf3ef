"""Per-phase clock64 marks of the cluster bond kernel (dev tool; the phase
clocks exist only in the -DTTP_DEV library, so this loads it)."""
import ctypes
import os
import sys
import time

os.environ["TTP_DEV_LIBRARY"] = "1"

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import _lib, configs  # noqa: E402

lib = _lib.load_library()
names = ["load", "colbasis", "-", "start1", "start2", "swaps1", "swaps2", "final", "end"]
cases = [tuple(int(x) for x in c.split(":")) for c in os.environ.get("PT_CASES", "4:1,4:148,2:1,1:1").split(",")]
for cid, nb in cases:
    spec = configs.CONFIGS[cid]
    models = [configs.make_model(cid, i) for i in range(nb)]
    shape = (spec.grid.points_per_axis,) * spec.d
    cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed, max_sweeps=1)
    ob = P.OracleBatch([P.PhiGridOracle(m, spec.grid) for m in models])
    P.tt_cross_batch(ob, shape, cfg, with_reports=False)
    torch.cuda.synchronize()
    lib.ttp_dev_phase_clocks(1, None, 0)
    out = (ctypes.c_int64 * 32)()
    _lib.profile_reset(); _lib.profile_enable(True)
    t0 = time.perf_counter()
    P.tt_cross_batch(ob, shape, cfg, with_reports=False)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    _lib.profile_enable(False)
    st = _lib.profile_read()
    lib.ttp_dev_phase_clocks(0, out, 32)
    clk = [out[i] for i in range(9)]
    ghz = 1.965
    marks = []
    for k in range(1, 9):
        if clk[k] and clk[k - 1] and clk[k] >= clk[0]:
            marks.append(f"{names[k]}={(clk[k] - clk[k - 1]) / ghz / 1e3:.1f}us")
    print(f"cfg{cid} batch {nb}: wall {wall * 1e3:.1f} ms; bond kernel {st['cluster_bond_kernel'][2] + st['bond_kernel'][2]:.2f} ms / "
          f"{st['cluster_bond_kernel'][0] + st['bond_kernel'][0]} launches; conv {st['conv_site_kernel'][2]:.2f} ms; last bond phases: "
          + " ".join(marks) + f"; total {(clk[8] - clk[0]) / ghz / 1e3:.1f}us", flush=True)
    sub = ["pivot+recomp", "partials", "clsync", "reduce", "update", "wy.gram", "wy.exchange"]
    print("    colbasis sub-phases (all bonds of the sweep): " + " ".join(
        f"{sub[k]}={out[16 + k] / ghz / 1e3:.1f}us" for k in range(7))
        + f" wy.T={out[16 + 14] / ghz / 1e3:.1f}us wy.M+sync={out[16 + 15] / ghz / 1e3:.1f}us"
        + f" | slot6={out[16 + 6] / ghz / 1e3:.1f}us slot7={out[16 + 7] / ghz / 1e3:.1f}us raw14={out[16 + 14]} raw15={out[16 + 15]}", flush=True)
    sub2 = ["sw.publish", "sw.clsync", "sw.winner", "sw.barrier", "sw.selb", "sw.rowpass"]
    print("    swap sub-phases (all bonds, both runs): " + " ".join(
        f"{sub2[k]}={out[24 + k] / ghz / 1e3:.1f}us" for k in range(6)), flush=True)
