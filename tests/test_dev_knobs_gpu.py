"""The release library reads no environment: its A/B knobs are compiled in only
under -DTTP_DEV (csrc/dev_knobs.h, `make -C paper_2203_02804_b200/csrc dev`).
These tests load the dev library in subprocesses (TTP_DEV_LIBRARY=1) and check
that every knob setting which claims to be bitwise neutral reproduces the
release library's cores exactly, on a cfg4 batch of 17 (the global-slice
throughput path the benchmark runs, blocks of 4128 x 32)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEV_LIB = os.path.join(ROOT, "paper_2203_02804_b200", "libttpricer_b200_dev.so")

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2203_02804_b200 as P
from paper_2203_02804_b200 import _lib, configs
spec = configs.CONFIGS[4]
shape = (spec.grid.points_per_axis,) * spec.d
cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
ms = [configs.make_model(4, i) for i in range(17)]
out = {"lib": np.array(_lib.LIB_PATH)}
for tag, mk in (("phi", lambda m: P.PhiGridOracle(m, spec.grid)),
                ("v", lambda m: P.PayoffGridOracle(m, spec.grid, conj=True))):
    b = P.tt_cross_batch([mk(m) for m in ms], shape, cfg, with_reports=False)
    assert all(s == 0 for s in b.status)
    tr = b.trains.to_trains()
    for i in (0, 8, 16):
        for k, c in enumerate(tr[i].cores):
            out[f"{tag}_{i}_{k}"] = c
np.savez(sys.argv[1], **out)
"""


def _run(tmp_path, name, env_extra):
    script = tmp_path / "knob.py"
    script.write_text(_SCRIPT)
    env = {k: v for k, v in os.environ.items() if not k.startswith("TTP_")}
    env.update(env_extra)
    path = tmp_path / f"{name}.npz"
    subprocess.run([sys.executable, str(script), str(path)], check=True, env=env, cwd=ROOT, timeout=900)
    return np.load(path)


def _assert_same(a, b):
    keys = [k for k in a.files if k != "lib"]
    assert keys and sorted(keys) == sorted(k for k in b.files if k != "lib")
    for k in keys:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.fixture(scope="module")
def release(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("release")
    out = _run(tmp, "release", {})
    assert str(out["lib"]).endswith("libttpricer_b200.so")
    return out


def test_dev_library_is_built():
    assert os.path.exists(DEV_LIB), "build it with `make -C paper_2203_02804_b200/csrc dev`"


@pytest.mark.parametrize("knobs", [
    {},                          # dev build, knobs at their defaults
    {"TTP_SWAP_FILTER": "0"},    # every deferred swap pass over all rows
    {"TTP_LAZY": "1"},           # eager rank-1 swap updates
], ids=["defaults", "no_swap_filter", "eager_swaps"])
def test_dev_knob_is_bitwise_neutral(tmp_path, release, knobs):
    dev = _run(tmp_path, "dev", dict(knobs, TTP_DEV_LIBRARY="1"))
    assert str(dev["lib"]).endswith("libttpricer_b200_dev.so")
    _assert_same(dev, release)


def test_throughput_and_latency_instantiations_agree(tmp_path):
    """The 256-thread two-CTAs-per-SM instantiation (shipped for r <= 32) and
    the 512-thread one (shipped for r = 64) give the same cores when the
    column basis is the restated zlaqp2 with separate partials passes
    (TTP_TSQR=0, TTP_FUSED_QR=0): the TSQR splits rows per warp and the fused
    pass sums its dot products per warp, so both round by the CTA width."""
    knobs = {"TTP_DEV_LIBRARY": "1", "TTP_FUSED_QR": "0", "TTP_TSQR": "0"}
    tp = _run(tmp_path, "tp", dict(knobs, TTP_CK="tp"))
    lat = _run(tmp_path, "lat", dict(knobs, TTP_CK="lat"))
    _assert_same(tp, lat)
