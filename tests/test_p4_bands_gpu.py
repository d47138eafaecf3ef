"""P4 per instance: the device TT price against the REFERENCE's own price
(tests/golden/ref_prices_r02.json, ttpricer.price_fourier_tt on the same
seeded instances) within that instance's reproducibility band
(tests/golden/noise_bands.json): how far the reference's price moves when its
oracle values are perturbed by 1e-15 relative noise, the maximum over 12-16
noise seeds.  The end-to-end price cannot be held to 1e-8 by any independent
implementation (the sampled unfoldings are numerically rank
deficient, so rounding picks the trailing interpolation directions); this is
the honest yardstick, instance by instance.  BAND_FACTOR covers the finite
number of noise seeds behind each band."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2203_02804_b200 as P
from paper_2203_02804_b200 import configs

pytestmark = pytest.mark.gpu

BAND_FACTOR = 2.0


def _golden():
    with open(os.path.join(GOLDEN, "ref_prices_r02.json")) as fh:
        ref = json.load(fh)
    with open(os.path.join(GOLDEN, "noise_bands.json")) as fh:
        bands = json.load(fh)
    return ref, bands


@pytest.mark.parametrize("cid,n_inst", [(1, 1), (2, 4), (3, 8), (4, 16)])
def test_p4_prices_within_per_instance_reference_band(cid, n_inst):
    ref, bands = _golden()
    spec = configs.CONFIGS[cid]
    models = [configs.make_model(cid, i) for i in range(n_inst)]
    cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
    res = P.price_fourier_tt_batch(models, spec.grid, cfg, cfg)
    rows = []
    for i, r in enumerate(res):
        key = f"cfg{cid}_i{i}"
        want = ref[key]["price"] if key in ref else bands[key]["unperturbed"]
        assert bands[key]["unperturbed"] == want  # the band was measured around the reference's price
        dev = abs(r.price - want) / abs(want)
        band = bands[key]["max"]
        rows.append((i, dev, band))
        if key in ref:
            assert r.diagnostics["cross_phi"].oracle_calls == ref[key]["cross_phi"]["oracle_calls"]
            assert r.diagnostics["cross_v"].sweeps_used == ref[key]["cross_v"]["sweeps_used"]
    print("\n" + "\n".join(f"  cfg{cid} i{i}: |gpu-ref|/ref {dev:.2e}  reference band {band:.2e}  ratio {dev / band:.2f}"
                           for i, dev, band in rows))
    for i, dev, band in rows:
        assert dev <= BAND_FACTOR * band, f"cfg{cid} instance {i}: {dev:.3e} > {BAND_FACTOR} x {band:.3e}"
    devs = np.array([r[1] for r in rows])
    meds = np.array([bands[f"cfg{cid}_i{i}"]["median"] for i in range(n_inst)])
    # typical deviations are the size of the reference's typical noise response
    assert np.median(devs) <= BAND_FACTOR * max(np.median(meds), 1e-12)
