"""bench.py's parity judge (host logic, no GPU): per instance, in price units,
within BAND_FACTOR x max(the instance's own reference noise band, the config's
median absolute band) of the reference's price (tests/golden/ref_prices_r02.json,
noise_bands.json -- both produced by the reference itself)."""
import importlib.util
import json
import os

import numpy as np

from conftest import GOLDEN

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_module", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _refs(cid, n):
    bands = json.load(open(os.path.join(GOLDEN, "noise_bands.json")))
    return np.array([bands[f"cfg{cid}_i{i}"]["unperturbed"] for i in range(n)]), \
        np.array([bands[f"cfg{cid}_i{i}"]["max"] for i in range(n)])


def test_reference_prices_pass_with_zero_ratio():
    b = _bench()
    ref, _ = _refs(4, 16)
    out = b.parity_check(4, list(ref), None)
    assert out["ok"] and out["n"] == 16 and out["max_band_ratio"] == 0.0
    assert out["against"] == ["reference golden"]
    assert b.reference_prices(4, 16, None) == list(ref)


def test_a_price_three_bands_off_fails():
    b = _bench()
    ref, band = _refs(4, 16)
    # the instance with the widest absolute band: the floor cannot rescue it
    i = int(np.argmax(band * np.abs(ref)))
    prices = list(ref)
    prices[i] = ref[i] * (1.0 + 3.0 * b.BAND_FACTOR * band[i])
    out = b.parity_check(4, prices, None)
    assert not out["ok"]
    assert out["worst"]["instance"] == i and out["max_band_ratio"] > 1.0


def test_near_zero_price_is_judged_in_price_units():
    """Config 3, instance 10 (a 9.5e-4 option): 3.6% off its reference price is
    1.4x its own relative band but 3.5e-5 in price units, inside twice the
    config's median absolute band; the judge reports both."""
    b = _bench()
    ref, band = _refs(3, 16)
    prices = list(ref)
    prices[10] = 0.00091529717  # the device price measured on the B200 (tools/cfg3_probe.py)
    out = b.parity_check(3, prices, None)
    assert out["ok"]
    assert out["worst"]["instance"] == 10
    assert out["n_within_own_band"] == 15
    assert 1.0 < out["max_ratio_to_own_band"] < 2.0
    floor = float(np.median(band * np.abs(ref)))
    assert abs(out["abs_band_floor"] - floor) <= 1e-18
    # the same relative miss on a large price is not excused by the floor
    prices = list(ref)
    prices[2] = ref[2] * (1.0 + 0.036)
    assert not b.parity_check(3, prices, None)["ok"]


def test_live_port_prices_are_the_fallback():
    """Instances without a committed reference price are judged against the
    live CPU port's price of the same instance."""
    b = _bench()
    ref, _ = _refs(2, 4)
    port = list(ref) + [3.0, 4.0, 5.0, 6.0]   # config 2 has goldens for instances 0-3 only
    out = b.parity_check(2, list(port), port)
    assert out["ok"] and out["n"] == 8 and out["max_band_ratio"] == 0.0
    assert out["against"] == ["live CPU port", "reference golden"]
    bad = list(port)
    bad[6] *= 1.5
    assert not b.parity_check(2, bad, port)["ok"]
