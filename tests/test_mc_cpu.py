"""Monte Carlo pricer: CPU-side checks.

* Philox4x32-10 known-answer vectors (Random123, the published algorithm
  the device sampler uses) through the numpy restatement AND through the
  library's own C routine (ttp_philox4x32, host-callable, no GPU needed).
* Host validation mirrors the reference's price_monte_carlo
  (pricers.py:309-312) and fires before any device work.
"""
import ctypes

import numpy as np
import pytest

import paper_2203_02804_b200 as P
from paper_2203_02804_b200 import _lib
from paper_2203_02804_b200.montecarlo import mc_params
from oracle import mc_philox as M
from conftest import BENCH

# Random123 kat_vectors: philox4x32_10 (counter, key) -> output
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers_numpy(ctr, key, want):
    got = M.philox4x32_10(*[[c] for c in ctr], *key)
    assert tuple(int(g[0]) for g in got) == want


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers_library(ctr, key, want):
    lib = _lib.load_library()
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    assert lib.ttp_philox4x32(c, k, o) == 0
    assert tuple(o) == want


def test_normals_are_standard():
    z = M.normals(np.arange(200_000, dtype=np.uint64), 0, 4, seed=11)
    assert abs(z.mean()) < 5e-3
    assert abs(z.std() - 1.0) < 5e-3
    c = np.corrcoef(z.T)
    assert np.max(np.abs(c - np.eye(4))) < 1e-2


def test_validation_matches_reference():
    m = P.MarketModel(d=1, **BENCH)
    with pytest.raises(ValueError):
        P.price_monte_carlo(m, 1, seed=0)            # pricers.py:309-310
    with pytest.raises(ValueError):
        P.price_monte_carlo(m, 100, seed=0, scheme="milstein")  # :311-312
    with pytest.raises(ValueError):
        P.price_monte_carlo(m, 100, seed=-1)
    with pytest.raises(ValueError):
        P.price_monte_carlo_batch([m, P.MarketModel(d=2, **BENCH)], 100, [0, 1])


def test_param_packing():
    m = P.MarketModel.with_plus_correlation(d=3, beta=0.5, **BENCH)
    lib = _lib.load_library()
    p = mc_params(m, "euler_path", n_steps=16, t=0.25)
    d = 3
    assert len(p) == lib.ttp_mc_param_count(d)
    np.testing.assert_array_equal(p[:d], m.s0)
    np.testing.assert_allclose(p[d:2 * d], (m.rates - 0.5 * m.sigma ** 2) * m.T)
    np.testing.assert_allclose(p[5 * d:5 * d + d * d].reshape(d, d), m.chol)
    assert p[-3] == m.strike
    assert p[-2] == pytest.approx(np.exp(-m.r * (m.T - 0.25)))
    assert p[-1] == pytest.approx(m.T / 16)
