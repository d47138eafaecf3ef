"""P3 at the benchmark's block sizes: the reference's tt_cross
(cross.py:358-453) on a seeded rank-32 tensor train over (129,)^10 -- the
cfg4 shape, unfoldings of 4128 x 32 that are numerically full rank, so the
maxvol decisions are well posed -- with both sweep directions
forced (tests/golden/make_golden_r02.py tt32).  Every bond kernel the
benchmark launches takes part: bonds whose blocks are >= 1 MB run the
global-slice cluster kernel (fused QR, fused starts, filtered deferred swaps),
the 129 x 32 edge bonds run the one-CTA kernel.  Left/right pivot sets, call
counts and sweeps must be identical to the reference's."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, sets_as_lists
import paper_2203_02804_b200 as P

pytestmark = pytest.mark.gpu


def tt32_target():
    # same draw as make_golden_r02.tt32_target
    rng = np.random.default_rng(2032)
    d, n, D = 10, 129, 32
    bonds = [1] + [D] * (d - 1) + [1]
    cores = []
    for k in range(d):
        shp = (bonds[k], n, bonds[k + 1])
        cores.append((rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / np.sqrt(2.0 * bonds[k]))
    return P.TensorTrain(cores)


@pytest.fixture(scope="module")
def golden32():
    with open(os.path.join(GOLDEN, "tt32_cross.json")) as fh:
        return json.load(fh)


def _check(rep, g):
    assert rep.sweeps_used == g["report"]["sweeps_used"] == 2
    assert rep.converged == g["report"]["converged"]
    assert rep.oracle_calls == g["report"]["oracle_calls"]
    assert rep.conv_check_calls == g["report"]["conv_check_calls"]
    assert sets_as_lists(rep.left_sets) == g["left_sets"]
    assert sets_as_lists(rep.right_sets) == g["right_sets"]
    # exact-rank target: both sides reconstruct it to rounding
    assert rep.final_diff <= 1e-12 and g["report"]["final_diff"] <= 1e-12


def test_rank32_cross_decisions_identical_to_reference(golden32):
    target = tt32_target()
    c = golden32["cfg"]
    cfg = P.CrossConfig(bond_dim=c["bond_dim"], eps_tol=c["eps_tol"], max_sweeps=c["max_sweeps"],
                        n_conv_samples=c["n_conv_samples"], seed=c["seed"])
    tt, rep = P.tt_cross(P.TTOracle(target), (129,) * 10, cfg)
    _check(rep, golden32)
    inner = P.tt_inner(tt, tt)
    want = complex(*golden32["inner_self"])
    assert abs(inner - want) <= 1e-10 * abs(want)


def test_rank32_cross_decisions_in_a_batch(golden32):
    """The same cross as instance 0 and 16 of a batch of 17 (two instances
    per SM on the throughput kernel): identical decisions and cores."""
    target = tt32_target()
    c = golden32["cfg"]
    cfg = P.CrossConfig(bond_dim=c["bond_dim"], eps_tol=c["eps_tol"], max_sweeps=c["max_sweeps"],
                        n_conv_samples=c["n_conv_samples"], seed=c["seed"])
    batch = P.tt_cross_batch([P.TTOracle(target) for _ in range(17)], (129,) * 10, cfg)
    assert all(s == 0 for s in batch.status)
    trains = batch.trains.to_trains()
    for i in (0, 16):
        _check(batch.reports[i], golden32)
    for a, b in zip(trains[0].cores, trains[16].cores):
        np.testing.assert_array_equal(a, b)
