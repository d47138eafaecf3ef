"""Device error paths of the cross (reference cross.py:343-355 and
_column_basis cross.py:110-118): a zero unfolding block raises
SingularMatrixError carrying the bond index -- the reference raises
"singular cross block at bond 1: matrix of shape (8, 2) is zero" for a zero
oracle on (8, 8, 8) at bond_dim 2 -- and inside a batch the failing instance
is reported through its status while its neighbours are priced exactly as
they are alone.  Covered on both bond kernels: the one-CTA kernel (small
blocks) and the global-slice cluster kernel with the TSQR column basis
(4128 x 32 blocks, the benchmark's shape)."""

import numpy as np
import pytest

import paper_2203_02804_b200 as P

pytestmark = pytest.mark.gpu


def _sep(rng, n, d, zero=False):
    w = [rng.standard_normal(n) + 1j * rng.standard_normal(n) for _ in range(d)]
    if zero:
        w[0] = np.zeros(n, dtype=np.complex128)
    return P.SeparableOracle(w)


def test_zero_block_raises_with_bond_index():
    rng = np.random.default_rng(3)
    with pytest.raises(P.SingularMatrixError) as ei:
        P.tt_cross(_sep(rng, 8, 3, zero=True), (8, 8, 8), P.CrossConfig(bond_dim=2, n_conv_samples=100, seed=0))
    assert ei.value.bond == 1


def _tt(rng, n, d, bond, zero=False):
    bonds = [1] + [min(bond, n ** k, n ** (d - k)) for k in range(1, d)] + [1]
    cores = [(rng.standard_normal((bonds[k], n, bonds[k + 1])) + 1j * rng.standard_normal((bonds[k], n, bonds[k + 1])))
             / np.sqrt(2.0 * bonds[k]) for k in range(d)]
    if zero:
        cores[0] = np.zeros_like(cores[0])
    return P.TTOracle(P.TensorTrain(cores))


@pytest.mark.parametrize("n,d,bond", [(8, 3, 2), (129, 4, 32)], ids=["one-cta", "global-slice"])
def test_failing_instance_in_a_batch_leaves_neighbours_intact(n, d, bond):
    """The zero instance fails at bond 1 and is skipped by every later launch
    (at (129,)^4, D = 32 the later bonds run the global-slice cluster kernel
    with the TSQR column basis on 4128 x 32 blocks); its neighbours' cores are
    bitwise their single-instance cores."""
    rng = np.random.default_rng([n, d])
    oracles = [_tt(rng, n, d, bond), _tt(rng, n, d, bond, zero=True), _tt(rng, n, d, bond)]
    cfg = P.CrossConfig(bond_dim=bond, n_conv_samples=200, seed=5, max_sweeps=1)
    shape = (n,) * d
    res = P.tt_cross_batch(oracles, shape, cfg)
    err = res.error_for(1)
    assert isinstance(err, P.SingularMatrixError) and err.bond == 1
    assert res.error_for(0) is None and res.error_for(2) is None
    trains = res.trains.to_trains()
    for i in (0, 2):
        alone, rep = P.tt_cross(oracles[i], shape, cfg)
        for a, b in zip(alone.cores, trains[i].cores):
            np.testing.assert_array_equal(a, b)
        assert rep.final_diff <= 1e-10  # an exact-rank target is reconstructed to rounding
