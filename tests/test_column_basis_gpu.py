"""_column_basis (cross.py:103-119) as the bond kernel's global-slice path
computes it: TSQR (per-warp Householder chunks, triangle in tensor memory,
binary merge tree, cluster merge) followed by zlaqp2 on the final triangle
(csrc/k_tsqr.cuh), exported as ttp_column_basis.  Checked against the
reference's own algorithm -- scipy's pivoted QR, restated bit for bit by the
pinned oracle (oracle/ttp_oracle.py column_basis):

* orthonormality and span on every input, including the numerically
  rank-deficient phi / conj(vhat) unfolding blocks the cross actually factors
  (Householder QR keeps Q orthonormal whatever the conditioning);
* the same pivot order and the same columns up to a unimodular phase on
  well-conditioned inputs (the pivots depend on A only through A^H A, which
  the TSQR triangle carries exactly), and on the leading, well-separated
  pivots of the real blocks;
* the singular-input contract (zero block, rank_tol)."""

import numpy as np
import pytest

from conftest import load_npz
import paper_2203_02804_b200 as P
from paper_2203_02804_b200 import configs
from oracle import ttp_oracle as O

pytestmark = pytest.mark.gpu


def _rand(rng, n, m, r, scales=None):
    a = (rng.standard_normal((n, m, r)) + 1j * rng.standard_normal((n, m, r))) / np.sqrt(2.0)
    if scales is not None:
        a = a * scales
    return a


def _check_basis(a, q, tol=1e-13):
    r = a.shape[1]
    assert q.shape == a.shape
    assert np.max(np.abs(q.conj().T @ q - np.eye(r))) <= tol
    resid = a - q @ (q.conj().T @ a)
    assert np.linalg.norm(resid) <= tol * np.linalg.norm(a)


def _phase_match(q, qref, cols):
    """|<q_j, qref_j>| = 1 for j in cols: same pivot, same column up to phase."""
    ov = np.abs(np.einsum("ij,ij->j", q.conj(), qref))
    return ov[list(cols)]


@pytest.mark.parametrize("m,r", [(4128, 32), (4200, 20), (16448, 32), (8256, 8)])
def test_column_basis_matches_reference_on_well_conditioned_blocks(m, r):
    rng = np.random.default_rng([m, r])
    # graded column norms make the pivot order decisive, not a near tie
    scales = np.exp(rng.uniform(-3.0, 3.0, size=r))
    mats = _rand(rng, 3, m, r, scales)
    qs = P.column_basis(mats)
    for a, q in zip(mats, qs):
        _check_basis(a, q)
        qref = O.column_basis(a, 0.0)
        assert np.all(np.abs(_phase_match(q, qref, range(r)) - 1.0) <= 1e-10)


def test_column_basis_on_the_cross_blocks():
    """The cfg4 middle-bond unfoldings of phi(-z) and conj(vhat(z)) (the
    reference's own _block index sets, tests/golden/fibers.npz): sigma_min /
    sigma_max ~ 1e-16 or below, so only the leading pivots are decided by the
    data; Q stays orthonormal and spans the block."""
    fb = load_npz("fibers.npz")
    spec = configs.CONFIGS[4]
    grid = spec.grid
    shape = (grid.points_per_axis,) * spec.d
    m = configs.make_model(4)
    cases = [tuple(int(v) for v in c) for c in fb["cases"] if int(c[0]) == 4]
    checked = 0
    for cid, k, layout in cases:
        pre = f"c{cid}_k{k}_l{layout}"
        left, right = fb[pre + "_left"], fb[pre + "_right"]
        axis = k - 1 if layout == 0 else k
        for oracle in (P.PhiGridOracle(m, grid), P.PayoffGridOracle(m, grid, conj=True)):
            a = P.OracleBatch([oracle]).fiber_blocks(left, right, axis, shape, layout)[0]
            if a.size * 16 < (1 << 20):  # edge bonds: the one-CTA kernel's shapes
                continue
            q = P.column_basis(a)
            _check_basis(a, q, tol=1e-12)
            qref = O.column_basis(a, 0.0)
            sv = np.linalg.svd(a, compute_uv=False)
            lead = int(np.sum(sv > 1e-8 * sv[0]))  # numerically decided directions
            lead = min(lead, 8)
            assert np.all(np.abs(_phase_match(q, qref, range(lead)) - 1.0) <= 1e-8)
            checked += 1
    assert checked >= 2


def test_column_basis_singular_contract():
    rng = np.random.default_rng(5)
    with pytest.raises(ValueError):
        P.column_basis(np.ones((129, 32), dtype=np.complex128))  # below the global-slice block size
    a = _rand(rng, 1, 4128, 32)[0]
    with pytest.raises(P.SingularMatrixError):
        P.column_basis(np.zeros((4128, 32), dtype=np.complex128))
    dup = a.copy()
    dup[:, 7] = dup[:, 3]
    with pytest.raises(P.SingularMatrixError):
        P.column_basis(dup, rank_tol=1e-12)
    # rank_tol = 0 (the cross path, cross.py:343) accepts it; Q still orthonormal
    _check_basis(dup, P.column_basis(dup), tol=1e-12)


def test_column_basis_is_deterministic_and_batch_independent():
    rng = np.random.default_rng(11)
    mats = _rand(rng, 5, 4128, 32)
    one = P.column_basis(mats[3])
    batch = P.column_basis(mats)
    again = P.column_basis(mats)
    assert np.array_equal(batch, again)
    assert np.array_equal(one, batch[3])
