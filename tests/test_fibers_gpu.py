"""P0 at the blocks the cores are built from: ttp_eval_fibers -- the same
separable device evaluation the bond kernels' fiber loads use
(fiber_fast.cuh) -- against unfolding blocks the REFERENCE's own ``_block``
(cross.py:310-332) produced with one oracle call each
(tests/golden/make_golden_r02.py fibers): phi(-z) and conj(vhat(z)) on
BASELINE configs 1-5, left-to-right and right-to-left layouts, edge and
middle bonds.  Tolerance: 1e-12 relative per entry (2e-12 at cfg5, d=20),
the P0 contract of SURVEY.md 8(c)."""

import numpy as np
import pytest

from conftest import load_npz
import paper_2203_02804_b200 as P
from paper_2203_02804_b200 import configs

pytestmark = pytest.mark.gpu


def _cases():
    return [tuple(int(v) for v in c) for c in load_npz("fibers.npz")["cases"]]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"cfg{c[0]}-bond{c[1]}-{'l2r' if c[2] == 0 else 'r2l'}")
def test_fiber_blocks_match_reference_block(case):
    cid, k, layout = case
    fb = load_npz("fibers.npz")
    spec = configs.CONFIGS[cid]
    grid, d = spec.grid, spec.d
    shape = (grid.points_per_axis,) * d
    axis = k - 1 if layout == 0 else k
    pre = f"c{cid}_k{k}_l{layout}"
    left, right = fb[pre + "_left"], fb[pre + "_right"]
    m = configs.make_model(cid)
    tol = 2e-12 if cid == 5 else 1e-12
    for kind, oracle in (("phi", P.PhiGridOracle(m, grid)), ("vhat", P.PayoffGridOracle(m, grid, conj=True))):
        tall = P.OracleBatch([oracle]).fiber_blocks(left, right, axis, shape, layout)[0]
        n_left, n_right = left.shape[0], right.shape[0]
        assert tall.shape == ((n_left * grid.points_per_axis, n_right) if layout == 0
                              else (grid.points_per_axis * n_right, n_left))
        # one reference oracle call per block, of rows x cols entries
        assert int(fb[f"{pre}_{kind}_calls"][0]) == tall.size
        rows, want = fb[f"{pre}_{kind}_rows"], fb[f"{pre}_{kind}_vals"]
        got = tall[rows]
        err = np.max(np.abs(got - want) / np.abs(want))
        assert err <= tol, f"{kind}: max rel err {err:.3e}"


def test_sample_block_is_reference_block_shaped():
    """cross.sample_block returns the reference's (block, row_tuples,
    col_tuples) orientation for both sweep directions."""
    fb = load_npz("fibers.npz")
    spec = configs.CONFIGS[2]
    m = configs.make_model(2)
    o = P.PhiGridOracle(m, spec.grid)
    n = spec.grid.points_per_axis
    for layout, k in ((0, 2), (1, 2)):
        pre = f"c2_k{k}_l{layout}"
        left = [tuple(t) for t in fb[pre + "_left"]]
        right = [tuple(t) for t in fb[pre + "_right"]]
        block, rows, cols = P.cross.sample_block(o, left, n, right, axis_first=(layout == 1))
        assert block.shape == (len(rows), len(cols))
        want = o(np.array([r + c for r in rows[:3] for c in cols]))
        np.testing.assert_allclose(block[:3].ravel(), want, rtol=1e-13)
        tall = block if layout == 0 else block.T
        ref_rows = fb[pre + "_phi_rows"]
        np.testing.assert_allclose(tall[ref_rows], fb[pre + "_phi_vals"], rtol=1e-12)
