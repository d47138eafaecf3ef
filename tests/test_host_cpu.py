"""Host-side logic and the C-ABI boundary, on the CPU (no kernel launches)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
from oracle import ttp_oracle as O
from paper_2203_02804_b200 import (
    CrossConfig,
    DeviceError,
    GridSpec,
    MarketModel,
    PhiGridOracle,
    PayoffGridOracle,
    SeparableOracle,
    TensorTrain,
    configs,
    tt_cross,
    tt_load_json,
    tt_save_json,
)
from paper_2203_02804_b200 import _lib
from paper_2203_02804_b200.cross import _Layout, initial_right_sets, rank_profile
from paper_2203_02804_b200.tensor_train import sample_indices

HEADER = os.path.join(REPO, "include", "ttpricer_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|void|size_t|const char\*)\s+(ttp_\w+)\s*\(",
                                 text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    names = declared_symbols()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(names) == bound
    assert lib.ttp_abi_version() == 1


def test_library_is_sm100a_only():
    so = os.path.join(REPO, "paper_2203_02804_b200", _lib.LIB_NAME)
    data = open(so, "rb").read()
    assert b"sm_100a" in data


def test_struct_sizes_match_header_layout():
    # sanity on ctypes mirrors of the C structs (natural alignment, x86-64)
    assert ctypes.sizeof(_lib.Oracle) == 56
    assert ctypes.sizeof(_lib.CrossCfg) == 40
    assert ctypes.sizeof(_lib.CrossLayout) == 4 * 65 + 4 + 8 * 65 + 8 + 8 * 65 + 8 + 8 + 4 + 4


@pytest.mark.parametrize("shape,bond", [((33,) * 3, 10), ((65,) * 5, 20), ((129,) * 10, 32),
                                        ((257,) * 20, 64), ((6, 6, 6), 1), ((8, 8, 8, 8), 4),
                                        ((5, 3, 9), 7), ((7,), 3)])
def test_layout_ranks_match_reference_rule(shape, bond):
    lay = _Layout(shape, bond)
    want = rank_profile(shape, bond)
    assert lay.ranks == want
    if len(shape) > 1:
        assert want == O.rank_profile(shape, bond)
    sizes = [want[k] * shape[k] * want[k + 1] for k in range(len(shape))]
    assert lay.core_offsets == list(np.concatenate([[0], np.cumsum(sizes)]))


@pytest.mark.parametrize("cid", [1, 2, 4, 5])
def test_initial_right_sets_bitwise(cid):
    spec = configs.CONFIGS[cid]
    shape = (spec.grid.points_per_axis,) * spec.d
    ranks = rank_profile(shape, spec.bond_dim)
    ours = initial_right_sets(shape, ranks, spec.cross_seed)
    ref = O.initial_right(shape, ranks, spec.cross_seed)
    for k in range(1, spec.d):
        np.testing.assert_array_equal(ours[k], ref[k])


def test_initial_right_sets_match_reference_fixture(golden):
    # the reference's right sets after a single L2R sweep are the initial draw
    rep = golden["prices"]["cfg4_i0"]["cross_phi"]
    assert rep["sweeps_used"] == 1
    shape = (129,) * 10
    ours = initial_right_sets(shape, rank_profile(shape, 32), 1244)
    for k in range(1, 10):
        assert [list(map(int, t)) for t in ours[k]] == rep["right_sets"][k]


def test_conv_samples_bitwise():
    a = sample_indices((129,) * 10, 50_000, 1244)
    b = O.draw_samples((129,) * 10, 50_000, 1244)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_model_arrays_bitwise(cid):
    m = configs.make_model(cid, 0)
    mu, cov = O.model_arrays(m.sigma, m.corr, m.T, m.s0, m.rates)
    np.testing.assert_array_equal(m.log_drift, mu)
    np.testing.assert_array_equal(m.log_cov, cov)


def test_oracle_descriptor_packing():
    m = configs.make_model(2, 0)
    g = configs.CONFIGS[2].grid
    p = PhiGridOracle(m, g).params()
    assert p[0] == g.eta and p[1] == g.alpha and p[2] == g.n // 2
    np.testing.assert_array_equal(p[3:8], m.log_drift)
    np.testing.assert_array_equal(p[8:].reshape(5, 5), m.log_cov)
    v = PayoffGridOracle(m, g).params()
    assert list(v) == [g.eta, g.alpha, g.n // 2, m.strike, 1.0]
    s = SeparableOracle([np.ones(3), np.arange(4)])
    assert list(s.table_offsets()) == [0, 3, 7]


def test_python_callables_are_rejected():
    with pytest.raises(TypeError, match="device oracle"):
        tt_cross(lambda idx: np.ones(len(idx)), (4, 4), CrossConfig(bond_dim=2))


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only check")
def test_no_cpu_fallback_without_device():
    m = configs.make_model(1, 0)
    g = configs.CONFIGS[1].grid
    from paper_2203_02804_b200 import price_fourier_tt
    with pytest.raises(DeviceError):
        price_fourier_tt(m, g, CrossConfig(bond_dim=4), CrossConfig(bond_dim=4))


def test_config_validation():
    for kw in (dict(bond_dim=0), dict(bond_dim=2, eps_tol=0.0), dict(bond_dim=2, max_sweeps=0),
               dict(bond_dim=2, n_conv_samples=0), dict(bond_dim=2, maxvol_slack=-0.1),
               dict(bond_dim=2, oracle_call_budget=0)):
        with pytest.raises(ValueError):
            CrossConfig(**kw)
    for kw in (dict(n=3, eta=0.5, alpha=1.0, d=1), dict(n=0, eta=0.5, alpha=1.0, d=1),
               dict(n=10, eta=-0.5, alpha=1.0, d=1)):
        with pytest.raises(ValueError):
            GridSpec(**kw)
    with pytest.raises(ValueError):
        MarketModel(r=0.1, sigma=[0.2, 0.2], T=1.0, s0=100.0, strike=100.0,
                    corr=np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_status_mapping():
    from paper_2203_02804_b200.errors import (CapacityError, MaxvolIterationError,
                                              OracleBudgetError, SingularMatrixError)
    for st, exc in ((_lib.TTP_ERR_SINGULAR, SingularMatrixError),
                    (_lib.TTP_ERR_MAXVOL_ITER, MaxvolIterationError),
                    (_lib.TTP_ERR_BUDGET, OracleBudgetError),
                    (_lib.TTP_ERR_CAPACITY, CapacityError),
                    (_lib.TTP_ERR_INVALID, ValueError),
                    (_lib.TTP_ERR_CUDA, DeviceError)):
        with pytest.raises(exc):
            _lib.raise_for(st, "ctx", bond=3)


def test_json_container_roundtrip(tmp_path):
    rng = np.random.default_rng(47)
    cores = [rng.standard_normal(s) + 1j * rng.standard_normal(s) for s in ((1, 4, 3), (3, 3, 3), (3, 5, 1))]
    tt = TensorTrain(cores)
    path = tmp_path / "t.json"
    tt_save_json(tt, path)
    back = tt_load_json(path)
    for a, b in zip(tt.cores, back.cores):
        np.testing.assert_array_equal(a, b)


def test_json_interchange_with_reference(tmp_path):
    """a container written by the REFERENCE's tt_save_json
    (tests/golden/ref_tt.json, tensor_train.py:228-245) loads into the same
    cores here, and this package's writer produces byte-identical files (the
    generator, make_golden_r02.py json, also reads the repo's output back
    with the reference's tt_load_json)."""
    import os
    from conftest import GOLDEN
    want = np.load(os.path.join(GOLDEN, "ref_tt_cores.npy"))
    back = tt_load_json(os.path.join(GOLDEN, "ref_tt.json"))
    np.testing.assert_array_equal(np.concatenate([c.ravel() for c in back.cores]), want)
    assert back.phys_dims == (5, 2, 6, 3) and back.bond_dims == (1, 3, 4, 2, 1)
    path = tmp_path / "repo.json"
    tt_save_json(back, path)
    assert path.read_text() == open(os.path.join(GOLDEN, "ref_tt.json")).read()


def test_tensor_train_container_rules():
    with pytest.raises(ValueError, match="bond mismatch"):
        TensorTrain([np.zeros((1, 2, 3)), np.zeros((4, 2, 1))])
    with pytest.raises(ValueError, match="boundary"):
        TensorTrain([np.zeros((2, 3, 1))])
    tt = TensorTrain([np.ones((1, 3, 2)), np.ones((2, 4, 1))])
    assert tt.bond_dims == (1, 2, 1) and tt.n_entries == 12
    with pytest.raises(ValueError):
        tt.cores[0][0, 0, 0] = 1.0


def test_balanced_chunks_are_equal_and_fit():
    """The batch API's chunking: the fewest chunks that respect the memory
    limit, of equal size (never a short last chunk)."""
    from paper_2203_02804_b200.pricers import balanced_chunk
    assert balanced_chunk(148, 122) == 74          # config 5 on one B200: 74 + 74, not 122 + 26
    assert balanced_chunk(4096, 1585) == 1366      # config 3: three equal chunks
    assert balanced_chunk(592, 592) == 592 and balanced_chunk(592, 5000) == 592
    assert balanced_chunk(5, 1) == 1 and balanced_chunk(1, 10) == 1
    for n in (1, 7, 100, 1023, 4096):
        for limit in (1, 3, 64, 999, 5000):
            c = balanced_chunk(n, limit)
            k = -(-n // c)
            assert 1 <= c <= max(limit, 1) and k == -(-n // min(limit, n))
            assert k * c - n < k                   # chunk sizes differ by at most one
