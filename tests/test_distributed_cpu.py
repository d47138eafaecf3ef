"""Multi-rank sharding + result gather, world_size 2 over gloo on the CPU.

The GPU path is identical except for the backend (nccl) and the tensors'
device: each rank prices its contiguous shard, then one all-gather of the
per-option records.  Here each rank "prices" its shard with the CPU oracle's
dense sum on a tiny grid so the gathered values can be checked exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2203_02804_b200.distributed import RECORD_FIELDS, gather_records, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dense_value(i):
    from oracle import ttp_oracle as O
    from paper_2203_02804_b200 import configs
    m = configs.make_model(3, i)
    gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, 4, 0.3, 1.0)
    return O.price_dense(gm)


def _worker(rank, world, port, n_total, out_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(n_total, rank, world)
    local = np.zeros((hi - lo, len(RECORD_FIELDS)))
    for j, i in enumerate(range(lo, hi)):
        local[j, 0] = _dense_value(i)
        local[j, 2] = rank
    full = gather_records(local, n_total)
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [5, 8])
def test_gloo_world2_gather(tmp_path, n_total):
    out = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), n_total, out), nprocs=2, join=True)
    full = np.load(out)
    assert full.shape == (n_total, len(RECORD_FIELDS))
    want = np.array([_dense_value(i) for i in range(n_total)])
    np.testing.assert_array_equal(full[:, 0], want)
    owners = [0] * (n_total // 2) + [1] * (n_total - n_total // 2)
    np.testing.assert_array_equal(full[:, 2], owners)


def test_shard_ranges_partition():
    for n in (0, 1, 7, 1024, 4096):
        for w in (1, 2, 4, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _oracle_range_sum(model, grid, first, count):
    """CPU stand-in for ttp_dense_sum_range: the oracle's terms over a flat range."""
    from oracle import ttp_oracle as O
    gm = O.GridModel(model.r, model.sigma, model.T, model.s0, model.strike, model.corr, grid.n,
                     grid.eta, grid.alpha)
    n = grid.points_per_axis
    flat = np.arange(first, first + count)
    idx = np.stack(np.unravel_index(flat, (n,) * grid.d), axis=1)
    return complex(np.sum(gm.phi_oracle()(idx) * np.conj(gm.vhat_oracle()(idx))))


def _dense_worker(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2203_02804_b200 import configs
    from paper_2203_02804_b200.distributed import dense_contour_sum_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = configs.CONFIGS[1]
    m = configs.make_model(1)
    total = dense_contour_sum_sharded(m, spec.grid, partial_fn=_oracle_range_sum)
    np.save(out_path + f".{rank}.npy", np.array([total]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_dense_sum(tmp_path):
    """the dense cross-check split by flat index range over two
    ranks combines (in rank order, identically on both ranks) to the full sum."""
    from paper_2203_02804_b200 import configs
    out = str(tmp_path / "dense")
    mp.spawn(_dense_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r0, r1 = np.load(out + ".0.npy")[0], np.load(out + ".1.npy")[0]
    assert r0 == r1
    spec = configs.CONFIGS[1]
    full = _oracle_range_sum(configs.make_model(1), spec.grid, 0, spec.grid.n_terms)
    assert abs(r0 - full) <= 1e-12 * abs(full)


def _split2_worker(rank, world, port, out_path):
    import torch.distributed as dist
    from oracle import ttp_oracle as O
    from paper_2203_02804_b200 import CrossConfig, TensorTrain, configs
    from paper_2203_02804_b200.distributed import price_fourier_tt_split2
    from paper_2203_02804_b200.oracles import PhiGridOracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def cross_fn(o, shape, cfg):  # CPU restatement in place of the device cross
        m, g = o.model, o.grid
        gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, g.n, g.eta, g.alpha)
        f = gm.phi_oracle() if isinstance(o, PhiGridOracle) else gm.vhat_oracle()
        cores, _ = O.tt_cross(f, shape, cfg.bond_dim, n_conv=cfg.n_conv_samples, seed=cfg.seed)
        return TensorTrain(cores)

    def inner_fn(bra, ket):
        return O.tt_inner(list(bra.cores), list(ket.cores))

    spec = configs.CONFIGS[1]
    cfg = CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed, n_conv_samples=2000)
    p = price_fourier_tt_split2(configs.make_model(1), spec.grid, cfg, cfg, cross_fn=cross_fn, inner_fn=inner_fn)
    np.save(out_path + f".{rank}.npy", np.array([p]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_split_crosses():
    """SURVEY 8(e) optional split: phi on rank 0, vhat on rank 1, cores sent
    point-to-point, contraction on rank 0, price broadcast; equals the
    one-process pipeline on the same CPU restatement."""
    import tempfile
    from oracle import ttp_oracle as O
    from paper_2203_02804_b200 import configs
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "split")
        mp.spawn(_split2_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        p0, p1 = np.load(out + ".0.npy")[0], np.load(out + ".1.npy")[0]
    assert p0 == p1
    spec = configs.CONFIGS[1]
    m = configs.make_model(1)
    gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, spec.grid.n, spec.grid.eta, spec.grid.alpha)
    want, _ = O.price_tt(gm, spec.bond_dim, spec.bond_dim, spec.cross_seed, spec.cross_seed, n_conv=2000)
    assert p0 == pytest.approx(want, rel=1e-13)


def _cpu_pricer(models, grid, cfg_phi, cfg_v, t=0.0, raise_errors=True):
    """CPU stand-in for the device batch pricer (same signature and result
    shape as price_fourier_tt_batch): the pinned restatement per option; a
    strike of 77 raises OracleBudgetError to exercise the error path."""
    from oracle import ttp_oracle as O
    from paper_2203_02804_b200 import CrossReport, OracleBudgetError, PricingResult
    out = []
    for m in models:
        if m.strike == 77.0:
            out.append(OracleBudgetError("injected budget failure"))
            continue
        gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, grid.n, grid.eta, grid.alpha)
        price, info = O.price_tt(gm, cfg_phi.bond_dim, cfg_v.bond_dim, cfg_phi.seed, cfg_v.seed, t=t,
                                 n_conv=cfg_phi.n_conv_samples)

        def rep(r, cfg):
            return CrossReport(converged=bool(r["converged"]), sweeps_used=int(r["sweeps_used"]),
                               oracle_calls=int(r["oracle_calls"]), conv_check_calls=int(r["conv_check_calls"]),
                               final_diff=float(r["final_diff"]),
                               compression_ratio=int(r["oracle_calls"]) / grid.n_terms)
        value = gm.prefactor(t) * info["raw"]
        out.append(PricingResult(price, "fourier_tt", 0.0, {
            "cross_phi": rep(info["cross_phi"], cfg_phi), "cross_v": rep(info["cross_v"], cfg_v),
            "imag_part": float(value.imag), "oracle_calls_total": 0}))
    if raise_errors:
        for r in out:
            if isinstance(r, Exception):
                raise r
    return out


def _models_cfg1(n, bad=None):
    from paper_2203_02804_b200 import MarketModel, configs
    out = []
    for i in range(n):
        m = configs.make_model(3, i)
        if i == bad:
            m = MarketModel(r=m.r, sigma=m.sigma, T=m.T, s0=m.s0, strike=77.0, corr=m.corr, d=m.d)
        out.append(m)
    return out


def _sharded_worker(rank, world, port, out_path, n, bad):
    import pickle
    import torch.distributed as dist
    from paper_2203_02804_b200 import CrossConfig, GridSpec
    from paper_2203_02804_b200.distributed import price_batch_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid = GridSpec(n=8, eta=0.3, alpha=1.0, d=5)
    cfg = CrossConfig(bond_dim=4, seed=1239, n_conv_samples=500)
    models = _models_cfg1(n, bad)
    res = {"rank": rank}
    try:
        out = price_batch_sharded(models, grid, cfg, cfg, group=dist.group.WORLD, local_pricer=_cpu_pricer)
        res["prices"] = [r.price for r in out]
        res["owners"] = [r.diagnostics.get("rank", rank) for r in out]
        res["reports"] = [r.diagnostics["cross_phi"].to_dict() for r in out]
    except Exception as exc:  # noqa: BLE001 - recorded for the assertion
        res["error"] = type(exc).__name__
    with open(out_path + f".{rank}.pkl", "wb") as fh:
        pickle.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [5, 6])
def test_gloo_world2_sharded_batch_api(tmp_path, n):
    """price_fourier_tt_batch(..., group=...) -> distributed.price_batch_sharded:
    both ranks get the whole batch in input order, identical prices, each
    option priced by its contiguous owner; the gathered records rebuild the
    reports' counters exactly."""
    import pickle
    from paper_2203_02804_b200 import CrossConfig, GridSpec
    out = str(tmp_path / "sh")
    mp.spawn(_sharded_worker, args=(2, _free_port(), out, n, None), nprocs=2, join=True)
    r0, r1 = (pickle.load(open(out + f".{r}.pkl", "rb")) for r in (0, 1))
    assert "error" not in r0 and "error" not in r1
    assert r0["prices"] == r1["prices"] and r0["reports"] == r1["reports"]
    assert r0["owners"] == r1["owners"] == [0] * (n // 2) + [1] * (n - n // 2)
    grid = GridSpec(n=8, eta=0.3, alpha=1.0, d=5)
    cfg = CrossConfig(bond_dim=4, seed=1239, n_conv_samples=500)
    want = _cpu_pricer(_models_cfg1(n), grid, cfg, cfg)
    assert r0["prices"] == [w.price for w in want]
    assert r0["reports"] == [w.diagnostics["cross_phi"].to_dict() for w in want]


def test_gloo_world2_sharded_batch_error_raises_on_every_rank(tmp_path):
    """An option failing on rank 1 is raised on BOTH ranks (same class) after
    the one collective -- no rank is left blocked in the all-gather."""
    import pickle
    out = str(tmp_path / "err")
    mp.spawn(_sharded_worker, args=(2, _free_port(), out, 6, 4), nprocs=2, join=True)
    r0, r1 = (pickle.load(open(out + f".{r}.pkl", "rb")) for r in (0, 1))
    assert r0["error"] == r1["error"] == "OracleBudgetError"


def _split2_err_worker(rank, world, port, out_path):
    import pickle
    import torch.distributed as dist
    from paper_2203_02804_b200 import CrossConfig, SingularMatrixError, configs
    from paper_2203_02804_b200.distributed import price_fourier_tt_split2
    from paper_2203_02804_b200.oracles import PhiGridOracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def cross_fn(o, shape, cfg):
        if not isinstance(o, PhiGridOracle):
            raise SingularMatrixError("injected", bond=2)
        from paper_2203_02804_b200 import TensorTrain
        return TensorTrain([np.ones((1, n, 1), complex) for n in shape])

    spec = configs.CONFIGS[1]
    cfg = CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed, n_conv_samples=2000)
    res = {}
    try:
        price_fourier_tt_split2(configs.make_model(1), spec.grid, cfg, cfg, cross_fn=cross_fn,
                                inner_fn=lambda a, b: 1.0)
    except Exception as exc:  # noqa: BLE001
        res["error"] = type(exc).__name__
    with open(out_path + f".{rank}.pkl", "wb") as fh:
        pickle.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_split_crosses_error_does_not_hang(tmp_path):
    """If the vhat cross raises on rank 1, rank 0 raises too instead of
    waiting forever for the cores (status word exchanged first)."""
    import pickle
    out = str(tmp_path / "s2e")
    mp.spawn(_split2_err_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r0, r1 = (pickle.load(open(out + f".{r}.pkl", "rb")) for r in (0, 1))
    assert r0["error"] == r1["error"] == "SingularMatrixError"
