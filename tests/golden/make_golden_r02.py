"""Round-2 golden fixtures, generated from the REFERENCE package (test
infrastructure; run in the build container, where /root/reference is
importable -- the GPU box only reads the committed outputs):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_r02.py [fibers] [prices] [tt32] [json]

fibers  -> fibers.npz: sampled unfolding blocks of phi(-z) and conj(vhat(z))
           built by the reference's own ``_block`` (cross.py:310-332) with one
           oracle call each, for BASELINE configs 1-5, left-to-right and
           right-to-left layouts, edge and middle bonds.  Index sets are
           seeded random tuples of the right lengths and counts; up to 256
           rows of each tall matrix are kept (cfg5 blocks are 16 MB).
prices  -> ref_prices_r02.json: the reference's price_fourier_tt
           (pricers.py:256-294) on cfg4 instances 0-15 and cfg2/cfg3
           instances 0-3 / 0-7, one process per option, one BLAS thread.
tt32    -> tt32_cross.json (+ tt32_target.npy): the reference's tt_cross
           (cross.py:358-453) of a seeded rank-32 tensor train on (129,)^10
           -- the benchmark's block shapes (4128 x 32), numerically full rank
           -- with both sweep directions forced (eps_tol tiny, 2 sweeps).
json    -> ref_tt.json written by the reference's tt_save_json
           (tensor_train.py:228-245); asserts the reference's tt_load_json
           reads the repo's writer's output back exactly.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
import time
from concurrent.futures import ProcessPoolExecutor

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import ttpricer as ref  # noqa: E402
from ttpricer import cross as ref_cross  # noqa: E402

from paper_2203_02804_b200 import configs  # noqa: E402

KEEP_ROWS = 256


def ref_model(cid, inst=0):
    return ref.MarketModel(**configs.model_kwargs(configs.make_model(cid, inst)))


def ref_grid(cid):
    g = configs.CONFIGS[cid].grid
    return ref.GridSpec(n=g.n, eta=g.eta, alpha=g.alpha, d=g.d)


def rank_at(shape, bond, k):
    return min(bond, int(np.prod(shape[:k], dtype=object)), int(np.prod(shape[k:], dtype=object)))


def gen_fibers():
    data = {}
    cases = []
    for cid in range(1, 6):
        spec = configs.CONFIGS[cid]
        d, n = spec.d, spec.grid.points_per_axis
        shape = (n,) * d
        model, grid = ref_model(cid), ref_grid(cid)
        mid = d // 2
        # (bond k, layout): layout 0 = left-to-right (axis k-1), 1 = right-to-left (axis k)
        for k, layout in sorted({(1, 0), (mid, 0), (mid, 1), (d - 1, 1)}):
            axis = k - 1 if layout == 0 else k
            nl = rank_at(shape, spec.bond_dim, axis)
            nr = rank_at(shape, spec.bond_dim, axis + 1)
            rng = np.random.default_rng([cid, k, layout])
            left = [tuple(int(v) for v in row) for row in rng.integers(0, n, size=(nl, axis))]
            right = [tuple(int(v) for v in row) for row in rng.integers(0, n, size=(nr, d - axis - 1))]
            for kind, oracle in (("phi", ref.phi_grid_oracle(model, grid)),
                                 ("vhat", ref.payoff_grid_oracle(model, grid))):
                counter = ref_cross._CallCounter(oracle, None)
                block, _, _ = ref_cross._block(counter, left, n, right, axis_first=(layout == 1))
                tall = block if layout == 0 else block.T   # the matrix _interp_core factorizes
                keep = np.sort(rng.choice(tall.shape[0], size=min(KEEP_ROWS, tall.shape[0]), replace=False))
                key = f"c{cid}_k{k}_l{layout}_{kind}"
                data[key + "_rows"] = keep.astype(np.int32)
                data[key + "_vals"] = tall[keep]
                data[key + "_calls"] = np.array([counter.construction])
            data[f"c{cid}_k{k}_l{layout}_left"] = np.asarray(left, dtype=np.int32).reshape(nl, axis)
            data[f"c{cid}_k{k}_l{layout}_right"] = np.asarray(right, dtype=np.int32).reshape(nr, d - axis - 1)
            cases.append([cid, k, layout])
            print(f"fibers cfg{cid} bond {k} layout {layout}: {nl}x{n}x{nr}", flush=True)
    data["cases"] = np.asarray(cases, dtype=np.int32)
    np.savez_compressed(os.path.join(HERE, "fibers.npz"), **data)


def _price(job):
    cid, inst = job
    spec = configs.CONFIGS[cid]
    model, grid = ref_model(cid, inst), ref_grid(cid)
    cfg = ref.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
    t0 = time.perf_counter()
    res = ref.price_fourier_tt(model, grid, cfg, cfg, dense_reference="never")
    rp, rv = res.diagnostics["cross_phi"], res.diagnostics["cross_v"]
    return job, {"price": res.price, "wall_s": time.perf_counter() - t0,
                 "imag_part": res.diagnostics["imag_part"],
                 "cross_phi": {"oracle_calls": rp.oracle_calls, "sweeps_used": rp.sweeps_used,
                               "converged": rp.converged, "final_diff": rp.final_diff},
                 "cross_v": {"oracle_calls": rv.oracle_calls, "sweeps_used": rv.sweeps_used,
                             "converged": rv.converged, "final_diff": rv.final_diff}}


def gen_prices():
    jobs = [(4, i) for i in range(16)] + [(2, i) for i in range(4)] + [(3, i) for i in range(8)]
    out = {}
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        for (cid, inst), rec in ex.map(_price, jobs):
            out[f"cfg{cid}_i{inst}"] = rec
            print(f"cfg{cid} i{inst}: {rec['price']!r} ({rec['wall_s']:.1f} s)", flush=True)
    out["generator"] = "tests/golden/make_golden_r02.py prices: ttpricer.price_fourier_tt(dense_reference='never'), 1 BLAS thread"
    with open(os.path.join(HERE, "ref_prices_r02.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def gen_prices5():
    """Config 5 (d=20, 257 points, D=64): the reference needs ~10 minutes per
    option on one core; instances 0-7 (SURVEY.md 8(d)'s subset rule) ->
    ref_prices_cfg5.json."""
    jobs = [(5, i) for i in range(8)]
    out = {}
    with ProcessPoolExecutor(max_workers=min(8, os.cpu_count())) as ex:
        for (cid, inst), rec in ex.map(_price, jobs):
            out[f"cfg{cid}_i{inst}"] = rec
            print(f"cfg{cid} i{inst}: {rec['price']!r} ({rec['wall_s']:.1f} s)", flush=True)
    out["generator"] = "tests/golden/make_golden_r02.py prices5: ttpricer.price_fourier_tt(dense_reference='never'), 1 BLAS thread"
    with open(os.path.join(HERE, "ref_prices_cfg5.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def tt32_target():
    """Seeded rank-32 train on (129,)^10, cores scaled so entries stay O(1)."""
    rng = np.random.default_rng(2032)
    d, n, D = 10, 129, 32
    bonds = [1] + [D] * (d - 1) + [1]
    cores = []
    for k in range(d):
        shp = (bonds[k], n, bonds[k + 1])
        cores.append((rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / np.sqrt(2.0 * bonds[k]))
    return cores


def gen_tt32():
    cores = tt32_target()
    target = ref.TensorTrain(cores)

    def oracle(idx):  # chunked: tt_evaluate_many gathers (D, m, D) per site
        return np.concatenate([ref.tt_evaluate_many(target, idx[i:i + 16384])
                               for i in range(0, len(idx), 16384)])

    cfg = ref.CrossConfig(bond_dim=32, eps_tol=1e-300, max_sweeps=2, n_conv_samples=20000, seed=77)
    t0 = time.perf_counter()
    tt, rep = ref.tt_cross(oracle, (129,) * 10, cfg)
    wall = time.perf_counter() - t0
    sets = lambda s: [None if x is None else [list(map(int, t)) for t in x] for x in s]  # noqa: E731
    out = {"target_seed": 2032, "shape": [129] * 10, "bond_dim": 32,
           "cfg": {"bond_dim": 32, "eps_tol": 1e-300, "max_sweeps": 2, "n_conv_samples": 20000, "seed": 77},
           "wall_s": wall, "report": {k: v for k, v in rep.to_dict().items()},
           "left_sets": sets(rep.left_sets), "right_sets": sets(rep.right_sets),
           "inner_self": [complex(ref.tt_inner(tt, tt)).real, complex(ref.tt_inner(tt, tt)).imag]}
    print(f"tt32 cross: {wall:.1f} s, sweeps {rep.sweeps_used}, diff {rep.final_diff:.3e}", flush=True)
    with open(os.path.join(HERE, "tt32_cross.json"), "w") as fh:
        json.dump(out, fh)


def gen_json():
    from paper_2203_02804_b200.tensor_train import TensorTrain, tt_save_json
    rng = np.random.default_rng(515)
    bonds = [1, 3, 4, 2, 1]
    phys = [5, 2, 6, 3]
    cores = [rng.standard_normal((bonds[k], phys[k], bonds[k + 1]))
             + 1j * rng.standard_normal((bonds[k], phys[k], bonds[k + 1])) for k in range(4)]
    ref.tt_save_json(ref.TensorTrain(cores), os.path.join(HERE, "ref_tt.json"))
    np.save(os.path.join(HERE, "ref_tt_cores.npy"), np.concatenate([c.ravel() for c in cores]))
    # the reference reads the repo's container back exactly
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "repo.json")
        tt_save_json(TensorTrain(cores), path)
        back = ref.tt_load_json(path)
        for a, b in zip(back.cores, cores):
            assert np.array_equal(a, b)
        assert open(path).read() == open(os.path.join(HERE, "ref_tt.json")).read()
    print("json: reference reads the repo container exactly; files are byte-identical")


if __name__ == "__main__":
    what = sys.argv[1:] or ["fibers", "prices", "tt32", "json"]
    for w in what:
        globals()[f"gen_{w}"]()
