"""Generate the golden fixtures in this directory from the REFERENCE package.

Run in the build container (the reference is importable there, not on the
GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [--cfg2-dense]

Everything is produced by calling the reference's public API
(``/root/reference/pkg/src/ttpricer``) on seeded inputs; nothing here is
product code.  The committed .npz/.json files are what the tests compare
against, on the CPU (oracle pinning) and on the GPU (parity).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import ttpricer as ref  # noqa: E402

from paper_2203_02804_b200 import configs  # noqa: E402


def ref_model(cid, inst=0):
    kw = configs.model_kwargs(configs.make_model(cid, inst))
    return ref.MarketModel(**kw)


def ref_grid(cid):
    g = configs.CONFIGS[cid].grid
    return ref.GridSpec(n=g.n, eta=g.eta, alpha=g.alpha, d=g.d)


def random_tt(rng, phys, bond, scale=1.0):
    d = len(phys)
    bonds = [1] + [bond] * (d - 1) + [1]
    cores = []
    for k in range(d):
        shape = (bonds[k], phys[k], bonds[k + 1])
        cores.append(scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)))
    return ref.TensorTrain(cores)


def flat_cores(tt):
    return np.concatenate([c.ravel() for c in tt.cores])


def sets_to_json(sets):
    return [None if s is None else [list(t) for t in s] for s in sets]


def report_to_json(rep):
    d = rep.to_dict()
    d["left_sets"] = sets_to_json(rep.left_sets)
    d["right_sets"] = sets_to_json(rep.right_sets)
    return d


def gen_evaluators(out):
    data = {}
    for cid in range(1, 6):
        model = ref_model(cid)
        grid = ref_grid(cid)
        rng = np.random.default_rng(1000 + cid)
        idx = rng.integers(0, grid.points_per_axis, size=(2000, grid.d))
        # include the grid corners (largest phases / moduli)
        idx[0] = 0
        idx[1] = grid.n
        idx[2] = grid.n // 2
        phi = ref.phi_grid_oracle(model, grid)(idx)
        vhat = ref.payoff_grid_oracle(model, grid)(idx)
        data[f"c{cid}_idx"] = idx
        data[f"c{cid}_phi"] = phi
        data[f"c{cid}_vhat_conj"] = vhat
    np.savez_compressed(os.path.join(out, "evaluators.npz"), **data)


def gen_contractions(out):
    data = {}
    cases = [((5, 5, 5), 4, 7), ((4, 3, 5), 3, 11), ((6, 6, 6, 6), 5, 23),
             ((33, 33, 33), 10, 5), ((9,) * 6, 8, 3), ((3,), 1, 1)]
    meta = []
    for q, (phys, bond, seed) in enumerate(cases):
        rng = np.random.default_rng(seed)
        a = random_tt(rng, phys, bond)
        b = random_tt(rng, phys, bond)
        idx = np.column_stack([rng.integers(0, n, 300) for n in phys])
        data[f"t{q}_a"] = flat_cores(a)
        data[f"t{q}_b"] = flat_cores(b)
        data[f"t{q}_inner"] = np.array([ref.tt_inner(a, b), ref.tt_inner(b, a), ref.tt_inner(a, a)])
        data[f"t{q}_idx"] = idx
        data[f"t{q}_eval"] = ref.tt_evaluate_many(a, idx)
        w = [rng.standard_normal(n) + 1j * rng.standard_normal(n) for n in phys]

        def sep(ix, w=w):
            o = np.ones(len(ix), dtype=complex)
            for axis, wa in enumerate(w):
                o *= wa[ix[:, axis]]
            return o

        data[f"t{q}_sepw"] = np.concatenate(w)
        data[f"t{q}_diff"] = np.array([ref.tt_rand_sample_diff(a, sep, 5000, 17),
                                       ref.tt_rand_sample_diff(a, lambda ix, a=a: ref.tt_evaluate_many(a, ix), 700, 3)])
        meta.append({"phys": list(phys), "bond": bond, "seed": seed})
    np.savez_compressed(os.path.join(out, "contractions.npz"), **data)
    return meta


def gen_dense(out):
    res = {}
    bench = dict(r=0.3, sigma=0.5, T=1.0, s0=100.0, strike=100.0)
    m1 = ref.MarketModel(d=1, **bench)
    for n in (30, 50):
        g = ref.GridSpec(n=n, eta=0.5, alpha=3.0, d=1)
        res[f"d1_n{n}"] = ref.price_fourier_dense(m1, g).price
    res["bs_bench"] = ref.black_scholes_price(m1)
    m2 = ref.MarketModel.with_plus_correlation(d=2, beta=0.5, **bench)
    g2 = ref.GridSpec(n=50, eta=0.5, alpha=2.5, d=2)
    res["d2_bench"] = ref.price_fourier_dense(m2, g2).price
    res["d2_bench_t025"] = ref.price_fourier_dense(m2, g2, t=0.25).price
    m3 = ref.MarketModel.with_plus_correlation(d=3, beta=0.5, **bench)
    g3 = ref.GridSpec(n=50, eta=0.4, alpha=5.0 / 3, d=3)
    res["d3_bench"] = ref.price_fourier_dense(m3, g3).price
    res["cfg1"] = ref.price_fourier_dense(ref_model(1), ref_grid(1)).price
    # a few cfg3-style instances on a coarser d=5 grid (fast on the CPU)
    g5 = ref.GridSpec(n=16, eta=0.3, alpha=1.0, d=5)
    res["cfg3_n16"] = [ref.price_fourier_dense(ref_model(3, i), g5).price for i in range(4)]
    return res


def gen_maxvol(out):
    data = {}
    rng = np.random.default_rng(4)
    shapes = [(8, 2), (12, 3), (24, 5), (48, 8), (64, 8), (97, 8), (120, 9), (330, 10),
              (1300, 20), (4128, 32)]
    for q, (n, r) in enumerate(shapes):
        m = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
        data[f"m{q}"] = m
        data[f"m{q}_sel"] = ref.maxvol(m, slack=0.01)
    np.savez_compressed(os.path.join(out, "maxvol.npz"), **data)


def gen_cross(out):
    data = {}
    res = {}
    # rank-1 separable (test_cross.py:123-131 style)
    rng = np.random.default_rng(10)
    w = [rng.standard_normal(6) + 1j * rng.standard_normal(6) for _ in range(3)]

    def sep(ix):
        o = np.ones(len(ix), dtype=complex)
        for axis, wa in enumerate(w):
            o *= wa[ix[:, axis]]
        return o

    cfg = ref.CrossConfig(bond_dim=1, eps_tol=1e-10, n_conv_samples=2000, seed=0)
    tt, rep = ref.tt_cross(sep, (6, 6, 6), cfg)
    data["sep_w"] = np.concatenate(w)
    data["sep_cores"] = flat_cores(tt)
    res["sep"] = report_to_json(rep)
    # self-reconstruction of a random rank-4 train
    target = random_tt(np.random.default_rng(12), (8, 8, 8, 8), 4)
    cfg = ref.CrossConfig(bond_dim=4, eps_tol=1e-8, n_conv_samples=5000, seed=3)
    tt, rep = ref.tt_cross(lambda ix: ref.tt_evaluate_many(target, ix), (8, 8, 8, 8), cfg)
    data["selfrec_target"] = flat_cores(target)
    data["selfrec_cores"] = flat_cores(tt)
    res["selfrec"] = report_to_json(rep)
    # characteristic-function oracles on bench grids
    bench = dict(r=0.3, sigma=0.5, T=1.0, s0=100.0, strike=100.0)
    for d, bond, seed, beta in ((2, 6, 7, 0.5), (3, 10, 101, 0.5), (3, 4, 17, 1.0)):
        model = ref.MarketModel.with_plus_correlation(d=d, beta=beta, **bench)
        eta = ref.table1_hyperparams(d)[0]
        g = ref.GridSpec(n=50, eta=eta, alpha=5.0 / d, d=d)
        cfg = ref.CrossConfig(bond_dim=bond, seed=seed, n_conv_samples=2000)
        tt, rep = ref.tt_cross(ref.phi_grid_oracle(model, g), (51,) * d, cfg)
        key = f"phi_d{d}_D{bond}_s{seed}"
        data[key + "_cores"] = flat_cores(tt)
        res[key] = report_to_json(rep)
    np.savez_compressed(os.path.join(out, "cross.npz"), **data)
    return res


def gen_prices(out, cids):
    data = {}
    res = {}
    for cid in cids:
        spec = configs.CONFIGS[cid]
        n_inst = 1 if cid in (1, 2, 4) else 4
        for inst in range(n_inst):
            model = ref_model(cid, inst)
            grid = ref_grid(cid)
            cfg = ref.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
            t0 = time.perf_counter()
            phi_tt, rep_phi = ref.tt_cross(ref.phi_grid_oracle(model, grid), (grid.points_per_axis,) * grid.d, cfg)
            v_tt, rep_v = ref.tt_cross(ref.payoff_grid_oracle(model, grid), (grid.points_per_axis,) * grid.d, cfg)
            raw = ref.tt_inner(v_tt, phi_tt)
            wall = time.perf_counter() - t0
            pref = np.exp(-model.r * model.T) * grid.eta ** grid.d / (2 * np.pi) ** grid.d
            key = f"cfg{cid}_i{inst}"
            res[key] = {
                "price": float((pref * raw).real),
                "raw": [raw.real, raw.imag],
                "wall_s": wall,
                "cross_phi": report_to_json(rep_phi),
                "cross_v": report_to_json(rep_v),
            }
            if cid in (1, 2) and inst == 0:
                data[key + "_phi"] = flat_cores(phi_tt)
                data[key + "_v"] = flat_cores(v_tt)
            print(f"{key}: price {res[key]['price']:.12g} in {wall:.1f}s", flush=True)
    np.savez_compressed(os.path.join(out, "prices_cores.npz"), **data)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg2-dense", action="store_true", help="also run the 13-minute cfg2 dense sum")
    ap.add_argument("--skip-prices", action="store_true")
    args = ap.parse_args()
    out = HERE
    summary = {"reference": "ttpricer " + ref.__version__, "numpy": np.__version__,
               "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}
    gen_evaluators(out)
    summary["contractions"] = gen_contractions(out)
    summary["dense"] = gen_dense(out)
    gen_maxvol(out)
    summary["cross"] = gen_cross(out)
    if not args.skip_prices:
        summary["prices"] = gen_prices(out, (1, 2, 3, 4))
    if args.cfg2_dense:
        t0 = time.perf_counter()
        summary["dense"]["cfg2"] = ref.price_fourier_dense(ref_model(2), ref_grid(2), term_cap=2_000_000_000).price
        summary["dense"]["cfg2_wall_s"] = time.perf_counter() - t0
    else:
        old = os.path.join(out, "golden.json")
        if os.path.exists(old):
            prev = json.load(open(old))
            if "cfg2" in prev.get("dense", {}):
                summary["dense"]["cfg2"] = prev["dense"]["cfg2"]
                summary["dense"]["cfg2_wall_s"] = prev["dense"].get("cfg2_wall_s")
    with open(os.path.join(out, "golden.json"), "w") as fh:
        json.dump(summary, fh, indent=1, default=float)


if __name__ == "__main__":
    main()
