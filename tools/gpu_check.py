"""Quick GPU parity probe against the committed reference fixtures (dev tool)."""
import json
import os
import sys
import time
import traceback

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_2203_02804_b200 as P  # noqa: E402
from paper_2203_02804_b200 import configs  # noqa: E402

G = os.path.join(REPO, "tests", "golden")
gold = json.load(open(os.path.join(G, "golden.json")))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def unflat(flat, phys, bond):
    d = len(phys)
    bonds = [1] + [bond] * (d - 1) + [1]
    out, off = [], 0
    for k in range(d):
        sz = bonds[k] * phys[k] * bonds[k + 1]
        out.append(flat[off:off + sz].reshape(bonds[k], phys[k], bonds[k + 1]))
        off += sz
    return P.TensorTrain(out)


def section(name, fn):
    t0 = time.time()
    try:
        fn()
        print(f"[ok] {name} ({time.time() - t0:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def evaluators():
    ev = np.load(os.path.join(G, "evaluators.npz"))
    for cid in range(1, 6):
        m = configs.make_model(cid)
        g = configs.CONFIGS[cid].grid
        idx = ev[f"c{cid}_idx"]
        phi = P.PhiGridOracle(m, g)(idx)
        vh = P.PayoffGridOracle(m, g)(idx)
        print(f"   cfg{cid}: phi rel {rel(phi, ev[f'c{cid}_phi']):.2e}  vhat rel {rel(vh, ev[f'c{cid}_vhat_conj']):.2e}")


def contractions():
    ct = np.load(os.path.join(G, "contractions.npz"))
    for q, meta in enumerate(gold["contractions"]):
        a = unflat(ct[f"t{q}_a"], meta["phys"], meta["bond"])
        b = unflat(ct[f"t{q}_b"], meta["phys"], meta["bond"])
        inner = np.array([P.tt_inner(a, b), P.tt_inner(b, a), P.tt_inner(a, a)])
        ev = P.tt_evaluate_many(a, ct[f"t{q}_idx"])
        phys = meta["phys"]
        w = ct[f"t{q}_sepw"]
        ws, off = [], 0
        for n in phys:
            ws.append(w[off:off + n])
            off += n
        d1 = P.tt_rand_sample_diff(a, P.SeparableOracle(ws), 5000, 17)
        d2 = P.tt_rand_sample_diff(a, P.TTOracle(a), 700, 3)
        print(f"   case {q} {phys} D={meta['bond']}: inner {rel(inner, ct[f't{q}_inner']):.2e} "
              f"eval {rel(ev, ct[f't{q}_eval']):.2e} diff {d1:.6g}/{ct[f't{q}_diff'][0]:.6g} {d2}/{ct[f't{q}_diff'][1]}")


def dense():
    bench = dict(r=0.3, sigma=0.5, T=1.0, s0=100.0, strike=100.0)
    m1 = P.MarketModel(d=1, **bench)
    for n in (30, 50):
        g = P.GridSpec(n=n, eta=0.5, alpha=3.0, d=1)
        v = P.price_fourier_dense(m1, g).price
        print(f"   d1 n{n}: {v!r} vs {gold['dense'][f'd1_n{n}']!r} rel {rel(v, gold['dense'][f'd1_n{n}']):.2e}")
    m2 = P.MarketModel.with_plus_correlation(d=2, beta=0.5, **bench)
    g2 = P.GridSpec(n=50, eta=0.5, alpha=2.5, d=2)
    v = P.price_fourier_dense(m2, g2).price
    print(f"   d2: rel {rel(v, gold['dense']['d2_bench']):.2e}")
    v = P.price_fourier_dense(configs.make_model(1), configs.CONFIGS[1].grid).price
    print(f"   cfg1: rel {rel(v, gold['dense']['cfg1']):.2e}")
    g5 = P.GridSpec(n=16, eta=0.3, alpha=1.0, d=5)
    vs = [r.price for r in P.price_fourier_dense_batch([configs.make_model(3, i) for i in range(4)], g5)]
    print(f"   cfg3 n16 batch: rel {rel(vs, gold['dense']['cfg3_n16']):.2e}")
    if "cfg2" in gold["dense"]:
        t0 = time.time()
        v = P.price_fourier_dense(configs.make_model(2), configs.CONFIGS[2].grid, term_cap=2_000_000_000).price
        print(f"   cfg2 dense: rel {rel(v, gold['dense']['cfg2']):.2e} in {time.time() - t0:.3f}s")


def maxvol():
    mv = np.load(os.path.join(G, "maxvol.npz"))
    q = 0
    while f"m{q}" in mv:
        m = mv[f"m{q}"]
        sel = P.maxvol(m, slack=0.01)
        same = np.array_equal(sel, mv[f"m{q}_sel"])
        b = m @ np.linalg.inv(m[sel])
        print(f"   {m.shape}: same={same} dominance {np.abs(b).max():.4f}")
        q += 1


def cross():
    cr = np.load(os.path.join(G, "cross.npz"))
    w = cr["sep_w"]
    ws = [w[0:6], w[6:12], w[12:18]]
    tt, rep = P.tt_cross(P.SeparableOracle(ws), (6, 6, 6),
                         P.CrossConfig(bond_dim=1, eps_tol=1e-10, n_conv_samples=2000, seed=0))
    g = gold["cross"]["sep"]
    print(f"   sep: {rep.to_dict()} ref {dict((k, g[k]) for k in rep.to_dict())}")
    print(f"   sep sets equal: {[list(map(list, s)) if s else s for s in rep.left_sets] == g['left_sets']}")
    target = unflat(cr["selfrec_target"], (8, 8, 8, 8), 4)
    tt, rep = P.tt_cross(P.TTOracle(target), (8, 8, 8, 8),
                         P.CrossConfig(bond_dim=4, eps_tol=1e-8, n_conv_samples=5000, seed=3))
    g = gold["cross"]["selfrec"]
    print(f"   selfrec: {rep.to_dict()}\n      ref {dict((k, g[k]) for k in rep.to_dict())}")
    bench = dict(r=0.3, sigma=0.5, T=1.0, s0=100.0, strike=100.0)
    for d, bond, seed, beta in ((2, 6, 7, 0.5), (3, 10, 101, 0.5), (3, 4, 17, 1.0)):
        model = P.MarketModel.with_plus_correlation(d=d, beta=beta, **bench)
        eta = P.table1_hyperparams(d)[0]
        grid = P.GridSpec(n=50, eta=eta, alpha=5.0 / d, d=d)
        tt, rep = P.tt_cross(P.phi_grid_oracle(model, grid), (51,) * d,
                             P.CrossConfig(bond_dim=bond, seed=seed, n_conv_samples=2000))
        key = f"phi_d{d}_D{bond}_s{seed}"
        g = gold["cross"][key]
        lsame = [None if s is None else [list(t) for t in s] for s in rep.left_sets] == g["left_sets"]
        rsame = [None if s is None else [list(t) for t in s] for s in rep.right_sets] == g["right_sets"]
        print(f"   {key}: {rep.to_dict()}\n      ref {dict((k, g[k]) for k in rep.to_dict())} sets L={lsame} R={rsame}")


def prices():
    for cid in (1, 2, 3, 4):
        spec = configs.CONFIGS[cid]
        n_inst = 1 if cid in (1, 2, 4) else 4
        models = [configs.make_model(cid, i) for i in range(n_inst)]
        cfg = P.CrossConfig(bond_dim=spec.bond_dim, seed=spec.cross_seed)
        t0 = time.time()
        res = P.price_fourier_tt_batch(models, spec.grid, cfg, cfg)
        wall = time.time() - t0
        for i, r in enumerate(res):
            g = gold["prices"][f"cfg{cid}_i{i}"]
            same_l = [None if s is None else [list(t) for t in s] for s in r.diagnostics["cross_phi"].left_sets] == g["cross_phi"]["left_sets"]
            print(f"   cfg{cid} i{i}: price {r.price:.12g} ref {g['price']:.12g} rel {rel(r.price, g['price']):.2e} "
                  f"sweeps {r.diagnostics['cross_phi'].sweeps_used}/{r.diagnostics['cross_v'].sweeps_used} "
                  f"ref {g['cross_phi']['sweeps_used']}/{g['cross_v']['sweeps_used']} phiL={same_l} "
                  f"diff {r.diagnostics['cross_phi'].final_diff:.3e}/{g['cross_phi']['final_diff']:.3e}")
        print(f"   cfg{cid}: {n_inst} options in {wall:.3f}s")


if __name__ == "__main__":
    which = sys.argv[1:] or ["evaluators", "contractions", "dense", "maxvol", "cross", "prices"]
    for name in which:
        section(name, globals()[name])
