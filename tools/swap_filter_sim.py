"""Replay of the oracle's cfg4 maxvol swap runs with per-row bounds on max|B|
(dev tool for the filtered swap passes).  Usage:
python tools/swap_filter_sim.py INSTANCE FLUSH {warp|cta} K -- prints the
fraction of rows a filtered pass must read in full when the threshold is the
warp's (or CTA's) max over the new pivot column and its top-K entries of
the previous pass."""
import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
from oracle import ttp_oracle as O
from paper_2203_02804_b200 import configs
calls = []
orig = O.swaps
def rec(q, start, slack, max_iters):
    calls.append((q.copy(), np.asarray(start).copy(), slack))
    return orig(q, start, slack, max_iters)
O.swaps = rec
sp = configs.CONFIGS[4]
m = configs.make_model(4, int(sys.argv[1]) if len(sys.argv) > 1 else 0)
g = sp.grid
gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, g.n, g.eta, g.alpha)
O.price_tt(gm, sp.bond_dim, sp.bond_dim, sp.cross_seed, sp.cross_seed)
MODE = sys.argv[3]; K = int(sys.argv[4]); prevtop = []
F = int(sys.argv[2]) if len(sys.argv) > 2 else 4
C, CT = 2, 256
stats = {"full": 0, "filt": 0, "filt_rows": 0, "rows": 0}
for q, start, slack in calls:
    mrows, r = q.shape
    if mrows < 1000: continue
    ms = (mrows + C - 1) // C
    # warp id of each row
    gl = np.arange(mrows); cta = gl // ms; l = gl - cta * ms
    wid = cta * 8 + (l % CT) // 32
    rows = start.copy()
    b = np.linalg.solve(q[rows].T, q.T).T
    np_ = 0; valid = False
    bound = None
    for it in range(10 * mrows):
        a = np.abs(b)
        i, j = np.unravel_index(np.argmax(a), b.shape)
        piv = b[i, j]
        if abs(piv) <= 1.0 + slack: break
        w = (b[rows[j], :] - b[i, :]) / piv
        cvec = b[:, j].copy()
        b += np.outer(b[:, j], b[rows[j], :] - b[i, :]) / piv
        rows[j] = i
        nq = np_ + 1
        flush = nq >= F
        a = np.abs(b)
        if flush or not valid:
            stats["full"] += 1; bound = a.max(1); valid = True
        else:
            bound = bound + np.abs(cvec) * np.abs(w).max()
            colj = a[:, j]
            Tw = np.full(wid.max() + 1, 0.0); np.maximum.at(Tw, wid, colj)
            for (kk, ll, ww) in prevtop:
                Tw[ww] = max(Tw[ww], a[kk, ll])
            if MODE == "cta":
                Tc = np.zeros(C)
                for ww in range(len(Tw)): Tc[ww // 8] = max(Tc[ww // 8], Tw[ww])
                Tw = np.array([Tc[ww // 8] for ww in range(len(Tw))])
            cand = ~(bound < Tw[wid])
            stats["filt"] += 1; stats["filt_rows"] += cand.sum(); stats["rows"] += mrows
            bound[cand] = a[cand].max(1)
        np_ = 0 if flush else nq
        # each warp's top-K entries among this pass's values (exact)
        prevtop = []
        for ww in range(wid.max() + 1):
            rr = np.nonzero(wid == ww)[0]
            sub = a[rr]
            flat = np.argsort(-sub.ravel(), kind="stable")[:K]
            for f in flat:
                prevtop.append((rr[f // r], f % r, ww))
        if (it + 1) % 64 == 0:
            b = np.linalg.solve(q[rows].T, q.T).T; valid = False; np_ = 0
print(stats, "filtered row fraction", stats["filt_rows"] / max(1, stats["rows"]))
