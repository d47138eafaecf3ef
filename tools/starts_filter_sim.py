"""Replay of the maxvol starts (QRCP of Q^H and LU of Q, cross.py:172-177) on
the oracle's cfg4 Q matrices, with per-row bounds (dev tool, DESIGN.md
section 5).  Prints, per bond, the fraction of rows a bound-filtered start
round must read in full (the QRCP side: stale norms are upper bounds; the
LU side: Cauchy-Schwarz |s_gk| <= ||q_g[:k+1]|| ||(-w_k, 1)||) and the
fraction of Q entries either side reads.  Usage:
python tools/starts_filter_sim.py [INSTANCE]"""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle import ttp_oracle as O
from paper_2203_02804_b200 import configs

qs = []
orig = O.dominant_rows


def rec(q, slack, max_iters):
    qs.append(q.copy())
    return orig(q, slack, max_iters)


O.dominant_rows = rec
sp = configs.CONFIGS[4]
m = configs.make_model(4, int(sys.argv[1]) if len(sys.argv) > 1 else 0)
g = sp.grid
gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, g.n, g.eta, g.alpha)
O.price_tt(gm, sp.bond_dim, sp.bond_dim, sp.cross_seed, sp.cross_seed)

C, CT, W = 2, 256, 8
GROUP = len(sys.argv) > 2 and sys.argv[2] == 'group'
tot = {"q_eval": 0, "lu_eval": 0, "rows": 0, "bytes_now": 0, "bytes_filt": 0}
for q in qs:
    n, r = q.shape
    if n < 1000:
        continue
    ms = (n + C - 1) // C
    gl = np.arange(n)
    cta = gl // ms
    wid = cta * W + ((gl - cta * ms) % CT) // 32
    # ---- QRCP of Q^H: greedy residual norms (exact), stale bounds
    E = np.zeros((r, r), complex)  # orthonormal basis of the chosen rows
    norm2 = np.sum(np.abs(q) ** 2, 1)
    exact = norm2.copy()
    bound = norm2.copy()
    chosen = np.zeros(n, bool)
    prevbest = {}
    # ---- LU with partial pivoting (|Re|+|Im|)
    A = q.copy()
    luchosen = np.zeros(n, bool)
    pref2 = np.cumsum(np.abs(q) ** 2, 1)  # ||q_g[:k+1]||^2
    Minv = None
    q_eval = lu_eval = 0
    bytes_now = bytes_filt = 0
    Ls = np.zeros((n, 0), complex)
    for k in range(r):
        # QRCP round k: exact residual norms after k reflectors
        if k > 0:
            proj = q.conj() @ E[:, k - 1]
            exact = np.maximum(exact - np.abs(proj) ** 2, 0.0)
        cand = ~chosen
        # threshold per warp: the previous round's warp winner re-evaluated
        T = np.zeros(wid.max() + 1)
        for w, row in prevbest.items():
            if cand[row]:
                T[w] = exact[row]
        need = cand & (bound >= T[wid])
        grp = gl // 32  # 32 consecutive rows = one warp's row group of a pass
        gneed = np.zeros(grp.max() + 1, bool)
        np.logical_or.at(gneed, grp, need)
        need = cand & gneed[grp] if GROUP else need
        bound[need] = exact[need]
        # QRCP winner (exact argmax over candidates)
        v = np.where(cand, exact, -1)
        p = int(np.argmax(v))
        for w in range(wid.max() + 1):
            sel = cand & (wid == w)
            if sel.any():
                ii = np.where(sel)[0]
                prevbest[w] = int(ii[np.argmax(exact[ii])])
        q_eval += int(need.sum())
        # new orthonormal direction from row p
        x = q[p].conj().copy()
        x -= E[:, :k] @ (E[:, :k].conj().T @ x)
        E[:, k] = x / np.linalg.norm(x)
        chosen[p] = True
        # LU round k: Schur column k
        s = A[:, k]
        luc = ~luchosen
        wk = np.linalg.norm(Minv[:, k]) if Minv is not None else 0.0
        lub = np.sqrt(2.0) * np.sqrt(pref2[:, k]) * np.sqrt(1.0 + wk ** 2)
        mag = np.abs(s.real) + np.abs(s.imag)
        TL = np.zeros(wid.max() + 1)
        np.maximum.at(TL, wid[luc], np.where(luc, mag, 0)[luc] * 0)  # placeholder
        need_lu = luc.copy()  # LU: Cauchy-Schwarz bound vs the warp max (oracle threshold)
        TLw = np.zeros(wid.max() + 1)
        np.maximum.at(TLw, wid[luc], mag[luc])
        need_lu = luc & (lub >= TLw[wid])
        lu_eval += int(need_lu.sum())
        pl = int(np.argmax(np.where(luc, mag, -1)))
        piv = A[pl, k]
        l = A[:, k] / piv
        l[luchosen] = 0
        l[pl] = 0
        A = A - np.outer(l, A[pl])
        luchosen[pl] = True
        # M_k for the bound: U_k^-1 U[:k+1, :]
        U = q[np.where(luchosen)[0]]
        Minv = np.linalg.lstsq(U[:, : k + 1], U, rcond=None)[0] if k + 1 < r else None
        # bytes: now every candidate row reads r entries; filtered: QRCP-needed rows r, others k+1
        bytes_now += int((cand | luc).sum()) * r
        need_any = need
        bytes_filt += int(need_any.sum()) * r + int((~need_any & (cand | luc)).sum()) * (k + 1)
    tot["q_eval"] += q_eval
    tot["lu_eval"] += lu_eval
    tot["rows"] += n * r
    tot["bytes_now"] += bytes_now
    tot["bytes_filt"] += bytes_filt
    print(f"bond {n}x{r}: QRCP rows evaluated {q_eval / (n * r):.3f}, LU (C-S bound) {lu_eval / (n * r):.3f}, "
          f"entries read {bytes_filt / bytes_now:.3f} of now")
print(f"total: QRCP {tot['q_eval'] / tot['rows']:.3f}  LU {tot['lu_eval'] / tot['rows']:.3f}  "
      f"entries {tot['bytes_filt'] / tot['bytes_now']:.3f}")
