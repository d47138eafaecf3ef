"""Device start sets (TTP_DEBUG_START=1|2) vs scipy's on the golden matrices (dev tool)."""
import os
import sys
import numpy as np
import scipy.linalg as sl
sys.path.insert(0, ".")
import paper_2203_02804_b200 as P  # noqa: E402
which = int(os.environ.get("TTP_DEBUG_START", "1"))
mv = np.load("tests/golden/maxvol.npz")
for q in range(9):
    A = mv[f"m{q}"]
    Q = sl.qr(A, mode="economic", pivoting=True)[0]
    m, r = Q.shape
    if which == 1:
        want = np.sort(sl.qr(Q.conj().T, mode="economic", pivoting=True)[2][:r])
    else:
        want = np.sort(np.argsort(sl.lu(Q, p_indices=True)[0])[:r])
    got = P.maxvol(A, slack=0.01)
    print(q, A.shape, np.array_equal(np.sort(got), want), np.sort(got), want)
