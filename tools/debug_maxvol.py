"""Device maxvol on the golden matrices vs the reference selections (dev tool)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2203_02804_b200 as P  # noqa: E402
mv = np.load("tests/golden/maxvol.npz")
q = 0
while f"m{q}" in mv:
    got = P.maxvol(mv[f"m{q}"], slack=0.01)
    print(q, mv[f"m{q}"].shape, np.array_equal(got, mv[f"m{q}_sel"]), got, mv[f"m{q}_sel"])
    q += 1
