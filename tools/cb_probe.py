"""Dev probe of ttp_column_basis: orthonormality, span and pivot agreement
with the pinned oracle's scipy QR on one graded random matrix."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2203_02804_b200 as P
from oracle import ttp_oracle as O

m, r = int(os.environ.get("M", 4128)), int(os.environ.get("R", 32))
rng = np.random.default_rng([m, r])
scales = np.exp(rng.uniform(-3.0, 3.0, size=r))
a = (rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r))) / np.sqrt(2.0) * scales
q = P.column_basis(a)
qref = O.column_basis(a, 0.0)
orth = np.max(np.abs(q.conj().T @ q - np.eye(r)))
res = np.linalg.norm(a - q @ (q.conj().T @ a), axis=0) / np.linalg.norm(a, axis=0)
ov = np.abs(np.einsum("ij,ij->j", q.conj(), qref))
print(f"m={m} r={r} orth {orth:.2e}; span residual per column max {res.max():.2e} (cols>1e-10: {np.nonzero(res > 1e-10)[0].tolist()})")
print("diag overlap with reference Q:", np.round(ov, 6).tolist())
blk = np.abs(q.conj().T @ qref)
print("overlap matrix argmax per dev column:", blk.argmax(axis=1).tolist())
# which rows of Q are wrong: compare projections of A rows
rowres = np.linalg.norm((a - q @ (q.conj().T @ a)), axis=1) / np.linalg.norm(a, axis=1)
bad = np.nonzero(rowres > 1e-8)[0]
print(f"rows with bad span: {len(bad)}; first/last {bad[:5].tolist()} {bad[-5:].tolist()}")
