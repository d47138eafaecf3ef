import json
import os
import sys

# Golden fixtures were generated with one BLAS thread; the CPU oracle is only
# bitwise equal to them under the same setting.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402
import pytest  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

# pytest plugins may import numpy before this file runs, so the environment
# variables above can be too late; pin the BLAS pool at runtime as well.
_BLAS_LIMIT = threadpool_limits(limits=1, user_api="blas")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def unflat_cores(flat, phys, bonds):
    """Split packed row-major cores (make_golden.flat_cores) into arrays."""
    out, off = [], 0
    for k, n in enumerate(phys):
        size = bonds[k] * n * bonds[k + 1]
        out.append(np.asarray(flat[off:off + size]).reshape(bonds[k], n, bonds[k + 1]))
        off += size
    assert off == len(flat)
    return out


def uniform_bonds(d, bond):
    return [1] + [bond] * (d - 1) + [1]


def sets_as_lists(sets):
    return [None if s is None else [list(map(int, t)) for t in s] for s in sets]


BENCH = dict(r=0.3, sigma=0.5, T=1.0, s0=100.0, strike=100.0)
