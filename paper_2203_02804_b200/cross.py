"""TT-cross and maxvol on the GPU (reference cross.py).

The host keeps what must be bit-exact with the reference and is O(d*D)
work: the seeded draws of the initial right index sets (cross.py:296-307,
402-403) and of the convergence samples (tensor_train.py:191-194), both with
numpy's Generator.  Everything else -- fibers, column bases, maxvol,
interpolation factors, the convergence check -- runs in the native sweep
driver of ``libttpricer_b200.so`` (``ttp_cross_run``), batched over
independent instances.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import MaxvolIterationError, OracleBudgetError, SingularMatrixError
from .oracles import OracleBatch, check_device_oracle
from .tensor_train import DeviceTTBatch, TensorTrain, sample_indices

__all__ = ["CrossConfig", "CrossReport", "maxvol", "tt_cross", "tt_cross_batch", "CrossBatchResult",
           "sample_block"]

COND_LIMIT = 1e12
RANK_TOL = 1e-12
MAX_BOND = 64


@dataclass(frozen=True)
class CrossConfig:
    """Controls for one TT-cross run (same fields/defaults as cross.py:40-70)."""

    bond_dim: int
    eps_tol: float = 0.005
    max_sweeps: int = 4
    n_conv_samples: int = 50_000
    seed: int = 0
    maxvol_slack: float = 0.01
    oracle_call_budget: int | None = None

    def __post_init__(self):
        if self.bond_dim < 1:
            raise ValueError("bond_dim must be >= 1")
        if self.eps_tol <= 0:
            raise ValueError("eps_tol must be > 0")
        if self.max_sweeps < 1:
            raise ValueError("max_sweeps must be >= 1")
        if self.n_conv_samples < 1:
            raise ValueError("n_conv_samples must be >= 1")
        if self.maxvol_slack < 0:
            raise ValueError("maxvol_slack must be >= 0")
        if self.oracle_call_budget is not None and self.oracle_call_budget < 1:
            raise ValueError("oracle_call_budget must be >= 1 when set")


class CrossReport:
    """Outcome record of a TT-cross run (cross.py:73-100).

    Same fields and equality as the reference dataclass (the pivot sets are
    excluded from comparison).  The pivot sets of a batched run are decoded
    from the device arrays only when first accessed.
    """

    _FIELDS = ("converged", "sweeps_used", "oracle_calls", "conv_check_calls", "final_diff",
               "compression_ratio")

    def __init__(self, converged, sweeps_used, oracle_calls, conv_check_calls, final_diff,
                 compression_ratio, left_sets=None, right_sets=None):
        self.converged = converged
        self.sweeps_used = sweeps_used
        self.oracle_calls = oracle_calls
        self.conv_check_calls = conv_check_calls
        self.final_diff = final_diff
        self.compression_ratio = compression_ratio
        self._left = left_sets
        self._right = right_sets

    @property
    def left_sets(self):
        if callable(self._left):
            self._left = self._left()
        return self._left

    @left_sets.setter
    def left_sets(self, value):
        self._left = value

    @property
    def right_sets(self):
        if callable(self._right):
            self._right = self._right()
        return self._right

    @right_sets.setter
    def right_sets(self, value):
        self._right = value

    def __eq__(self, other):
        if not isinstance(other, CrossReport):
            return NotImplemented
        return all(getattr(self, f) == getattr(other, f) for f in self._FIELDS)

    def __repr__(self):
        inner = ", ".join(f"{f}={getattr(self, f)!r}" for f in self._FIELDS)
        return f"CrossReport({inner})"

    def to_dict(self):
        return {
            "converged": self.converged,
            "sweeps_used": self.sweeps_used,
            "oracle_calls": self.oracle_calls,
            "conv_check_calls": self.conv_check_calls,
            "final_diff": self.final_diff,
            "compression_ratio": self.compression_ratio,
        }


def sample_block(oracle, left, axis_size, right, axis_first):
    """One bond's sampled unfolding on the GPU -- the reference's ``_block``
    (cross.py:310-332): rows ``left x axis`` and columns ``right`` when
    ``axis_first`` is False (left-to-right sweep), rows ``left`` and columns
    ``axis x right`` when True.  Returns ``(block, row_tuples, col_tuples)``
    in the reference's orientation.  The values come from ttp_eval_fibers,
    i.e. the separable evaluation the bond kernels fill their blocks with."""
    o = check_device_oracle(oracle)
    left = [tuple(int(v) for v in t) for t in left]
    right = [tuple(int(v) for v in t) for t in right]
    axis = len(left[0])
    if len(right[0]) != o.d - axis - 1 or any(len(t) != axis for t in left):
        raise ValueError("left/right tuples do not span the oracle's dimension")
    shape = list(o.shape) if o.shape is not None else [int(axis_size)] * o.d
    shape[axis] = int(axis_size)
    tall = OracleBatch([o]).fiber_blocks(left, right, axis, shape, 1 if axis_first else 0)[0]
    if axis_first:
        return tall.T, left, [(s,) + b for s in range(axis_size) for b in right]
    return tall, [a + (s,) for a in left for s in range(axis_size)], right


def rank_profile(shape, bond_dim):
    """r_k = min(D, prod(shape[:k]), prod(shape[k:])), k = 0..d (cross.py:397-400)."""
    d = len(shape)
    if d == 1:
        return [1, 1]
    return [min(bond_dim, math.prod(shape[:k]), math.prod(shape[k:])) for k in range(d + 1)]


def initial_right_sets(shape, ranks, seed):
    """Nested random right sets with the reference's exact RNG call sequence."""
    d = len(shape)
    rng = np.random.default_rng(seed)
    right = [None] * (d + 1)
    right[d] = np.zeros((1, 0), dtype=np.int64)
    for k in range(d - 1, 0, -1):
        tail = right[k + 1]
        n_cand = shape[k] * len(tail)
        want = min(ranks[k], n_cand)
        pick = np.sort(rng.choice(n_cand, size=want, replace=False))
        s, b = np.divmod(pick, len(tail))
        right[k] = np.column_stack([s, tail[b]]).astype(np.int64)
    return right


class _Layout:
    def __init__(self, shape, bond_dim):
        lib = _lib.load_library()
        self.d = len(shape)
        self.shape = np.asarray(shape, dtype=np.int32)
        lay = _lib.CrossLayout()
        st = lib.ttp_cross_layout_of(self.d, self.shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                     bond_dim, ctypes.byref(lay))
        _lib.raise_for(st, "cross layout")
        d = self.d
        self.ranks = [int(lay.ranks[k]) for k in range(d + 1)]
        self.core_offsets = [int(lay.core_offsets[k]) for k in range(d + 1)]
        self.core_stride = int(lay.core_stride)
        self.set_offsets = [int(lay.set_offsets[k]) for k in range(d + 1)]
        self.set_stride = int(lay.set_stride)

    def pack_sets(self, sets):
        buf = np.zeros(self.set_stride, dtype=np.int32)
        for k, rows in enumerate(sets):
            if rows is None or rows.shape[1] == 0:
                continue
            blk = np.zeros((rows.shape[0], self.d), dtype=np.int32)
            blk[:, : rows.shape[1]] = rows
            buf[self.set_offsets[k]: self.set_offsets[k] + blk.size] = blk.ravel()
        return buf

    def unpack_set(self, buf, k, length):
        r = self.ranks[k]
        blk = buf[self.set_offsets[k]: self.set_offsets[k] + r * self.d].reshape(r, self.d)
        return [tuple(int(v) for v in row[:length]) for row in blk]


class _ConvSamples:
    """Seeded convergence samples and their per-site buckets, cached per key."""

    _cache = {}

    def __init__(self, shape, m, seed):
        torch = _lib.require_device()
        idx = sample_indices(shape, m, seed)
        perms, offs = [], []
        for k, n in enumerate(shape):
            col = idx[:, k]
            perms.append(np.argsort(col, kind="stable").astype(np.int32))
            counts = np.bincount(col, minlength=n)
            offs.append(np.concatenate([[0], np.cumsum(counts)]).astype(np.int32))
        dev = torch.device("cuda")
        self.idx = torch.from_numpy(idx.astype(np.int32)).to(dev)
        self.perm = torch.from_numpy(np.concatenate(perms)).to(dev)
        self.off = torch.from_numpy(np.concatenate(offs)).to(dev)

    @classmethod
    def get(cls, shape, m, seed):
        # the tensors live on the device that was current when they were made
        torch = _lib.require_device()
        key = (tuple(shape), int(m), seed, torch.cuda.current_device())
        if key not in cls._cache:
            if len(cls._cache) > 8:
                cls._cache.clear()
            cls._cache[key] = cls(shape, m, seed)
        return cls._cache[key]


@dataclass
class CrossBatchResult:
    """Device-resident result of a batched cross."""

    trains: DeviceTTBatch
    reports: list
    status: np.ndarray
    error_bond: np.ndarray
    counters: dict = None

    def error_for(self, i):
        return _status_error(int(self.status[i]), int(self.error_bond[i]))


def _status_error(status, bond):
    if status == _lib.TTP_OK:
        return None
    if status == _lib.TTP_ERR_SINGULAR:
        return SingularMatrixError(f"singular cross block at bond {bond}", bond=bond)
    if status == _lib.TTP_ERR_MAXVOL_ITER:
        return MaxvolIterationError("maxvol did not settle within the row-swap guard")
    if status == _lib.TTP_ERR_BUDGET:
        return OracleBudgetError("oracle budget exceeded")
    return RuntimeError(f"cross failed with status {status}")


def cross_bytes_per_instance(shape, cfg):
    """Device bytes one instance of tt_cross_batch needs (workspace + cores +
    index sets), from the library's own workspace rule (ttp_cross_workspace)."""
    lib = _lib.load_library()
    shape = tuple(int(n) for n in shape)
    d = len(shape)
    lay = _Layout(shape, min(cfg.bond_dim, MAX_BOND))

    def ws(n):
        prob = _lib.CrossProblem(
            d=d, n_inst=n, h_shape=lay.shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            cfg=_lib.CrossCfg(bond_dim=cfg.bond_dim if d > 1 else 1, max_sweeps=cfg.max_sweeps,
                              eps_tol=cfg.eps_tol, n_conv_samples=cfg.n_conv_samples,
                              maxvol_slack=cfg.maxvol_slack, oracle_call_budget=-1))
        return lib.ttp_cross_workspace(ctypes.byref(prob))

    return (ws(2) - ws(1)) + 16 * lay.core_stride + 8 * lay.set_stride


class _PreparedCross:
    """Problem + output buffers of one batched cross (shared by tt_cross_batch
    and the one-call pricer); keeps every buffer the C structs point at alive."""


def _prepare_cross(oracles, shape, cfg):
    torch = _lib.require_device()
    lib = _lib.load_library()
    shape = tuple(int(n) for n in shape)
    if len(shape) < 1 or min(shape) < 1:
        raise ValueError(f"invalid shape {shape}")
    if cfg.bond_dim > MAX_BOND and len(shape) > 1:
        raise ValueError(f"bond_dim {cfg.bond_dim} above the device limit {MAX_BOND}")
    batch = oracles if isinstance(oracles, OracleBatch) else OracleBatch(list(oracles))
    if batch.d != len(shape):
        raise ValueError(f"oracle has d={batch.d} but shape has {len(shape)} axes")
    d, n = len(shape), batch.n_inst
    lay = _Layout(shape, min(cfg.bond_dim, MAX_BOND))
    ranks = lay.ranks
    right0 = initial_right_sets(shape, ranks, cfg.seed) if d > 1 else [None, np.zeros((1, 0), np.int64)]
    dev = torch.device("cuda")
    d_right_init = torch.from_numpy(lay.pack_sets(right0)).to(dev)
    conv = _ConvSamples.get(shape, cfg.n_conv_samples, cfg.seed)
    d_shape = torch.tensor(shape, dtype=torch.int32, device=dev)
    prob = _lib.CrossProblem(
        d=d,
        n_inst=n,
        h_shape=lay.shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        d_shape=d_shape.data_ptr(),
        oracle=batch.struct,
        cfg=_lib.CrossCfg(
            bond_dim=cfg.bond_dim if d > 1 else 1,
            max_sweeps=cfg.max_sweeps,
            eps_tol=cfg.eps_tol,
            n_conv_samples=cfg.n_conv_samples,
            maxvol_slack=cfg.maxvol_slack,
            oracle_call_budget=-1 if cfg.oracle_call_budget is None else cfg.oracle_call_budget,
        ),
        d_right_init=d_right_init.data_ptr(),
        d_conv_idx=conv.idx.data_ptr(),
        d_conv_perm=conv.perm.data_ptr(),
        d_conv_off=conv.off.data_ptr(),
    )
    if d == 1:
        prob.cfg.bond_dim = 1
    cores = torch.zeros(n * lay.core_stride, dtype=torch.complex128, device=dev)
    left = torch.zeros(n * lay.set_stride, dtype=torch.int32, device=dev)
    right = torch.zeros(n * lay.set_stride, dtype=torch.int32, device=dev)
    h = {
        "status": np.zeros(n, np.int32), "bond": np.zeros(n, np.int32),
        "conv": np.zeros(n, np.int32), "sweeps": np.zeros(n, np.int32),
        "lvalid": np.zeros(n * (d + 1), np.int32), "calls": np.zeros(n, np.int64),
        "ccalls": np.zeros(n, np.int64), "diff": np.zeros(n, np.float64),
    }
    P32, P64, PF = (ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                    ctypes.POINTER(ctypes.c_double))
    out = _lib.CrossOut(
        d_cores=cores.data_ptr(), d_left=left.data_ptr(), d_right=right.data_ptr(),
        h_status=h["status"].ctypes.data_as(P32), h_error_bond=h["bond"].ctypes.data_as(P32),
        h_converged=h["conv"].ctypes.data_as(P32), h_sweeps=h["sweeps"].ctypes.data_as(P32),
        h_left_valid=h["lvalid"].ctypes.data_as(P32), h_oracle_calls=h["calls"].ctypes.data_as(P64),
        h_conv_calls=h["ccalls"].ctypes.data_as(P64), h_final_diff=h["diff"].ctypes.data_as(PF),
    )
    pc = _PreparedCross()
    pc.__dict__.update(prob=prob, out=out, lay=lay, shape=shape, ranks=ranks, cores=cores, left=left,
                       right=right, h=h, n=n, d=d,
                       keep=(batch, d_right_init, conv, d_shape, lay, h))
    return pc

class _LazyHost:
    """A device tensor copied to a host array on first use (then cached)."""

    def __init__(self, t, shape):
        self._t, self._shape, self._a = t, shape, None
        self._lock = threading.Lock()

    def get(self):
        with self._lock:
            if self._a is None:
                self._a = self._t.cpu().numpy().reshape(self._shape)
                self._t = None
            return self._a


def _finish_cross(pc, with_reports):
    shape, ranks, cores, n, d, lay, h = pc.shape, pc.ranks, pc.cores, pc.n, pc.d, pc.lay, pc.h
    left, right = pc.left, pc.right
    trains = DeviceTTBatch(shape, ranks, cores, n)
    if not with_reports:
        return CrossBatchResult(trains, None, h["status"].copy(), h["bond"].copy(), h)
    # the packed index sets stay on the device until a report's sets are
    # first read (most callers only read prices and counters)
    left_h = _LazyHost(left, (n, lay.set_stride))
    right_h = _LazyHost(right, (n, lay.set_stride))
    total = math.prod(shape)
    reports = []
    lvalid = h["lvalid"].reshape(n, d + 1)

    def left_of(i):
        if d == 1:
            return lambda: [[()], None]
        return lambda: ([[()]] + [lay.unpack_set(left_h.get()[i], k, k) if lvalid[i, k] else None
                                  for k in range(1, d)] + [None])

    def right_of(i):
        if d == 1:
            return lambda: [None, [()]]
        return lambda: [None] + [lay.unpack_set(right_h.get()[i], k, d - k) for k in range(1, d)] + [[()]]

    for i in range(n):
        lsets, rsets = left_of(i), right_of(i)
        reports.append(CrossReport(
            converged=bool(h["conv"][i]),
            sweeps_used=int(h["sweeps"][i]),
            oracle_calls=int(h["calls"][i]),
            conv_check_calls=int(h["ccalls"][i]),
            final_diff=float(h["diff"][i]),
            compression_ratio=int(h["calls"][i]) / total,
            left_sets=lsets,
            right_sets=rsets,
        ))
    return CrossBatchResult(trains, reports, h["status"].copy(), h["bond"].copy(), h)


def tt_cross_batch(oracles, shape, cfg, with_reports=True):
    """Batched TT-cross of independent oracles sharing ``shape`` and ``cfg``.

    Returns a :class:`CrossBatchResult` whose trains stay on the GPU; per
    instance errors are reported in ``status`` (not raised).
    """
    torch = _lib.require_device()
    lib = _lib.load_library()
    pc = _prepare_cross(oracles, shape, cfg)
    ws_bytes = lib.ttp_cross_workspace(ctypes.byref(pc.prob))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=torch.device("cuda"))
    st = lib.ttp_cross_run(ctypes.byref(pc.prob), ctypes.byref(pc.out), ctypes.c_void_p(ws.data_ptr()),
                           ws_bytes, _lib.stream_handle())
    _lib.raise_for(st, "tt_cross")
    del ws
    return _finish_cross(pc, with_reports)

def tt_cross(oracle, shape, cfg):
    """Tensor-train approximation of a device oracle (cross.py:358-453).

    Returns ``(TensorTrain, CrossReport)``; non-convergence is reported, not
    raised.  ``oracle`` must be a device descriptor.
    """
    check_device_oracle(oracle)
    res = tt_cross_batch([oracle], shape, cfg)
    err = res.error_for(0)
    if err is not None:
        raise err
    return res.trains.to_trains()[0], res.reports[0]


def column_basis(mats, rank_tol=0.0):
    """Orthonormal column bases by pivoted QR, with the rank check
    (_column_basis, cross.py:103-119), computed exactly as the bond kernel's
    global-slice path does it (ttp_column_basis).  ``mats``: one (rows x cols)
    matrix or a stack of them, of the shapes that path serves (rows >= 2 cols,
    blocks of >= 1 MiB).  Returns the Q factors
    (columns in pivot order; the reference's Q up to unimodular column
    phases) with the stack's shape.  Raises SingularMatrixError when a matrix
    is zero or rank deficient by ``rank_tol``."""
    mats = np.asarray(mats, dtype=np.complex128)
    single = mats.ndim == 2
    if single:
        mats = mats[None]
    if mats.ndim != 3:
        raise ValueError("column_basis expects a matrix or a stack of matrices")
    n_mat, n, r = mats.shape
    if r > MAX_BOND or n < 2 * r or n * r * 16 < (1 << 20):
        raise ValueError(f"column_basis runs the bond kernel's global-slice path: blocks of >= 1 MiB "
                         f"with rows >= 2 cols and cols <= {MAX_BOND}")
    torch = _lib.require_device()
    lib = _lib.load_library()
    d_mat = torch.from_numpy(np.ascontiguousarray(mats)).to("cuda")
    d_q = torch.empty((n_mat, r, n), dtype=torch.complex128, device="cuda")
    ws_bytes = lib.ttp_column_basis_workspace(n_mat, n, r)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    status = np.zeros(n_mat, dtype=np.int32)
    st = lib.ttp_column_basis(n_mat, n, r, ctypes.c_void_p(d_mat.data_ptr()), float(rank_tol),
                              ctypes.c_void_p(d_q.data_ptr()),
                              status.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                              ctypes.c_void_p(ws.data_ptr()), ws_bytes, _lib.stream_handle())
    _lib.raise_for(st, "column_basis")
    if np.any(status == _lib.TTP_ERR_SINGULAR):
        bad = int(np.argmax(status == _lib.TTP_ERR_SINGULAR))
        raise SingularMatrixError(f"matrix {bad} of shape {(n, r)} is numerically rank deficient (or zero)")
    for s_ in status:
        _lib.raise_for(int(s_), "column_basis")
    q = d_q.transpose(1, 2).cpu().numpy()
    return q[0] if single else q


def maxvol(mat, slack=0.01, max_iters=None, rank_tol=RANK_TOL):
    """Rows whose square submatrix has quasi-maximal volume (cross.py:208-230)."""
    mat = np.asarray(mat, dtype=np.complex128)
    if mat.ndim != 2:
        raise ValueError("maxvol expects a matrix")
    n, r = mat.shape
    if n < r:
        raise ValueError(f"need at least as many rows as columns, got {mat.shape}")
    if r > MAX_BOND:
        raise ValueError(f"maxvol on the device supports at most {MAX_BOND} columns")
    torch = _lib.require_device()
    lib = _lib.load_library()
    d_mat = torch.from_numpy(np.ascontiguousarray(mat)).to("cuda")
    ws_bytes = lib.ttp_maxvol_workspace(1, n, r)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    sel = np.zeros(r, dtype=np.int64)
    status = np.zeros(1, dtype=np.int32)
    st = lib.ttp_maxvol(1, n, r, ctypes.c_void_p(d_mat.data_ptr()), float(slack),
                        -1 if max_iters is None else int(max_iters), float(rank_tol),
                        sel.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                        status.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                        ctypes.c_void_p(ws.data_ptr()), ws_bytes, _lib.stream_handle())
    _lib.raise_for(st, "maxvol")
    if status[0] == _lib.TTP_ERR_SINGULAR:
        raise SingularMatrixError(
            f"matrix of shape {mat.shape} is numerically rank deficient (or zero)")
    if status[0] == _lib.TTP_ERR_MAXVOL_ITER:
        limit = max_iters if max_iters is not None else 10 * n
        raise MaxvolIterationError(f"maxvol did not settle within {limit} row swaps")
    _lib.raise_for(int(status[0]), "maxvol")
    return sel
