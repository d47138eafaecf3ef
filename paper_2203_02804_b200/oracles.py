"""Device oracle descriptors: the plugins tt_cross samples.

The reference's oracle is any Python callable ``(m, d) int64 -> (m,)
complex128`` (tensor_train.py:11-13).  A Python callback cannot run inside a
CUDA kernel, and the hot path has no host fallback, so oracles here are
*descriptors*: a kind plus parameters that the fiber kernels evaluate in
registers.  Every descriptor is still callable with the reference
convention -- the call evaluates on the GPU and returns numpy -- so tests read
like the reference's own.

Hot-path kinds: :class:`PhiGridOracle` (phi_grid_oracle, pricers.py:234-240)
and :class:`PayoffGridOracle` (payoff_grid_oracle, pricers.py:243-253).
Test kinds: :class:`SeparableOracle`, :class:`TTOracle`, :class:`TableOracle`.
Passing any other callable to the device paths raises ``TypeError``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


class DeviceOracle:
    """Base class.  Subclasses define kind, d, shape and per-instance arrays."""

    kind = 0

    def __init__(self, d, shape=None):
        self.d = int(d)
        self.shape = None if shape is None else tuple(int(n) for n in shape)

    # per-instance payloads (numpy); overridden by subclasses
    def params(self):
        return np.zeros(1, dtype=np.float64)

    def table(self):
        return np.zeros(1, dtype=np.complex128)

    def table_offsets(self):
        return np.zeros(self.d + 1, dtype=np.int64)

    def tt_bonds(self):
        return np.ones(self.d + 1, dtype=np.int32)

    def compatible(self, other):
        return (type(self) is type(other) and self.d == other.d
                and self.params().shape == other.params().shape
                and self.table().shape == other.table().shape
                and np.array_equal(self.table_offsets(), other.table_offsets())
                and np.array_equal(self.tt_bonds(), other.tt_bonds()))

    def __call__(self, idx):
        """Evaluate at an (m, d) integer index array on the GPU -> numpy (m,)."""
        idx = np.asarray(idx, dtype=np.int64)
        if idx.ndim != 2 or idx.shape[1] != self.d:
            raise IndexError(f"index array must have shape (m, {self.d}), got {idx.shape}")
        shape = self.shape if self.shape is not None else tuple(int(idx[:, k].max()) + 1 if len(idx) else 1 for k in range(self.d))
        batch = OracleBatch([self])
        return batch.evaluate(idx, shape)[0]


def check_device_oracle(oracle):
    if not isinstance(oracle, DeviceOracle):
        raise TypeError(
            "the B200 tt_cross samples device oracle descriptors only "
            "(PhiGridOracle, PayoffGridOracle, SeparableOracle, TTOracle, "
            f"TableOracle); got {type(oracle).__name__}. Python callables "
            "cannot run inside the fiber kernels and there is no CPU fallback."
        )
    return oracle


class GridOracleBase(DeviceOracle):
    def __init__(self, model, grid):
        if model.d != grid.d:
            raise ValueError(f"model has d={model.d} but grid has d={grid.d}")
        super().__init__(grid.d, (grid.points_per_axis,) * grid.d)
        self.model = model
        self.grid = grid


class PhiGridOracle(GridOracleBase):
    """idx -> phi_T(-z(idx)) on the contour (pricers.py:234-240)."""

    kind = _lib.ORACLE_PHI_GBM

    def params(self):
        g, m = self.grid, self.model
        head = np.array([g.eta, g.alpha, float(g.n // 2)])
        return np.concatenate([head, m.log_drift, m.log_cov.ravel()]).astype(np.float64)


class PayoffGridOracle(GridOracleBase):
    """idx -> conj(vhat_min(z(idx))) (pricers.py:243-253); ``conj=False`` gives
    vhat itself, as the dense sum uses it (pricers.py:196)."""

    kind = _lib.ORACLE_VHAT_MIN

    def __init__(self, model, grid, conj=True):
        super().__init__(model, grid)
        self.conj = bool(conj)

    def params(self):
        g = self.grid
        return np.array([g.eta, g.alpha, float(g.n // 2), self.model.strike,
                         1.0 if self.conj else 0.0], dtype=np.float64)


class SeparableOracle(DeviceOracle):
    """idx -> prod_k w_k[idx_k] (the test suite's rank-1 oracle)."""

    kind = _lib.ORACLE_SEPARABLE

    def __init__(self, weights):
        ws = [np.asarray(w, dtype=np.complex128).ravel() for w in weights]
        super().__init__(len(ws), tuple(len(w) for w in ws))
        self._w = ws

    def table(self):
        return np.concatenate(self._w)

    def table_offsets(self):
        return np.concatenate([[0], np.cumsum([len(w) for w in self._w])]).astype(np.int64)


class TableOracle(DeviceOracle):
    """idx -> values[idx] for an explicit (small) dense tensor."""

    kind = _lib.ORACLE_TABLE

    def __init__(self, values):
        vals = np.asarray(values, dtype=np.complex128)
        super().__init__(vals.ndim, vals.shape)
        self._vals = vals

    def table(self):
        return np.ascontiguousarray(self._vals).ravel()


class TTOracle(DeviceOracle):
    """idx -> entries of a target tensor train (tt_evaluate_many as an oracle)."""

    kind = _lib.ORACLE_TT

    def __init__(self, tt):
        super().__init__(tt.d, tt.phys_dims)
        if max(tt.bond_dims) > 64:
            raise ValueError("TT oracle supports bond dimensions <= 64")
        self.tt = tt

    def table(self):
        return np.concatenate([c.ravel() for c in self.tt.cores])

    def table_offsets(self):
        sizes = [c.size for c in self.tt.cores]
        return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)

    def tt_bonds(self):
        return np.asarray(self.tt.bond_dims, dtype=np.int32)


class OracleBatch:
    """n_inst compatible descriptors packed into device buffers.

    Holds the torch tensors alive for as long as the ctypes struct is used.
    """

    def __init__(self, oracles):
        oracles = [check_device_oracle(o) for o in oracles]
        if not oracles:
            raise ValueError("empty oracle batch")
        first = oracles[0]
        plist = [o.params() for o in oracles]
        tlist = [o.table() for o in oracles]
        # layout check (per-instance payloads computed once; the table
        # layouts only exist for the table-backed kinds)
        table_kind = first.kind in (_lib.ORACLE_SEPARABLE, _lib.ORACLE_TT, _lib.ORACLE_TABLE)
        off0, bonds0 = first.table_offsets(), first.tt_bonds()
        for o, p, t in zip(oracles[1:], plist[1:], tlist[1:]):
            same = (type(o) is type(first) and o.d == first.d and p.shape == plist[0].shape
                    and t.shape == tlist[0].shape)
            if same and table_kind:
                same = np.array_equal(o.table_offsets(), off0) and np.array_equal(o.tt_bonds(), bonds0)
            if not same:
                raise ValueError("oracles in one batch must share kind and layout")
        torch = _lib.require_device()
        self.kind = first.kind
        self.d = first.d
        self.n_inst = len(oracles)
        dev = torch.device("cuda")
        params = np.stack(plist).astype(np.float64)
        table = np.stack(tlist).astype(np.complex128)
        self._params = torch.from_numpy(np.ascontiguousarray(params)).to(dev)
        self._table = torch.from_numpy(np.ascontiguousarray(table)).to(dev)
        self._offsets = torch.from_numpy(first.table_offsets().astype(np.int64)).to(dev)
        self._bonds = torch.from_numpy(first.tt_bonds().astype(np.int32)).to(dev)
        self.struct = _lib.Oracle(
            kind=self.kind,
            d=self.d,
            param_stride=params.shape[1],
            params=self._params.data_ptr(),
            table_stride=table.shape[1],
            table=self._table.data_ptr(),
            table_offsets=self._offsets.data_ptr(),
            tt_bonds=self._bonds.data_ptr(),
        )

    def evaluate(self, idx, shape):
        """Values of every instance at the shared indices -> (n_inst, m) numpy."""
        m = np.asarray(idx).shape[0]
        return self.evaluate_device(idx, shape)[:, :m].cpu().numpy()

    def fiber_blocks(self, left, right, axis, shape, layout):
        """Sampled unfolding block of every instance (ttp_eval_fibers, the
        bond kernels' own separable evaluation; reference _block,
        cross.py:310-332).  ``left``: (n_left, axis) and ``right``:
        (n_right, d - axis - 1) integer tuples shared by all instances.
        Returns (n_inst, rows, cols) complex numpy: layout 0 rows a*n + s,
        columns b; layout 1 rows s*n_right + b, columns a (the transpose of
        the reference's axis-first block, as _interp_core receives it)."""
        torch = _lib.require_device()
        lib = _lib.load_library()
        shape = tuple(int(n) for n in shape)
        n = shape[axis]
        left = np.asarray(left, dtype=np.int64)
        right = np.asarray(right, dtype=np.int64)
        left = left.reshape(left.shape[0] if left.ndim else 1, axis)
        right = right.reshape(right.shape[0] if right.ndim else 1, self.d - axis - 1)
        for tup, lo in ((left, 0), (right, axis + 1)):
            for j in range(tup.shape[1]):
                if tup.size and (tup[:, j].min() < 0 or tup[:, j].max() >= shape[lo + j]):
                    raise IndexError(f"axis {lo + j}: index out of range [0, {shape[lo + j]})")
        nl, nr = left.shape[0], right.shape[0]
        rows, cols = (nl * n, nr) if layout == 0 else (n * nr, nl)
        dev = torch.device("cuda")
        d_left = torch.from_numpy(np.ascontiguousarray(left.astype(np.int32)).reshape(-1)).to(dev)
        d_right = torch.from_numpy(np.ascontiguousarray(right.astype(np.int32)).reshape(-1)).to(dev)
        d_shape = torch.tensor(shape, dtype=torch.int32, device=dev)
        out = torch.empty((self.n_inst, cols, rows), dtype=torch.complex128, device=dev)
        st = lib.ttp_eval_fibers(ctypes.byref(self.struct), ctypes.c_void_p(d_shape.data_ptr()),
                                 self.n_inst, int(layout), int(axis), n,
                                 ctypes.c_void_p(d_left.data_ptr() if d_left.numel() else d_shape.data_ptr()),
                                 nl, ctypes.c_void_p(d_right.data_ptr() if d_right.numel() else d_shape.data_ptr()),
                                 nr, ctypes.c_void_p(out.data_ptr()), rows * cols, _lib.stream_handle())
        _lib.raise_for(st, "fiber evaluation")
        return out.transpose(1, 2).cpu().numpy()  # column-major -> (rows, cols)

    def evaluate_device(self, idx, shape):
        """Values at the shared indices as a (n_inst, max(m, 1)) device tensor."""
        torch = _lib.require_device()
        lib = _lib.load_library()
        idx = np.asarray(idx, dtype=np.int64)
        m = idx.shape[0]
        shape = tuple(int(n) for n in shape)
        for axis, n in enumerate(shape):
            col = idx[:, axis]
            if col.size and (col.min() < 0 or col.max() >= n):
                bad = col[(col < 0) | (col >= n)][0]
                raise IndexError(f"axis {axis}: index {bad} out of range [0, {n})")
        dev = torch.device("cuda")
        d_idx = torch.from_numpy(np.ascontiguousarray(idx.astype(np.int32))).to(dev)
        d_shape = torch.tensor(shape, dtype=torch.int32, device=dev)
        out = torch.empty((self.n_inst, max(m, 1)), dtype=torch.complex128, device=dev)
        st = lib.ttp_oracle_eval(ctypes.byref(self.struct), ctypes.c_void_p(d_shape.data_ptr()),
                                 self.n_inst, ctypes.c_void_p(d_idx.data_ptr()), m,
                                 ctypes.c_void_p(out.data_ptr()), _lib.stream_handle())
        _lib.raise_for(st, "oracle evaluation")
        return out
