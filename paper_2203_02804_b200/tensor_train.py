"""Tensor trains: host container plus the device contractions.

:class:`TensorTrain` keeps the reference's container semantics (immutable
complex cores ``(D_{k-1}, n_k, D_k)`` with unit boundary bonds,
tensor_train.py:40-101).  The contractions run on the GPU through the C ABI:

* :func:`tt_inner`          -> ``ttp_tt_inner``  (K7, tensor_train.py:143-159)
* :func:`tt_evaluate_many`  -> ``ttp_tt_eval``   (K6, tensor_train.py:126-140)
* :func:`tt_rand_sample_diff` draws the reference's seeded samples on the
  host (numpy Generator, bit-exact with tensor_train.py:191-194) and runs the
  evaluation, the oracle and the fixed-order reduction on the device.

The JSON container (tensor_train.py:228-261) is host I/O and is provided so
cores can be exchanged with the reference.
"""

from __future__ import annotations

import ctypes
import json
import math

import numpy as np

from . import _lib
from .oracles import OracleBatch, check_device_oracle

__all__ = [
    "TensorTrain",
    "tt_evaluate",
    "tt_evaluate_many",
    "tt_inner",
    "tt_inner_batch",
    "tt_rand_sample_diff",
    "tt_save_json",
    "tt_load_json",
    "sample_indices",
]


class TensorTrain:
    """Immutable chain of complex order-3 cores ``(D_{k-1}, n_k, D_k)``."""

    __slots__ = ("cores",)

    def __init__(self, cores):
        if len(cores) == 0:
            raise ValueError("a tensor train needs at least one core")
        frozen = []
        for k, core in enumerate(cores):
            arr = np.array(core, dtype=np.complex128, copy=True)
            if arr.ndim != 3:
                raise ValueError(f"core {k} has {arr.ndim} axes, expected 3")
            if min(arr.shape) < 1:
                raise ValueError(f"core {k} has an empty axis: shape {arr.shape}")
            arr.flags.writeable = False
            frozen.append(arr)
        if frozen[0].shape[0] != 1 or frozen[-1].shape[2] != 1:
            raise ValueError(
                "boundary bond dimensions must be 1, got "
                f"{frozen[0].shape[0]} and {frozen[-1].shape[2]}"
            )
        for k in range(len(frozen) - 1):
            if frozen[k].shape[2] != frozen[k + 1].shape[0]:
                raise ValueError(
                    f"bond mismatch between cores {k} and {k + 1}: "
                    f"{frozen[k].shape[2]} vs {frozen[k + 1].shape[0]}"
                )
        self.cores = tuple(frozen)

    @property
    def d(self):
        return len(self.cores)

    @property
    def phys_dims(self):
        return tuple(c.shape[1] for c in self.cores)

    @property
    def bond_dims(self):
        return (1,) + tuple(c.shape[2] for c in self.cores)

    @property
    def n_entries(self):
        return math.prod(self.phys_dims)

    def __repr__(self):
        return (f"TensorTrain(d={self.d}, phys_dims={self.phys_dims}, "
                f"bond_dims={self.bond_dims})")


class DeviceTTBatch:
    """A batch of same-shaped trains resident on the GPU (packed cores)."""

    def __init__(self, shape, bonds, flat, n_inst):
        self.shape = np.asarray(shape, dtype=np.int32)
        self.bonds = np.asarray(bonds, dtype=np.int32)
        sizes = [int(self.bonds[k] * self.shape[k] * self.bonds[k + 1]) for k in range(len(shape))]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.stride = int(self.offsets[-1])
        self.flat = flat  # torch complex128 (n_inst * stride,)
        self.n_inst = int(n_inst)
        self.struct = _lib.TTBatch(
            d=len(shape),
            n_inst=self.n_inst,
            h_shape=self.shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            h_bonds=self.bonds.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            h_offsets=self.offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            stride=self.stride,
            d_cores=flat.data_ptr(),
        )

    @classmethod
    def from_trains(cls, trains):
        torch = _lib.require_device()
        first = trains[0]
        for t in trains[1:]:
            if t.phys_dims != first.phys_dims or t.bond_dims != first.bond_dims:
                raise ValueError("trains in one batch must share shape and bonds")
        host = np.concatenate([np.concatenate([c.ravel() for c in t.cores]) for t in trains])
        flat = torch.from_numpy(host).to(torch.device("cuda"))
        return cls(first.phys_dims, first.bond_dims, flat, len(trains))

    def to_trains(self):
        host = self.flat.cpu().numpy()
        out = []
        for i in range(self.n_inst):
            base = i * self.stride
            cores = []
            for k in range(len(self.shape)):
                lo, hi = base + self.offsets[k], base + self.offsets[k + 1]
                cores.append(host[lo:hi].reshape(self.bonds[k], self.shape[k], self.bonds[k + 1]))
            out.append(TensorTrain(cores))
        return out


def _check_bonds(tt):
    if max(tt.bond_dims) > 64:
        raise ValueError("device contractions support bond dimensions <= 64")


def tt_inner_batch(bras, kets):
    """Device tt_inner over aligned batches (DeviceTTBatch) -> numpy complex (n,)."""
    torch = _lib.require_device()
    lib = _lib.load_library()
    if bras.n_inst != kets.n_inst:
        raise ValueError("batch sizes differ")
    if not np.array_equal(bras.shape, kets.shape):
        raise ValueError(
            "physical shape mismatch: "
            f"bra {list(map(int, bras.shape))} vs ket {list(map(int, kets.shape))}"
        )
    out = torch.empty(max(bras.n_inst, 1), dtype=torch.complex128, device="cuda")
    st = lib.ttp_tt_inner(ctypes.byref(bras.struct), ctypes.byref(kets.struct),
                          ctypes.c_void_p(out.data_ptr()), _lib.stream_handle())
    _lib.raise_for(st, "tt_inner")
    return out[: bras.n_inst].cpu().numpy()


def tt_inner(bra, ket):
    """``sum_idx conj(bra[idx]) * ket[idx]`` by transfer contraction on the GPU."""
    if bra.phys_dims != ket.phys_dims:
        raise ValueError(
            "physical shape mismatch: "
            f"bra {list(bra.phys_dims)} vs ket {list(ket.phys_dims)}"
        )
    _check_bonds(bra)
    _check_bonds(ket)
    b = DeviceTTBatch.from_trains([bra])
    k = DeviceTTBatch.from_trains([ket])
    return complex(tt_inner_batch(b, k)[0])


def _check_indices(tt, idx):
    idx = np.asarray(idx, dtype=np.int64)
    if idx.ndim != 2 or idx.shape[1] != tt.d:
        raise IndexError(f"index array must have shape (m, {tt.d}), got {idx.shape}")
    for axis, n in enumerate(tt.phys_dims):
        col = idx[:, axis]
        if col.size and (col.min() < 0 or col.max() >= n):
            bad = col[(col < 0) | (col >= n)][0]
            raise IndexError(f"axis {axis}: index {bad} out of range [0, {n})")
    return idx


def _device_eval(batch, idx):
    torch = _lib.require_device()
    lib = _lib.load_library()
    m = idx.shape[0]
    d_idx = torch.from_numpy(np.ascontiguousarray(idx.astype(np.int32))).to("cuda")
    out = torch.empty((batch.n_inst, max(m, 1)), dtype=torch.complex128, device="cuda")
    st = lib.ttp_tt_eval(ctypes.byref(batch.struct), ctypes.c_void_p(d_idx.data_ptr()), m,
                         ctypes.c_void_p(out.data_ptr()), None, 0, _lib.stream_handle())
    _lib.raise_for(st, "tt_evaluate_many")
    return out[:, :m]


def tt_evaluate_many(tt, idx):
    """Entries of ``tt`` at an ``(m, d)`` index array (GPU)."""
    idx = _check_indices(tt, idx)
    _check_bonds(tt)
    batch = DeviceTTBatch.from_trains([tt])
    return _device_eval(batch, idx)[0].cpu().numpy()


def tt_evaluate(tt, idx):
    """Single entry (reference tensor_train.py:114-123)."""
    idx = tuple(int(i) for i in idx)
    if len(idx) != tt.d:
        raise IndexError(f"index has {len(idx)} entries for a {tt.d}-site train")
    for axis, (i, n) in enumerate(zip(idx, tt.phys_dims)):
        if not 0 <= i < n:
            raise IndexError(f"axis {axis}: index {i} out of range [0, {n})")
    return complex(tt_evaluate_many(tt, np.array([idx]))[0])


def sample_indices(phys_dims, m, seed):
    """The reference's seeded sample draw, column by column (tensor_train.py:191-194)."""
    if m < 1:
        raise ValueError("sample count must be >= 1")
    rng = np.random.default_rng(seed)
    idx = np.empty((m, len(phys_dims)), dtype=np.int64)
    for axis, n in enumerate(phys_dims):
        idx[:, axis] = rng.integers(0, n, size=m)
    return idx


def tt_rand_sample_diff(tt, oracle, m, seed):
    """``sum|oracle - tt| / sum|oracle|`` on m seeded samples (GPU evaluation).

    ``oracle`` must be a device descriptor (see :mod:`oracles`).
    """
    if m < 1:
        raise ValueError("sample count must be >= 1")
    check_device_oracle(oracle)
    torch = _lib.require_device()
    lib = _lib.load_library()
    idx = sample_indices(tt.phys_dims, m, seed)
    _check_bonds(tt)
    batch = DeviceTTBatch.from_trains([tt])
    approx = _device_eval(batch, idx)
    exact = OracleBatch([oracle]).evaluate_device(idx, tt.phys_dims)[0, :m].contiguous()
    ws = torch.empty(16, dtype=torch.float64, device="cuda")
    out = (ctypes.c_double * 1)()
    st = lib.ttp_sample_diff(1, m, ctypes.c_void_p(exact.data_ptr()),
                             ctypes.c_void_p(approx.contiguous().data_ptr()), out,
                             ctypes.c_void_p(ws.data_ptr()), 128, _lib.stream_handle())
    _lib.raise_for(st, "tt_rand_sample_diff")
    return float(out[0])


def tt_save_json(tt, path):
    """Self-describing JSON container; interleaved re/im, row-major cores."""
    payload = {
        "format": "tensor-train",
        "version": 1,
        "phys_dims": list(tt.phys_dims),
        "bond_dims": list(tt.bond_dims),
        "cores": [np.column_stack([c.real.ravel(), c.imag.ravel()]).ravel().tolist()
                  for c in tt.cores],
    }
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(payload, fh)


def tt_load_json(path):
    with open(path, "r", encoding="utf-8") as fh:
        payload = json.load(fh)
    if payload.get("format") != "tensor-train":
        raise ValueError(f"not a tensor-train container: {path}")
    phys, bonds = payload["phys_dims"], payload["bond_dims"]
    cores = []
    for k, flat in enumerate(payload["cores"]):
        pairs = np.asarray(flat, dtype=np.float64).reshape(-1, 2)
        cores.append((pairs[:, 0] + 1j * pairs[:, 1]).reshape(bonds[k], phys[k], bonds[k + 1]))
    return TensorTrain(cores)
