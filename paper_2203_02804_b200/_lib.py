"""ctypes binding of the C ABI in include/ttpricer_b200.h.

The shared library is built in-tree (``csrc/Makefile`` -> ``libttpricer_b200.so``
next to this file).  Loading never falls back to anything: a missing library
or a missing CUDA device raises :class:`DeviceError` at the first compute
call.  Device buffers are torch CUDA tensors; only their raw pointers cross
the ABI.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    CapacityError,
    DeviceError,
    MaxvolIterationError,
    OracleBudgetError,
    ResidueError,
    SingularMatrixError,
)

LIB_NAME = "libttpricer_b200.so"
# The dev variant (`make -C csrc dev`, -DTTP_DEV) carries the TTP_* A/B knobs;
# it is loaded only when TTP_DEV_LIBRARY=1 (tools/ and the knob-neutrality
# tests, each in its own process).  Everything else runs the release library.
DEV_LIB_NAME = "libttpricer_b200_dev.so"
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, DEV_LIB_NAME if os.environ.get("TTP_DEV_LIBRARY") == "1" else LIB_NAME)

TTP_OK = 0
TTP_ERR_INVALID = 1
TTP_ERR_CUDA = 2
TTP_ERR_SINGULAR = 3
TTP_ERR_MAXVOL_ITER = 4
TTP_ERR_BUDGET = 5
TTP_ERR_CAPACITY = 6
TTP_ERR_WORKSPACE = 7
TTP_ERR_RESIDUE = 8

ORACLE_PHI_GBM = 1
ORACLE_VHAT_MIN = 2
ORACLE_SEPARABLE = 3
ORACLE_TT = 4
ORACLE_TABLE = 5

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
_sz = ctypes.c_size_t


class Oracle(ctypes.Structure):
    _fields_ = [
        ("kind", _i32),
        ("d", _i32),
        ("param_stride", _i64),
        ("params", _p),
        ("table_stride", _i64),
        ("table", _p),
        ("table_offsets", _p),
        ("tt_bonds", _p),
    ]


class TTBatch(ctypes.Structure):
    _fields_ = [
        ("d", _i32),
        ("n_inst", _i32),
        ("h_shape", ctypes.POINTER(_i32)),
        ("h_bonds", ctypes.POINTER(_i32)),
        ("h_offsets", ctypes.POINTER(_i64)),
        ("stride", _i64),
        ("d_cores", _p),
    ]


class CrossCfg(ctypes.Structure):
    _fields_ = [
        ("bond_dim", _i32),
        ("max_sweeps", _i32),
        ("eps_tol", _f64),
        ("n_conv_samples", _i64),
        ("maxvol_slack", _f64),
        ("oracle_call_budget", _i64),
    ]


class CrossProblem(ctypes.Structure):
    _fields_ = [
        ("d", _i32),
        ("n_inst", _i32),
        ("h_shape", ctypes.POINTER(_i32)),
        ("d_shape", _p),
        ("oracle", Oracle),
        ("cfg", CrossCfg),
        ("d_right_init", _p),
        ("d_conv_idx", _p),
        ("d_conv_perm", _p),
        ("d_conv_off", _p),
    ]


class PriceProblem(ctypes.Structure):
    _fields_ = [
        ("phi", CrossProblem),
        ("vhat", CrossProblem),
        ("h_prefactor", ctypes.POINTER(_f64)),
    ]


class CrossLayout(ctypes.Structure):
    _fields_ = [
        ("ranks", _i32 * 65),
        ("core_offsets", _i64 * 65),
        ("core_stride", _i64),
        ("set_offsets", _i64 * 65),
        ("set_stride", _i64),
        ("max_rows", _i64),
        ("max_rank", _i32),
    ]


class CrossOut(ctypes.Structure):
    _fields_ = [
        ("d_cores", _p),
        ("d_left", _p),
        ("d_right", _p),
        ("h_status", ctypes.POINTER(_i32)),
        ("h_error_bond", ctypes.POINTER(_i32)),
        ("h_converged", ctypes.POINTER(_i32)),
        ("h_sweeps", ctypes.POINTER(_i32)),
        ("h_left_valid", ctypes.POINTER(_i32)),
        ("h_oracle_calls", ctypes.POINTER(_i64)),
        ("h_conv_calls", ctypes.POINTER(_i64)),
        ("h_final_diff", ctypes.POINTER(_f64)),
    ]


class KernelStat(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 32),
        ("launches", _i64),
        ("timed_launches", _i64),
        ("total_ms", _f64),
    ]


# (name, restype, argtypes) for every symbol declared in include/ttpricer_b200.h
SIGNATURES = [
    ("ttp_abi_version", _i32, []),
    ("ttp_last_error", ctypes.c_char_p, []),
    ("ttp_device_count", _i32, []),
    ("ttp_launch_count", _i64, []),
    ("ttp_profile_enable", None, [ctypes.c_int]),
    ("ttp_profile_reset", None, []),
    ("ttp_profile_read", _i32, [ctypes.POINTER(KernelStat), _i32]),
    ("ttp_oracle_eval", _i32, [ctypes.POINTER(Oracle), _p, _i32, _p, _i64, _p, _p]),
    ("ttp_eval_fibers", _i32, [ctypes.POINTER(Oracle), _p, _i32, _i32, _i32, _i32, _p, _i32, _p, _i32,
                                _p, _i64, _p]),
    ("ttp_tt_inner", _i32, [ctypes.POINTER(TTBatch), ctypes.POINTER(TTBatch), _p, _p]),
    ("ttp_tt_eval_workspace", _sz, [ctypes.POINTER(TTBatch), _i64]),
    ("ttp_tt_eval", _i32, [ctypes.POINTER(TTBatch), _p, _i64, _p, _p, _sz, _p]),
    ("ttp_sample_diff", _i32, [_i32, _i64, _p, _p, ctypes.POINTER(_f64), _p, _sz, _p]),
    ("ttp_dense_workspace", _sz, [_i32, _i64]),
    ("ttp_dense_sum", _i32, [ctypes.POINTER(Oracle), ctypes.POINTER(Oracle), ctypes.POINTER(_i32),
                             _p, _i32, ctypes.POINTER(_f64), _p, _sz, _p]),
    ("ttp_dense_sum_range", _i32, [ctypes.POINTER(Oracle), ctypes.POINTER(Oracle), ctypes.POINTER(_i32),
                                   _p, _i32, _i64, _i64, ctypes.POINTER(_f64), _p, _sz, _p]),
    ("ttp_cross_layout_of", _i32, [_i32, ctypes.POINTER(_i32), _i32, ctypes.POINTER(CrossLayout)]),
    ("ttp_cross_workspace", _sz, [ctypes.POINTER(CrossProblem)]),
    ("ttp_cross_run", _i32, [ctypes.POINTER(CrossProblem), ctypes.POINTER(CrossOut), _p, _sz, _p]),
    ("ttp_mc_param_count", _i32, [_i32]),
    ("ttp_mc_workspace", _sz, [_i32, _i64]),
    ("ttp_mc_price", _i32, [_p, _i64, _i32, _i32, _i64, ctypes.POINTER(ctypes.c_uint64), _i32, _i32,
                            ctypes.POINTER(_f64), _p, _sz, _p]),
    ("ttp_philox4x32", _i32, [ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                              ctypes.POINTER(ctypes.c_uint32)]),
    ("ttp_price_tt_workspace", _sz, [ctypes.POINTER(PriceProblem)]),
    ("ttp_price_tt_batch", _i32, [ctypes.POINTER(PriceProblem), ctypes.POINTER(CrossOut),
                                  ctypes.POINTER(CrossOut), ctypes.POINTER(_f64), ctypes.POINTER(_f64),
                                  _p, _sz, _p]),
    ("ttp_column_basis_workspace", _sz, [_i32, _i64, _i32]),
    ("ttp_column_basis", _i32, [_i32, _i64, _i32, _p, _f64, _p, ctypes.POINTER(_i32), _p, _sz, _p]),
    ("ttp_maxvol_workspace", _sz, [_i32, _i64, _i32]),
    ("ttp_maxvol", _i32, [_i32, _i64, _i32, _p, _f64, _i64, _f64, ctypes.POINTER(_i64),
                          ctypes.POINTER(_i32), _p, _sz, _p]),
]

_lock = threading.Lock()
_lib = None


def load_library(path=LIB_PATH):
    """Load (once) and return the ctypes handle; raise DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"{os.path.basename(path)} is not built (expected at {path}); run "
                "`make -C paper_2203_02804_b200/csrc` (or `... dev`) or __graft_entry__.build()"
            )
        lib = ctypes.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if hasattr(lib, "ttp_dev_phase_clocks"):  # dev build only
            lib.ttp_dev_phase_clocks.restype = _i32
            lib.ttp_dev_phase_clocks.argtypes = [ctypes.c_int, ctypes.POINTER(_i64), _i32]
        if lib.ttp_abi_version() != 1:
            raise DeviceError("libttpricer_b200.so ABI version mismatch")
        _lib = lib
        return lib


def last_error():
    msg = load_library().ttp_last_error()
    return msg.decode() if msg else ""


def raise_for(status, context="", bond=None):
    """Map a ttp_status to the reference's exception classes."""
    if status == TTP_OK:
        return
    msg = last_error() or context
    if context and context not in msg:
        msg = f"{context}: {msg}"
    if status == TTP_ERR_INVALID:
        raise ValueError(msg)
    if status == TTP_ERR_SINGULAR:
        raise SingularMatrixError(msg, bond=bond)
    if status == TTP_ERR_MAXVOL_ITER:
        raise MaxvolIterationError(msg)
    if status == TTP_ERR_BUDGET:
        raise OracleBudgetError(msg)
    if status == TTP_ERR_CAPACITY:
        raise CapacityError(msg)
    if status == TTP_ERR_RESIDUE:
        raise ResidueError(msg)
    raise DeviceError(msg or f"ttp status {status}")


def require_device():
    """Return the torch module after checking a CUDA device is usable."""
    import torch

    load_library()
    if not torch.cuda.is_available():
        raise DeviceError(
            "no CUDA device visible: the B200 pricer has no CPU fallback"
        )
    return torch


def launch_count():
    """Kernels launched by the library so far (diagnostic counter)."""
    return int(load_library().ttp_launch_count())


def profile_enable(on=True):
    load_library().ttp_profile_enable(1 if on else 0)


def profile_reset():
    load_library().ttp_profile_reset()


def profile_read():
    """{kernel class: (launches, timed_launches, total_ms)} since the last reset."""
    arr = (KernelStat * 32)()
    n = load_library().ttp_profile_read(arr, 32)
    return {arr[i].name.decode(): (int(arr[i].launches), int(arr[i].timed_launches),
                                   float(arr[i].total_ms)) for i in range(n)}


def stream_handle():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
