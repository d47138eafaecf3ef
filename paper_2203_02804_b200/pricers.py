"""Fourier pricing engines on the GPU (reference pricers.py).

``price_fourier_tt`` is the drop-in boundary of the hot path
(pricers.py:256-294): two device TT-crosses (phi and conj(vhat)) followed by
the device tt_inner.  ``price_fourier_tt_batch`` prices many independent
options per call -- the throughput path the benchmark measures -- and keeps
the trains resident on the GPU between the crosses and the contraction.
``price_fourier_dense`` is the full-grid cross-check (pricers.py:199-231,
kernel K8).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cross import CrossConfig, tt_cross_batch
from .errors import CapacityError, ResidueError, StripConditionError
from .oracles import OracleBatch, PayoffGridOracle, PhiGridOracle
from .tensor_train import tt_inner_batch

__all__ = [
    "GridSpec",
    "PricingResult",
    "grid_admissible",
    "table1_hyperparams",
    "phi_grid_oracle",
    "payoff_grid_oracle",
    "price_fourier_dense",
    "price_fourier_dense_batch",
    "price_fourier_tt",
    "price_fourier_tt_batch",
    "DENSE_TERM_CAP",
]

DENSE_TERM_CAP = 100_000_000


@dataclass(frozen=True)
class GridSpec:
    """Per-axis grid of n+1 points j = -n/2..n/2 (pricers.py:49-86)."""

    n: int
    eta: float
    alpha: float
    d: int

    def __post_init__(self):
        if self.n < 2 or self.n % 2 != 0:
            raise ValueError(f"n must be even and >= 2, got {self.n}")
        if self.eta <= 0:
            raise ValueError("eta must be > 0")
        if self.d < 1:
            raise ValueError("d must be >= 1")

    @property
    def points_per_axis(self):
        return self.n + 1

    @property
    def n_terms(self):
        return (self.n + 1) ** self.d

    def index_to_u(self, j):
        return self.eta * np.asarray(j)

    def contour(self, idx):
        return self.eta * (np.asarray(idx, dtype=np.int64) - self.n // 2) + 1j * self.alpha


@dataclass
class PricingResult:
    price: float
    method: str
    wall_time_s: float
    diagnostics: dict = field(default_factory=dict)

    def to_dict(self, include_timing=True):
        diag = {k: (v.to_dict() if hasattr(v, "to_dict") else v) for k, v in self.diagnostics.items()}
        out = {"price": self.price, "method": self.method, "diagnostics": diag}
        if include_timing:
            out["wall_time_s"] = self.wall_time_s
        return out


def grid_admissible(grid, payoff="min"):
    """Strip conditions of the payoff transform (pricers.py:108-127)."""
    reasons = []
    if payoff == "min":
        if grid.alpha <= 0:
            reasons.append(f"imaginary shift {grid.alpha} is not positive")
        if grid.d * grid.alpha <= 1:
            reasons.append(f"sum of shifts d*alpha = {grid.d * grid.alpha} is not above 1")
    elif payoff == "call":
        if grid.alpha <= 1:
            reasons.append(f"imaginary shift {grid.alpha} is not above 1")
    else:
        raise ValueError(f"unknown payoff kind {payoff!r}")
    return not reasons, reasons


def _require_admissible(grid):
    ok, reasons = grid_admissible(grid, "min")
    if not ok:
        raise StripConditionError("; ".join(reasons))


_TABLE1 = {2: (0.5, 20, 10), 3: (0.4, 20, 10), 4: (0.3, 30, 15), 5: (0.3, 30, 15),
           6: (0.2, 30, 15), 7: (0.2, 40, 20), 8: (0.2, 40, 20), 9: (0.2, 40, 20),
           10: (0.2, 40, 20)}


def table1_hyperparams(d):
    """(eta, bond_v, bond_phi) of the paper's Table I (pricers.py:136-151)."""
    if d < 2:
        raise ValueError("tabulated hyperparameters start at d=2")
    return _TABLE1.get(d, (0.2, 50, 25))


def phi_grid_oracle(model, grid):
    return PhiGridOracle(model, grid)


def payoff_grid_oracle(model, grid):
    return PayoffGridOracle(model, grid, conj=True)


def _prefactor(model, grid, t):
    return np.exp(-model.r * (model.T - t)) * grid.eta ** grid.d / (2.0 * np.pi) ** grid.d


def price_fourier_dense_batch(models, grid, t=0.0, term_cap=DENSE_TERM_CAP):
    """Dense contour sums for several models on one grid -> list of PricingResult."""
    for m in models:
        if m.d != grid.d:
            raise ValueError(f"model has d={m.d} but grid has d={grid.d}")
    _require_admissible(grid)
    if grid.n_terms > term_cap:
        raise CapacityError(f"dense sum needs {grid.n_terms} terms, cap is {term_cap}")
    torch = _lib.require_device()
    lib = _lib.load_library()
    start = time.perf_counter()
    phi = OracleBatch([PhiGridOracle(m, grid) for m in models])
    vhat = OracleBatch([PayoffGridOracle(m, grid, conj=False) for m in models])
    shape = np.full(grid.d, grid.points_per_axis, dtype=np.int32)
    d_shape = torch.from_numpy(shape).to("cuda")
    n = len(models)
    ws_bytes = lib.ttp_dense_workspace(n, grid.n_terms)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    sums = (ctypes.c_double * (2 * n))()
    st = lib.ttp_dense_sum(ctypes.byref(phi.struct), ctypes.byref(vhat.struct),
                           shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                           ctypes.c_void_p(d_shape.data_ptr()), n, sums,
                           ctypes.c_void_p(ws.data_ptr()), ws_bytes, _lib.stream_handle())
    _lib.raise_for(st, "dense sum")
    wall = time.perf_counter() - start
    out = []
    for i, m in enumerate(models):
        acc = complex(sums[2 * i], sums[2 * i + 1])
        value = _prefactor(m, grid, t) * acc
        residue = float(abs(value.imag) / abs(value)) if value != 0 else 0.0
        if residue > 1e-8 and abs(value.imag) > 1e-12:
            raise ResidueError(f"imaginary residue {residue:.3e} of the contour sum exceeds 1e-8")
        out.append(PricingResult(float(value.real), "fourier_dense", wall / n,
                                 {"n_terms": grid.n_terms, "imag_residue": residue}))
    return out


def dense_partial_sum(model, grid, first, count):
    """Raw contour sum (no prefactor) over the flat term range [first, first +
    count) on the device (ttp_dense_sum_range) -> complex."""
    _require_admissible(grid)
    torch = _lib.require_device()
    lib = _lib.load_library()
    phi = OracleBatch([PhiGridOracle(model, grid)])
    vhat = OracleBatch([PayoffGridOracle(model, grid, conj=False)])
    shape = np.full(grid.d, grid.points_per_axis, dtype=np.int32)
    d_shape = torch.from_numpy(shape).to("cuda")
    ws_bytes = lib.ttp_dense_workspace(1, grid.n_terms)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    out = (ctypes.c_double * 2)()
    st = lib.ttp_dense_sum_range(ctypes.byref(phi.struct), ctypes.byref(vhat.struct),
                                 shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                 ctypes.c_void_p(d_shape.data_ptr()), 1, int(first), int(count), out,
                                 ctypes.c_void_p(ws.data_ptr()), ws_bytes, _lib.stream_handle())
    _lib.raise_for(st, "dense sum")
    return complex(out[0], out[1])


def price_fourier_dense(model, grid, t=0.0, term_cap=DENSE_TERM_CAP):
    """Dense nested contour sum on the GPU (pricers.py:199-231)."""
    if model.d != grid.d:
        raise ValueError(f"model has d={model.d} but grid has d={grid.d}")
    return price_fourier_dense_batch([model], grid, t=t, term_cap=term_cap)[0]


_PAIR_STREAMS = {}


def run_cross_pair(phi_batch, v_batch, shape, cfg_phi, cfg_v, with_reports=True, concurrent=True):
    """The two independent crosses of price_fourier_tt (pricers.py:271-272)
    issued from two host threads on two CUDA streams, so the phi and vhat
    sweeps overlap on the GPU (each sweep driver blocks its own thread on the
    per-sweep convergence read-back).  Returns (phi_result, v_result).
    ``concurrent=False`` runs them one after the other on the caller's
    stream (bench.py's per-kernel timing step); results are identical."""
    torch = _lib.require_device()
    if not concurrent:
        return (tt_cross_batch(phi_batch, shape, cfg_phi, with_reports=with_reports),
                tt_cross_batch(v_batch, shape, cfg_v, with_reports=with_reports))
    dev = torch.cuda.current_device()
    if dev not in _PAIR_STREAMS:
        _PAIR_STREAMS[dev] = (torch.cuda.Stream(), torch.cuda.Stream())
    s_phi, s_v = _PAIR_STREAMS[dev]
    caller = torch.cuda.current_stream()
    # shared read-only inputs are staged on the caller's stream first
    from .cross import _ConvSamples
    _ConvSamples.get(shape, cfg_phi.n_conv_samples, cfg_phi.seed)
    _ConvSamples.get(shape, cfg_v.n_conv_samples, cfg_v.seed)
    s_phi.wait_stream(caller)
    s_v.wait_stream(caller)
    out, err = {}, {}

    def work(key, stream, batch, cfg):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(stream):
                out[key] = tt_cross_batch(batch, shape, cfg, with_reports=with_reports)
        except BaseException as exc:  # re-raised on the caller's thread
            err[key] = exc

    import threading
    th = threading.Thread(target=work, args=("v", s_v, v_batch, cfg_v))
    th.start()
    work("phi", s_phi, phi_batch, cfg_phi)
    th.join()
    for key in ("phi", "v"):
        if key in err:
            raise err[key]
    caller.wait_stream(s_phi)
    caller.wait_stream(s_v)
    # results were allocated on the side streams; keep them alive for the caller's stream
    for res in (out["phi"], out["v"]):
        res.trains.flat.record_stream(caller)
    return out["phi"], out["v"]


_PER_INSTANCE = {}
_DEVICE_TOTAL = {}


def max_batch(shape, cfg_phi, cfg_v, n=None, fraction=0.6):
    """Largest number of instances whose phi and vhat crosses fit together in
    `fraction` of the device memory currently free.  Batches of n instances
    that need under a third of the device's total memory skip the (slow)
    free-memory query and are returned as they are."""
    from .cross import cross_bytes_per_instance
    torch = _lib.require_device()
    key = (tuple(shape), cfg_phi.bond_dim, cfg_phi.n_conv_samples, cfg_v.bond_dim, cfg_v.n_conv_samples)
    if key not in _PER_INSTANCE:
        _PER_INSTANCE[key] = cross_bytes_per_instance(shape, cfg_phi) + cross_bytes_per_instance(shape, cfg_v)
    per = _PER_INSTANCE[key]
    dev = torch.cuda.current_device()
    if dev not in _DEVICE_TOTAL:
        _DEVICE_TOTAL[dev] = torch.cuda.get_device_properties(dev).total_memory
    if n is not None and n * per <= _DEVICE_TOTAL[dev] // 3:
        return n
    free, _ = torch.cuda.mem_get_info()
    # blocks torch's caching allocator holds but has not handed out are as good
    # as free (it reuses them, and releases them before giving up on a request):
    # without them a second call in the same process sees a fraction of the
    # memory the first saw and runs the same batch in many more chunks
    free += max(0, torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev))
    return max(1, int(fraction * free) // max(1, per))


def balanced_chunk(n, limit):
    """Chunk size for n instances when at most `limit` fit at once: the fewest
    chunks, of equal size (148 options with room for 122 run as 74 + 74, not
    122 + 26: a short last chunk costs a full chunk's latency)."""
    limit = max(1, int(limit))
    k = -(-n // limit)
    return -(-n // k) if k > 0 else limit


def price_fourier_tt_batch(models, grid, cfg_phi, cfg_v, t=0.0, dense_reference="never",
                           term_cap=DENSE_TERM_CAP, raise_errors=True, group=None):
    """Price many independent options on one grid with the device TT path.

    All instances share the grid and the two CrossConfigs (so they share the
    seeded pivot initialisation and convergence samples); parameters differ
    per instance.  Returns a list of PricingResult (or exceptions when
    ``raise_errors`` is False).

    ``group``: a torch.distributed process group (e.g. ``dist.group.WORLD``,
    one rank per GPU).  Every rank then passes the same full batch, prices
    its contiguous share on its own GPU, and one all-gather of a small
    per-option record returns the whole batch, in order, on every rank
    (distributed.price_batch_sharded).  Because the kernel
    path depends only on block shapes, each price is bitwise the one a
    single GPU computes.
    """
    if group is not None:
        if dense_reference != "never":
            raise ValueError("the sharded batch pricer takes dense_reference='never'")
        from .distributed import price_batch_sharded
        return price_batch_sharded(models, grid, cfg_phi, cfg_v, t=t, group=group, raise_errors=raise_errors)
    for m in models:
        if m.d != grid.d:
            raise ValueError(f"model has d={m.d} but grid has d={grid.d}")
    _require_admissible(grid)
    shape = (grid.points_per_axis,) * grid.d
    # memory-aware batching: instances that do not fit one launch pair run in
    # consecutive chunks (results identical: instances are independent)
    chunk = balanced_chunk(len(models), max_batch(shape, cfg_phi, cfg_v, n=len(models)))
    if len(models) > chunk:
        out = []
        for i0 in range(0, len(models), chunk):
            out.extend(price_fourier_tt_batch(models[i0:i0 + chunk], grid, cfg_phi, cfg_v, t=t,
                                              dense_reference=dense_reference, term_cap=term_cap,
                                              raise_errors=raise_errors))
        return out
    start = time.perf_counter()
    phi_res, v_res = run_cross_pair(OracleBatch([PhiGridOracle(m, grid) for m in models]),
                                    OracleBatch([PayoffGridOracle(m, grid, conj=True) for m in models]),
                                    shape, cfg_phi, cfg_v)
    raw = tt_inner_batch(v_res.trains, phi_res.trains)
    wall = time.perf_counter() - start
    results = []
    dense = None
    if dense_reference == "auto" and grid.n_terms <= term_cap:
        dense = price_fourier_dense_batch(models, grid, t=t, term_cap=term_cap)
    for i, m in enumerate(models):
        err = phi_res.error_for(i) or v_res.error_for(i)
        if err is not None:
            if raise_errors:
                raise err
            results.append(err)
            continue
        value = _prefactor(m, grid, t) * raw[i]
        diag = {
            "cross_phi": phi_res.reports[i],
            "cross_v": v_res.reports[i],
            "imag_part": float(value.imag),
            "oracle_calls_total": phi_res.reports[i].oracle_calls + v_res.reports[i].oracle_calls,
        }
        if dense is not None:
            diag["dense_price"] = dense[i].price
            diag["eps_trunc"] = float(abs(value.real - dense[i].price) / abs(dense[i].price))
        results.append(PricingResult(float(value.real), "fourier_tt", wall / len(models), diag))
    return results


def price_fourier_tt_batch_capi(models, grid, cfg_phi, cfg_v, t=0.0):
    """price_fourier_tt_batch through the single C entry point
    ttp_price_tt_batch (both crosses, the inner product and the prefactor in
    one call) -- the binding a non-Python host would use.
    Same prices as price_fourier_tt_batch; returns a list of PricingResult."""
    from .cross import _finish_cross, _prepare_cross
    for m in models:
        if m.d != grid.d:
            raise ValueError(f"model has d={m.d} but grid has d={grid.d}")
    _require_admissible(grid)
    torch = _lib.require_device()
    lib = _lib.load_library()
    start = time.perf_counter()
    shape = (grid.points_per_axis,) * grid.d
    pp = _prepare_cross(OracleBatch([PhiGridOracle(m, grid) for m in models]), shape, cfg_phi)
    pv = _prepare_cross(OracleBatch([PayoffGridOracle(m, grid, conj=True) for m in models]), shape, cfg_v)
    pref = np.array([_prefactor(m, grid, t) for m in models], dtype=np.float64)
    prob = _lib.PriceProblem(phi=pp.prob, vhat=pv.prob,
                             h_prefactor=pref.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    ws_bytes = lib.ttp_price_tt_workspace(ctypes.byref(prob))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    n = len(models)
    price = np.zeros(n)
    imag = np.zeros(n)
    st = lib.ttp_price_tt_batch(ctypes.byref(prob), ctypes.byref(pp.out), ctypes.byref(pv.out),
                                price.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                imag.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                ctypes.c_void_p(ws.data_ptr()), ws_bytes, _lib.stream_handle())
    _lib.raise_for(st, "price_tt_batch")
    del ws
    rp, rv = _finish_cross(pp, True), _finish_cross(pv, True)
    wall = time.perf_counter() - start
    out = []
    for i in range(n):
        err = rp.error_for(i) or rv.error_for(i)
        if err is not None:
            raise err
        out.append(PricingResult(float(price[i]), "fourier_tt", wall / n, {
            "cross_phi": rp.reports[i], "cross_v": rv.reports[i], "imag_part": float(imag[i]),
            "oracle_calls_total": rp.reports[i].oracle_calls + rv.reports[i].oracle_calls}))
    return out


def price_fourier_tt(model, grid, cfg_phi, cfg_v, t=0.0, dense_reference="auto",
                     term_cap=DENSE_TERM_CAP):
    """Tensor-train contraction of the contour sum (pricers.py:256-294)."""
    if model.d != grid.d:
        raise ValueError(f"model has d={model.d} but grid has d={grid.d}")
    return price_fourier_tt_batch([model], grid, cfg_phi, cfg_v, t=t,
                                  dense_reference=dense_reference, term_cap=term_cap)[0]


def price_strike_ladder(model, grid, strikes, cfg_phi, cfg_v, t=0.0, dense_reference="never",
                        term_cap=DENSE_TERM_CAP, raise_errors=True):
    """Price one model at a ladder of strikes (the
    reference's run_strike_sweep, bench.py:478-510, calls price_fourier_tt
    once per strike).

    phi(-z) does not depend on the strike (pricers.py:234-240), and the
    reference's per-strike phi crosses all see the same oracle and the same
    CrossConfig, so they build the same train; here it is built ONCE and
    reused for every strike, while the strike-dependent payoff crosses run
    as one batch.  Each price therefore equals the per-strike
    price_fourier_tt price, at one phi cross instead of len(strikes).
    """
    from .market import MarketModel
    from .tensor_train import DeviceTTBatch
    if model.d != grid.d:
        raise ValueError(f"model has d={model.d} but grid has d={grid.d}")
    strikes = [float(k) for k in strikes]
    if not strikes:
        return []
    _require_admissible(grid)
    start = time.perf_counter()
    shape = (grid.points_per_axis,) * grid.d
    ladder = [MarketModel(r=model.r, sigma=model.sigma, T=model.T, s0=model.s0, strike=k,
                          corr=model.corr, rates=model.rates, d=model.d) for k in strikes]
    phi_res, v_res = run_cross_pair(OracleBatch([PhiGridOracle(model, grid)]),
                                    OracleBatch([PayoffGridOracle(m, grid, conj=True) for m in ladder]),
                                    shape, cfg_phi, cfg_v)
    n = len(strikes)
    err_phi = phi_res.error_for(0)
    if err_phi is not None:
        if raise_errors:
            raise err_phi
        return [err_phi] * n
    ph = phi_res.trains
    kets = DeviceTTBatch(ph.shape, ph.bonds, ph.flat[: ph.stride].repeat(n), n)
    raw = tt_inner_batch(v_res.trains, kets)
    wall = time.perf_counter() - start
    dense = None
    if dense_reference == "auto" and grid.n_terms <= term_cap:
        dense = price_fourier_dense_batch(ladder, grid, t=t, term_cap=term_cap)
    out = []
    for i, m in enumerate(ladder):
        err = v_res.error_for(i)
        if err is not None:
            if raise_errors:
                raise err
            out.append(err)
            continue
        value = _prefactor(m, grid, t) * raw[i]
        diag = {
            "strike": m.strike,
            "cross_phi": phi_res.reports[0],
            "cross_v": v_res.reports[i],
            "imag_part": float(value.imag),
            "oracle_calls_total": phi_res.reports[0].oracle_calls + v_res.reports[i].oracle_calls,
            "phi_shared": True,
        }
        if dense is not None:
            diag["dense_price"] = dense[i].price
            diag["eps_trunc"] = float(abs(value.real - dense[i].price) / abs(dense[i].price))
        out.append(PricingResult(float(value.real), "fourier_tt", wall / n, diag))
    return out
