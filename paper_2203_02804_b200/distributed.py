"""Instance-level data parallelism across the GPUs of one box.

Options are independent, so a batch is sharded into contiguous instance
ranges (rank g gets [g*B/W, (g+1)*B/W)); each rank runs its
own batched TT-cross and there is no collective on the data path.  The only
exchange is one all-gather of a fixed-size per-option record at the end
(NCCL over NVLink on GPUs, gloo in the CPU tests).  The library entry point
is ``price_fourier_tt_batch(..., group=...)`` (pricers.py), which lands in
:func:`price_batch_sharded`.
"""

from __future__ import annotations

import time

import numpy as np

from .errors import (CapacityError, DeviceError, MaxvolIterationError, OracleBudgetError, ResidueError,
                     SingularMatrixError)

RECORD_FIELDS = ("price", "imag", "status", "sweeps_phi", "sweeps_v", "calls_phi",
                 "calls_v", "diff_phi", "diff_v", "error_bond")

# record status codes: the C ABI's ttp_status values (include/ttpricer_b200.h)
_STATUS_OF = ((SingularMatrixError, 3), (MaxvolIterationError, 4), (OracleBudgetError, 5),
              (CapacityError, 6), (ResidueError, 8), (DeviceError, 2), (ValueError, 1))
_ERROR_OF = {3: SingularMatrixError, 4: MaxvolIterationError, 5: OracleBudgetError, 6: CapacityError,
             8: ResidueError, 2: DeviceError, 1: ValueError}


def _status_code(exc):
    for cls, code in _STATUS_OF:
        if isinstance(exc, cls):
            return code
    return 2


def shard_range(n_total, rank, world):
    """Contiguous [lo, hi) slice of ``n_total`` instances owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    lo = (rank * n_total) // world
    hi = ((rank + 1) * n_total) // world
    return lo, hi


def results_to_records(results):
    """PricingResult list (or exceptions) -> (n, len(RECORD_FIELDS)) float64."""
    out = np.full((len(results), len(RECORD_FIELDS)), np.nan)
    for i, res in enumerate(results):
        if isinstance(res, Exception):
            out[i, 2] = _status_code(res)
            out[i, 9] = -1 if getattr(res, "bond", None) is None else res.bond
            continue
        cp, cv = res.diagnostics["cross_phi"], res.diagnostics["cross_v"]
        out[i] = (res.price, res.diagnostics["imag_part"], 0.0, cp.sweeps_used, cv.sweeps_used,
                  cp.oracle_calls, cv.oracle_calls, cp.final_diff, cv.final_diff, -1)
    return out


def _default_device(group):
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return None


def gather_records(local, n_total, device=None, group=None):
    """All-gather per-rank record blocks into the full (n_total, F) array.

    Uses torch.distributed with the process group already initialised
    (``nccl`` with CUDA tensors, ``gloo`` with CPU tensors).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    width = local.shape[1]
    cap = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world))
    buf = np.zeros((max(cap, 1), width))
    buf[: len(local)] = local
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    rows = []
    for r in range(world):
        lo, hi = shard_range(n_total, r, world)
        rows.append(parts[r].cpu().numpy()[: hi - lo])
    return np.concatenate(rows, axis=0)


def record_to_result(rec, grid, cfg_phi, cfg_v, owner, wall):
    """A gathered record of another rank's option -> PricingResult (or the
    exception it raised there).  The reports carry the counters and
    convergence figures; the pivot sets stay on the owning rank."""
    from .cross import CrossReport
    from .pricers import PricingResult
    status = int(rec[2])
    if status != 0:
        cls = _ERROR_OF.get(status, DeviceError)
        msg = f"option failed on rank {owner} (status {status})"
        return cls(msg, bond=int(rec[9]) if rec[9] >= 0 else None) if cls is SingularMatrixError else cls(msg)

    def rep(sweeps, calls, diff, cfg):
        sweeps, calls = int(sweeps), int(calls)
        return CrossReport(converged=bool(diff <= cfg.eps_tol), sweeps_used=sweeps, oracle_calls=calls,
                           conv_check_calls=sweeps * cfg.n_conv_samples, final_diff=float(diff),
                           compression_ratio=calls / grid.n_terms)
    rp = rep(rec[3], rec[5], rec[7], cfg_phi)
    rv = rep(rec[4], rec[6], rec[8], cfg_v)
    return PricingResult(float(rec[0]), "fourier_tt", wall, {
        "cross_phi": rp, "cross_v": rv, "imag_part": float(rec[1]),
        "oracle_calls_total": rp.oracle_calls + rv.oracle_calls, "rank": owner})


def price_batch_sharded(models, grid, cfg_phi, cfg_v, t=0.0, group=None, raise_errors=True,
                        local_pricer=None, device=None):
    """Price a batch across the ranks of ``group``.

    Every rank passes the SAME full ``models`` list.  Rank g prices the
    contiguous range [g*B/W, (g+1)*B/W) with the device pricer, then one
    all-gather of a RECORD_FIELDS record per option (NCCL over NVLink when
    the group's backend is nccl) gives every rank the whole batch in input
    order: its own options as full PricingResults, the others' rebuilt from
    their records (reports without pivot sets, diagnostics["rank"] = owner).
    Per-option errors travel in the record, so a failure on one rank is seen
    -- and raised, if ``raise_errors`` -- on every rank after the collective,
    never leaving a peer blocked in it.  ``local_pricer`` (same signature as
    price_fourier_tt_batch) replaces the device pricer in the CPU tests."""
    import torch.distributed as dist
    if local_pricer is None:
        from .pricers import price_fourier_tt_batch as local_pricer
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = len(models)
    lo, hi = shard_range(n, rank, world)
    start = time.perf_counter()
    local = []
    if hi > lo:
        try:
            local = local_pricer(models[lo:hi], grid, cfg_phi, cfg_v, t=t, raise_errors=False)
        except Exception as exc:  # a whole-shard failure still joins the collective
            local = [exc] * (hi - lo)
    full = gather_records(results_to_records(local), n,
                          device=device if device is not None else _default_device(group), group=group)
    wall = (time.perf_counter() - start) / max(1, n)
    out = []
    for i in range(n):
        if lo <= i < hi:
            out.append(local[i - lo])
        else:
            owner = next(r for r in range(world) if shard_range(n, r, world)[0] <= i < shard_range(n, r, world)[1])
            out.append(record_to_result(full[i], grid, cfg_phi, cfg_v, owner, wall))
    if raise_errors:
        for res in out:
            if isinstance(res, Exception):
                raise res
    return out


def combine_partials(local, device=None):
    """All-gather one complex partial per rank and sum them in rank order
    (fixed order: every rank gets the same bits; an all_reduce's order is
    the library's choice)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    t = torch.tensor([complex(local).real, complex(local).imag], dtype=torch.float64)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    acc = 0j
    for p in parts:
        v = p.cpu().numpy()
        acc += complex(v[0], v[1])
    return acc


def dense_contour_sum_sharded(model, grid, partial_fn=None, device=None):
    """Dense cross-check sum over the full grid sharded by flat C-order index
    range across the ranks of the default process group:
    rank g sums terms [g T / W, (g+1) T / W) with ttp_dense_sum_range and the
    partials combine in rank order.  ``partial_fn(model, grid, first, count)``
    overrides the per-rank device sum (the CPU tests use the oracle)."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    lo, hi = shard_range(grid.n_terms, rank, world)
    if partial_fn is None:
        from .pricers import dense_partial_sum
        partial_fn = dense_partial_sum
    return combine_partials(partial_fn(model, grid, lo, hi - lo), device=device)


def _send_train(tt, dst, device=None):
    import torch
    import torch.distributed as dist
    meta = np.array([len(tt.cores)] + [c.shape[0] for c in tt.cores] + [tt.cores[-1].shape[2]]
                    + [c.shape[1] for c in tt.cores], dtype=np.int64)
    m = torch.from_numpy(np.concatenate([[len(meta)], meta]).astype(np.int64))
    flat = torch.from_numpy(np.concatenate([c.ravel() for c in tt.cores]).view(np.float64))
    if device is not None:
        m, flat = m.to(device), flat.to(device)
    dist.send(torch.tensor([m.numel()], dtype=torch.int64, device=m.device), dst)
    dist.send(m, dst)
    dist.send(flat, dst)


def _recv_train(src, device=None):
    import torch
    import torch.distributed as dist
    from .tensor_train import TensorTrain
    dev = device if device is not None else torch.device("cpu")
    n = torch.empty(1, dtype=torch.int64, device=dev)
    dist.recv(n, src)
    m = torch.empty(int(n.item()), dtype=torch.int64, device=dev)
    dist.recv(m, src)
    meta = m.cpu().numpy()[1:]
    d = int(meta[0])
    bonds = meta[1:d + 2]
    phys = meta[d + 2:2 * d + 2]
    size = int(sum(bonds[k] * phys[k] * bonds[k + 1] for k in range(d)))
    flat = torch.empty(2 * size, dtype=torch.float64, device=dev)
    dist.recv(flat, src)
    z = flat.cpu().numpy().view(np.complex128)
    cores, off = [], 0
    for k in range(d):
        cnt = int(bonds[k] * phys[k] * bonds[k + 1])
        cores.append(z[off:off + cnt].reshape(int(bonds[k]), int(phys[k]), int(bonds[k + 1])))
        off += cnt
    return TensorTrain(cores)


def price_fourier_tt_split2(model, grid, cfg_phi, cfg_v, t=0.0, cross_fn=None, inner_fn=None, device=None):
    """One option on two ranks (optional split): the phi and
    vhat crosses are independent (pricers.py:271-272), so rank 0 builds the
    phi train while rank 1 builds the vhat train; rank 1 ships its cores to
    rank 0 (point-to-point, NVLink under NCCL), rank 0 contracts them and the
    price is broadcast.  Returns the price on every rank.  ``cross_fn(oracle,
    shape, cfg) -> TensorTrain`` and ``inner_fn(bra, ket)`` default to the
    device tt_cross / tt_inner (the CPU tests pass oracle restatements).

    ``device`` defaults to the current CUDA device under an NCCL group (the
    cores then move GPU to GPU) and to the host under gloo.  Before any core
    moves, both ranks exchange a status word: if either cross raised, every
    rank raises (the same exception class) instead of blocking in a send or
    receive its peer will never post."""
    import torch
    import torch.distributed as dist
    from .oracles import PayoffGridOracle, PhiGridOracle

    if dist.get_world_size() < 2:
        raise ValueError("price_fourier_tt_split2 needs at least two ranks")
    rank = dist.get_rank()
    if device is None:
        device = _default_device(None)
    dev = device if device is not None else torch.device("cpu")
    shape = (grid.points_per_axis,) * grid.d
    if cross_fn is None:
        from .cross import tt_cross
        cross_fn = lambda o, s, c: tt_cross(o, s, c)[0]  # noqa: E731
    if inner_fn is None:
        from .tensor_train import tt_inner
        inner_fn = tt_inner
    train, err = None, None
    if rank in (0, 1):
        try:
            if rank == 0:
                train = cross_fn(PhiGridOracle(model, grid), shape, cfg_phi)
            else:
                train = cross_fn(PayoffGridOracle(model, grid, conj=True), shape, cfg_v)
        except Exception as exc:  # reported to the peer before re-raising
            err = exc
    code = torch.tensor([_status_code(err) if err is not None else 0], dtype=torch.int64, device=dev)
    codes = [torch.empty_like(code) for _ in range(dist.get_world_size())]
    dist.all_gather(codes, code)
    codes = [int(c.item()) for c in codes]
    if err is not None:
        raise err
    for r in (0, 1):
        if codes[r] != 0:
            raise _ERROR_OF.get(codes[r], DeviceError)(f"the {'phi' if r == 0 else 'vhat'} cross failed on rank {r}")
    price = torch.zeros(1, dtype=torch.float64, device=dev)
    if rank == 0:
        v = _recv_train(1, device)
        raw = inner_fn(v, train)
        pref = np.exp(-model.r * (model.T - t)) * grid.eta ** grid.d / (2.0 * np.pi) ** grid.d
        price[0] = float((pref * raw).real)
    elif rank == 1:
        _send_train(train, 0, device)
    dist.broadcast(price, 0)
    return float(price.item())
