"""Instance-level data parallelism across the GPUs of one box.

Options are independent, so a batch is sharded into contiguous instance
ranges (rank g gets [g*B/W, (g+1)*B/W)); each rank runs its
own batched TT-cross and there is no collective on the data path.  The only
exchange is one all-gather of a fixed-size per-option record at the end
(NCCL over NVLink on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np

RECORD_FIELDS = ("price", "imag", "status", "sweeps_phi", "sweeps_v", "calls_phi",
                 "calls_v", "diff_phi", "diff_v")


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
            out[i, 2] = 1.0
            continue
        cp, cv = res.diagnostics["cross_phi"], res.diagnostics["cross_v"]
        out[i] = (res.price, res.diagnostics["imag_part"], 0.0, cp.sweeps_used, cv.sweeps_used,
                  cp.oracle_calls, cv.oracle_calls, cp.final_diff, cv.final_diff)
    return out


def gather_records(local, n_total, device=None):
    """All-gather per-rank record blocks into the full (n_total, F) array.

    Uses torch.distributed with the process group already initialised
    (``nccl`` with CUDA tensors, ``gloo`` with CPU tensors).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    rank = dist.get_rank()
    width = local.shape[1]
    cap = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world))
    buf = np.zeros((cap, width))
    buf[: len(local)] = local
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    rows = []
    for r in range(world):
        lo, hi = shard_range(n_total, r, world)
        rows.append(parts[r].cpu().numpy()[: hi - lo])
    del rank
    return np.concatenate(rows, axis=0)


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
    device tt_cross / tt_inner (the CPU tests pass oracle restatements)."""
    import torch
    import torch.distributed as dist
    from .oracles import PayoffGridOracle, PhiGridOracle

    if dist.get_world_size() < 2:
        raise ValueError("price_fourier_tt_split2 needs at least two ranks")
    rank = dist.get_rank()
    shape = (grid.points_per_axis,) * grid.d
    if cross_fn is None:
        from .cross import tt_cross
        cross_fn = lambda o, s, c: tt_cross(o, s, c)[0]  # noqa: E731
    if inner_fn is None:
        from .tensor_train import tt_inner
        inner_fn = tt_inner
    price = torch.zeros(1, dtype=torch.float64, device=device if device is not None else "cpu")
    if rank == 0:
        phi = cross_fn(PhiGridOracle(model, grid), shape, cfg_phi)
        v = _recv_train(1, device)
        raw = inner_fn(v, phi)
        pref = np.exp(-model.r * (model.T - t)) * grid.eta ** grid.d / (2.0 * np.pi) ** grid.d
        price[0] = float((pref * raw).real)
    elif rank == 1:
        v = cross_fn(PayoffGridOracle(model, grid, conj=True), shape, cfg_v)
        _send_train(v, 0, device)
    dist.broadcast(price, 0)
    return float(price.item())
