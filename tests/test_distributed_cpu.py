"""Multi-rank sharding + result gather, world_size 2 over gloo on the CPU.

The GPU path is identical except for the backend (nccl) and the tensors'
device: each rank prices its contiguous shard, then one all-gather of the
per-option records.  Here each rank "prices" its shard with the CPU oracle's
dense sum on a tiny grid so the gathered values can be checked exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2203_02804_b200.distributed import RECORD_FIELDS, gather_records, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dense_value(i):
    from oracle import ttp_oracle as O
    from paper_2203_02804_b200 import configs
    m = configs.make_model(3, i)
    gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, 4, 0.3, 1.0)
    return O.price_dense(gm)


def _worker(rank, world, port, n_total, out_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(n_total, rank, world)
    local = np.zeros((hi - lo, len(RECORD_FIELDS)))
    for j, i in enumerate(range(lo, hi)):
        local[j, 0] = _dense_value(i)
        local[j, 2] = rank
    full = gather_records(local, n_total)
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [5, 8])
def test_gloo_world2_gather(tmp_path, n_total):
    out = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), n_total, out), nprocs=2, join=True)
    full = np.load(out)
    assert full.shape == (n_total, len(RECORD_FIELDS))
    want = np.array([_dense_value(i) for i in range(n_total)])
    np.testing.assert_array_equal(full[:, 0], want)
    owners = [0] * (n_total // 2) + [1] * (n_total - n_total // 2)
    np.testing.assert_array_equal(full[:, 2], owners)


def test_shard_ranges_partition():
    for n in (0, 1, 7, 1024, 4096):
        for w in (1, 2, 4, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
