"""Multi-process host logic of the multi-GPU sweep, on CPU with gloo
(world_size 2): set partitioning and the end-of-sweep row gather."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_22337_b200.distributed import gather_rows, partition


def test_partition_covers_every_set_once():
    for n in (0, 1, 7, 1024, 1023):
        for world in (1, 2, 3, 4, 8):
            spans = [partition(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = partition(n, world, rank)
        # rows carry their global set index so the gathered order is checkable
        local = torch.arange(lo, hi, dtype=torch.float64).reshape(-1, 1).repeat(1, 3)
        local[:, 1] = rank
        out = gather_rows(torch, dist, local, n, world, rank)
        ranks = torch.tensor([[rank, lo, hi]], dtype=torch.int64)
        if rank == 0:
            q.put(out.numpy().tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1024, 7])
def test_gather_rows_world2_gloo(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows = np.asarray(rows)
    assert rows.shape == (n, 3)
    assert rows[:, 0].tolist() == list(range(n))
    want_rank = [0 if i < partition(n, 2, 0)[1] else 1 for i in range(n)]
    assert rows[:, 1].astype(int).tolist() == want_rank
