"""The multi-GPU sweep path end to end on one GPU: two ranks share cuda:0
over gloo (NCCL refuses two ranks on one device), each runs its slice of the
evidence sets with run_many_distributed, and rank 0's gathered outputs must
equal a single-rank run_many of all sets bit for bit (the
sets are independent, so sharding changes nothing)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_SETS = 71  # uneven per-rank slices for both world sizes


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sets(alarms, n):
    from paper_2509_22337_b200 import workloads as W
    return [W.evidence_set(alarms, j) for j in range(n)]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2509_22337_b200 as P
    from paper_2509_22337_b200 import distributed as D
    from paper_2509_22337_b200 import workloads as W

    torch.cuda.set_device(0)
    P.engine.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, alarms = W.graph("hedc")
        sel = np.sort(np.asarray(alarms.alarms, dtype=np.int32))
        out = D.run_many_distributed(g, _sets(alarms, N_SETS), P.EngineOptions(1000, 1e-9),
                                     select=sel, topk=50)
        if rank == 0:
            q.put((out.iterations.tolist(), out.converged.tolist(), out.last_delta.tobytes(),
                   out.p1_select.tobytes(), out.ranked.tolist(), out.failed.tolist(),
                   int(out.total_updates())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_run_many_distributed_equals_single_rank(world):
    import torch.multiprocessing as mp

    import paper_2509_22337_b200 as P
    from paper_2509_22337_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    it, conv, last, p1, ranked, failed, upd = got

    g, alarms = W.graph("hedc")
    sel = np.sort(np.asarray(alarms.alarms, dtype=np.int32))
    ref = P.run_many(g, _sets(alarms, N_SETS), None, P.EngineOptions(1000, 1e-9),
                     marginals=False, deltas=False, select=sel, topk=50)
    assert it == ref.iterations.tolist()
    assert conv == ref.converged.tolist()
    assert last == ref.last_delta.tobytes()
    assert p1 == ref.p1_select.tobytes()
    assert ranked == ref.ranked.tolist()
    assert not any(failed)
    assert upd == ref.total_updates()
