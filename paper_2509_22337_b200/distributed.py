"""Multi-GPU multi-evidence sweep: one process per GPU, sets sharded across
ranks, one NCCL gather at the end.

Each evidence set is an independent ``run`` from uniform messages
(ranking.py:122-123), so rank r takes the contiguous slice
``partition(n, world, r)`` of the sets, runs it with ``run_many`` on its own
GPU -- graph layout replicated, no per-iteration collective -- and the
per-set outputs (iterations, convergence, last delta, P1 of the selected
variables, the device top-k ranking) are gathered to rank 0 with a single
``all_gather_into_tensor`` per output (NCCL over NVLink; gloo on CPU in the
tests). The device outputs land directly in the tensors that are gathered:
no staging copy between the sweep and the collective.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np


def partition(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n sets for ``rank``."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad partition arguments")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class GatheredSweep:
    """Rank 0's view of the whole sweep (sets in global order)."""

    iterations: np.ndarray
    converged: np.ndarray
    last_delta: np.ndarray
    updates_per_iteration: np.ndarray
    p1_select: Optional[np.ndarray]
    ranked: Optional[np.ndarray]
    failed: np.ndarray                     # per-set underflow flag

    def total_updates(self) -> int:
        return int(np.dot(self.updates_per_iteration.astype(np.int64),
                          self.iterations.astype(np.int64)))


def gather_rows(torch, dist, local, n_total: int, world: int, rank: int, group=None):
    """All-gather a [n_local, ...] tensor whose rows are this rank's slice of
    ``partition(n_total, world, .)`` into the [n_total, ...] global tensor
    (rows padded to the largest slice for the collective, then compacted)."""
    counts = [partition(n_total, world, r)[1] - partition(n_total, world, r)[0]
              for r in range(world)]
    mx = max(counts) if counts else 0
    tail = tuple(local.shape[1:])
    if all(c == mx for c in counts):  # even split (1,024 sets on 1/2/4/8 GPUs): no padding copy
        out = torch.empty((world * mx,) + tail, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out
    padded = torch.zeros((mx,) + tail, dtype=local.dtype, device=local.device)
    if local.shape[0]:
        padded[: local.shape[0]] = local
    out = torch.empty((world * mx,) + tail, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    if all(c == mx for c in counts):
        return out
    parts = [out[r * mx: r * mx + counts[r]] for r in range(world)]
    return torch.cat(parts, dim=0)


def run_many_distributed(graph, evidence_sets: Sequence, options=None, *,
                         select: Optional[Sequence[int]] = None, topk: int = 0,
                         group=None, capacity: int = 0, return_local: bool = False):
    """Shard ``evidence_sets`` over the ranks of ``group`` (one GPU each, the
    current CUDA device), run them, gather to every rank's device and return
    the host copy on rank 0 (None elsewhere). PARALL only."""
    import torch
    import torch.distributed as dist

    from .engine import device_graph
    from .sweep import run_many

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(evidence_sets)
    lo, hi = partition(n, world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    sel = None if select is None else np.ascontiguousarray(np.asarray(select, dtype=np.int32))
    nsel = 0 if sel is None else len(sel)
    m = hi - lo
    p1 = torch.empty((m, max(nsel, 1)), dtype=torch.float64, device=dev)
    rk = torch.empty((m, max(topk, 1)), dtype=torch.int32, device=dev)
    device_out = {}
    if nsel:
        device_out["p1_select"] = p1
    if topk:
        device_out["ranked"] = rk
    dg = device_graph(graph)
    dg.set_stream(torch.cuda.current_stream(dev))
    try:
        local = run_many(graph, evidence_sets[lo:hi], None, options, marginals=False,
                         deltas=False, select=sel, topk=topk, capacity=capacity,
                         device_out=device_out)
    finally:
        dg.set_stream(None)
    stats = torch.tensor(np.stack([local.iterations.astype(np.float64),
                                   local.converged.astype(np.float64),
                                   local.last_delta,
                                   local.updates_per_iteration.astype(np.float64),
                                   np.array([e is not None for e in local.errors], dtype=np.float64)],
                                  axis=1) if m else np.zeros((0, 5)),
                         dtype=torch.float64, device=dev)
    g_stats = gather_rows(torch, dist, stats, n, world, rank, group)
    g_p1 = gather_rows(torch, dist, p1, n, world, rank, group) if nsel else None
    g_rk = gather_rows(torch, dist, rk, n, world, rank, group) if topk else None
    if rank != 0:
        return local if return_local else None
    st = g_stats.cpu().numpy()
    out = GatheredSweep(
        iterations=st[:, 0].astype(np.int32), converged=st[:, 1] != 0, last_delta=st[:, 2],
        updates_per_iteration=st[:, 3].astype(np.int64), failed=st[:, 4] != 0,
        p1_select=None if g_p1 is None else g_p1.cpu().numpy(),
        ranked=None if g_rk is None else g_rk.cpu().numpy())
    return (out, local) if return_local else out
