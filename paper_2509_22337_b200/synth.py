"""Deterministic synthetic derivation graphs (the BASELINE fixtures).

Produces the same (graph, alarms) as the reference generator
(``hornbp/synth.py:69-121``) for every ``SynthSpec``: the numpy ``Generator``
must be consumed call-for-call the same way (scalar ``integers`` for extra
conclusions, one ``geometric`` per clause, batched ``integers`` inside the
distinct sampler), because numpy's bounded-integer stream differs between a
size-1 call and a size-n call. The graph itself is emitted straight into the
flat-array form (``FactorGraph.from_arrays``) instead of via string-keyed DAG
nodes; ``tests/test_synth.py`` pins ``sha256(to_fastfg())`` for the four
BASELINE scales against the reference's output.

Variable numbering (= factor numbering, one factor per node) follows the
reference DAG conversion: tuples ``0..T-1`` (inputs first), then clauses
``T..T+C-1``; clause ``k`` is the k-th clause in sorted-conclusion order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import KIND_AND, KIND_OR, FactorGraph
from .ranking import AlarmSet


class SynthError(ValueError):
    """Infeasible generator parameters."""


@dataclass(frozen=True)
class SynthSpec:
    num_tuples: int
    num_clauses: int
    max_premises: int = 8
    seed: int = 0
    tree_only: bool = False
    clause_prob: float = 0.999

    def validate(self) -> None:
        """Same feasibility rules and messages as ``synth.py:33-50``."""
        t, c = self.num_tuples, self.num_clauses
        if t < 1:
            raise SynthError("clauses with zero tuples are infeasible" if c > 0
                             else "need at least one tuple")
        if c < 0:
            raise SynthError("clause count must be nonnegative")
        if c > 0 and t < 2:
            raise SynthError("clauses need at least two tuples (premise + conclusion)")
        if self.max_premises < 1:
            raise SynthError("max_premises must be at least 1")
        if self.tree_only and c > t - 1:
            raise SynthError("tree mode needs num_clauses <= num_tuples - 1 "
                             "(one clause derives one tuple from one premise)")
        if not 0.0 < self.clause_prob <= 1.0:
            raise SynthError("clause_prob must be in (0, 1]")


def _draw_distinct(rng: np.random.Generator, upper: int, count: int) -> list[int]:
    """``count`` distinct values from ``range(upper)`` in first-seen order;
    consumes the stream like ``synth.py:53-66`` (batched redraws of the
    shortfall, stop mid-batch once full)."""
    if count >= upper:
        return list(range(upper))
    out: list[int] = []
    have: set[int] = set()
    while len(out) < count:
        for v in rng.integers(0, upper, size=count - len(out)).tolist():
            if v in have:
                continue
            have.add(v)
            out.append(v)
            if len(out) == count:
                break
    return out


def generate(spec: SynthSpec) -> tuple[FactorGraph, AlarmSet]:
    """(graph, alarms) for ``spec``; alarms are a quarter of the sink tuples
    (at least one) with random ground-truth labels."""
    spec.validate()
    rng = np.random.default_rng(spec.seed)
    n_t, n_c = spec.num_tuples, spec.num_clauses
    derived = n_c if spec.tree_only else min(n_c, n_t - max(1, n_t // 3))
    n_in = n_t - derived

    # Every derived tuple gets one clause; surplus clauses re-derive a
    # random derived tuple (scalar draws, one per surplus clause).
    extra = [int(rng.integers(0, derived)) for _ in range(n_c - derived)]
    targets = np.sort(np.concatenate([np.arange(derived, dtype=np.int64),
                                      np.asarray(extra, dtype=np.int64)]))

    premises: list[list[int]] = []
    consumed = np.zeros(n_t, dtype=bool)
    for target in targets.tolist():
        pool = n_in + target
        if spec.tree_only:
            count = 1
        else:
            count = min(int(rng.geometric(0.7)), spec.max_premises, pool)
        chosen = _draw_distinct(rng, pool, count)
        premises.append(chosen)
        consumed[chosen] = True

    n_v = n_t + n_c
    p = spec.clause_prob
    kind = np.empty(n_v, dtype=np.int8)
    p1 = np.empty(n_v)
    p2 = np.empty(n_v)
    kind[:n_t] = KIND_OR
    kind[:n_in] = KIND_AND
    kind[n_t:] = KIND_AND
    p1[:n_in], p2[:n_in] = p, p          # input priors
    p1[n_in:n_t], p2[n_in:n_t] = 1.0, 0.0  # tuple OR over deriving clauses
    p1[n_t:], p2[n_t:] = p, 0.0          # clause AND over premises

    # Bodies: derived tuple (n_in + t) <- clauses deriving t, in clause order;
    # clause k <- its premises in draw order.
    first = np.searchsorted(targets, np.arange(derived), side="left")
    last = np.searchsorted(targets, np.arange(derived), side="right")
    degree = np.ones(n_v, dtype=np.int64)
    degree[n_in:n_t] += last - first
    degree[n_t:] += np.fromiter((len(x) for x in premises), dtype=np.int64, count=n_c)
    rowptr = np.zeros(n_v + 1, dtype=np.int64)
    np.cumsum(degree, out=rowptr[1:])
    flat = np.empty(int(rowptr[-1]), dtype=np.int64)
    flat[rowptr[:-1]] = np.arange(n_v)
    # derived tuples: clause ids are contiguous runs of the sorted targets
    if n_c:
        k = np.arange(n_c)
        flat[rowptr[n_in + targets] + 1 + (k - first[targets])] = n_t + k
    body_start = rowptr[n_t:-1] + 1
    if n_c:
        flat_premises = np.fromiter((v for x in premises for v in x), dtype=np.int64,
                                    count=int(degree[n_t:].sum() - n_c))
        pos = np.repeat(body_start, degree[n_t:] - 1) + (
            np.arange(len(flat_premises)) - np.repeat(np.cumsum(degree[n_t:] - 1) - (degree[n_t:] - 1),
                                                     degree[n_t:] - 1))
        flat[pos] = flat_premises
    names = [f"t{i}" for i in range(n_t)] + [f"c{k}" for k in range(n_c)]
    graph = FactorGraph.from_arrays(n_v, kind, p1, p2, rowptr, flat, names)

    sinks = np.flatnonzero(~consumed).tolist() or [n_t - 1]
    n_alarm = max(1, len(sinks) // 4)
    alarms = sorted(sinks[i] for i in _draw_distinct(rng, len(sinks), n_alarm))
    labels = rng.integers(0, 2, size=len(alarms)).astype(bool)
    return graph, AlarmSet(tuple(alarms), tuple(bool(b) for b in labels))
