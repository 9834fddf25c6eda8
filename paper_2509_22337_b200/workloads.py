"""The BASELINE.json configurations as reproducible workloads.

Each builder returns the synthetic graph from the reference generator specs
(pinned by sha256 of ``to_fastfg()`` in tests/test_synth.py), its alarms, the
strategy and the engine options the configuration is quoted on.

  C1 weblech  SynthSpec(313, 383, 8, 0)        PARALL, fixed 100 iterations
  C2 hedc     SynthSpec(1657, 3690, 8, 25)     SEQFIX over a default_rng(1234)
                                               permutation of the edges (k=224), tol 1e-9
  C3 avrora   SynthSpec(9424, 26667, 8, 3)     static residual-order SEQFIX (k=303), tol 1e-6
  C4 ftp      SynthSpec(101583, 109592, 8, 0)  PARALL (k=1) / canonical SEQFIX (k=476), tol 1e-9
  C5 ftp      C4 graph + evidence set j: default_rng(j).choice(#alarms, 8) sorted,
              clamped to the ground-truth labels; PARALL, tol 1e-9
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache
from typing import Optional

import numpy as np

from .graph import FactorGraph
from .ranking import AlarmSet
from .schedule import Strategy
from .synth import SynthSpec, generate

SPECS = {
    "weblech": SynthSpec(313, 383, 8, 0),
    "hedc": SynthSpec(1657, 3690, 8, 25),
    "avrora": SynthSpec(9424, 26667, 8, 3),
    "ftp": SynthSpec(101583, 109592, 8, 0),
}

# sha256(graph.to_fastfg())[:16] from the reference generator (numpy 2.3.5)
FASTFG_SHA = {
    "weblech": "7d0b8c9fca2eea16",
    "hedc": "126332fbae77deac",
    "avrora": "1c956889959b0dab",
    "ftp": "20f7a690d8bc209b",
}


@dataclass
class Workload:
    name: str
    graph: FactorGraph
    alarms: AlarmSet
    strategy: Strategy
    max_iterations: int
    tolerance: float


@lru_cache(maxsize=8)
def graph(name: str) -> tuple[FactorGraph, AlarmSet]:
    return generate(SPECS[name])


def residual_order(g: FactorGraph) -> np.ndarray:
    """C3's static residual priority: one PARALL iteration
    from uniform, r_e = |mu1/(mu0+mu1) after - before| per factor-to-variable
    message, edges sorted by (-r_e, edge id). Computed with the device
    single-pass kernels (bitwise equal to the reference engine)."""
    from .engine import update_ftov_batch, update_vtof_batch
    from .storage import initialize
    from .schedule import Strategy as S

    sched = S.parall().compile(g)
    s_off, s_e, t_off, t_e = sched.arrays(g)
    store = initialize(g)
    before = store.ftov1 / (store.ftov0 + store.ftov1)
    update_vtof_batch(store, g.edges_at(t_e))
    update_ftov_batch(store, g.edges_at(s_e))
    after = store.ftov1 / (store.ftov0 + store.ftov1)
    r = np.abs(after - before)                 # per ftov position
    r_edge = r[store.vtof_to_ftov]             # per canonical edge
    return np.lexsort((np.arange(g.num_edges), -r_edge))


def build(name: str) -> Workload:
    if name == "C1":
        g, a = graph("weblech")
        return Workload(name, g, a, Strategy.parall(), 100, 0.0)
    if name == "C2":
        g, a = graph("hedc")
        perm = np.random.default_rng(1234).permutation(g.num_edges)
        return Workload(name, g, a, Strategy.seqfix(g.edges_at(perm)), 1000, 1e-9)
    if name == "C2-canonical":
        g, a = graph("hedc")
        return Workload(name, g, a, Strategy.seqfix(), 1000, 1e-9)
    if name == "C3":
        g, a = graph("avrora")
        return Workload(name, g, a, Strategy.seqfix(g.edges_at(residual_order(g))), 1000, 1e-6)
    if name == "C4-PARALL":
        g, a = graph("ftp")
        return Workload(name, g, a, Strategy.parall(), 1000, 1e-9)
    if name == "C4-SEQFIX":
        g, a = graph("ftp")
        return Workload(name, g, a, Strategy.seqfix(), 1000, 1e-9)
    raise KeyError(name)


def evidence_set(alarms: AlarmSet, j: int, size: int = 8) -> tuple[np.ndarray, np.ndarray]:
    """C5 evidence set j: (variables, observed labels), variables ascending
    by alarm position."""
    rng = np.random.default_rng(j)
    pick = np.sort(rng.choice(len(alarms), size, replace=False))
    ids = np.asarray(alarms.alarms, dtype=np.int64)[pick]
    labels = np.asarray(alarms.labels, dtype=bool)[pick]
    return ids, labels


def clamped_graph(g: FactorGraph, ids, labels) -> FactorGraph:
    from .graph import clamp_evidence

    out = g
    for v, lab in zip(np.asarray(ids).tolist(), np.asarray(labels).tolist()):
        out = clamp_evidence(out, int(v), bool(lab))
    return out
