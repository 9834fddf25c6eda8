"""TEST INFRASTRUCTURE -- ctypes wrapper of the C oracle (oracle/lbp_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this module, and only as the checker /
CPU baseline. The product package never imports it.

``run(graph, schedule_arrays, ...)`` restates ``hornbp.engine.run`` bit for
bit (pinned against the reference and tests/golden/ by tests/test_oracle.py).
``graph`` is anything with the flat-array attributes of
``paper_2509_22337_b200.graph.FactorGraph`` (num_variables, rowptr, vars,
kind, p1, p2).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liborc.so")


class OrcResult(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("last_delta", C.c_double),
        ("underflow_kind", C.c_int32),
        ("underflow_iteration", C.c_int32),
        ("underflow_index", C.c_int64),
    ]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(
                os.path.join(HERE, "lbp_oracle.c")):
            build()
        L = C.CDLL(LIB)
        P = C.POINTER
        L.orc_run.restype = C.c_int
        L.orc_run.argtypes = [C.c_int64, C.c_int64, C.c_int64, P(C.c_int64), P(C.c_int32),
                              P(C.c_int8), P(C.c_double), P(C.c_double), C.c_int64,
                              P(C.c_int64), P(C.c_int32), P(C.c_int64), P(C.c_int32), C.c_int32,
                              C.c_double, C.c_int32, C.c_int32, P(C.c_double), P(C.c_double),
                              P(OrcResult)]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def run(graph, arrays, max_iterations: int = 1000, tolerance: float = 1e-9,
        normalize: bool = True, threads: int = 1) -> dict:
    """Returns dict(marginals, deltas, iterations, converged, last_delta,
    underflow=(kind, iteration, index) or None)."""
    s_off, s_e, t_off, t_e = (np.ascontiguousarray(a) for a in arrays)
    s_off = s_off.astype(np.int64)
    t_off = t_off.astype(np.int64)
    s_e = s_e.astype(np.int32)
    t_e = t_e.astype(np.int32)
    rowptr = np.ascontiguousarray(graph.rowptr, dtype=np.int64)
    ev = np.ascontiguousarray(graph.vars, dtype=np.int32)
    kind = np.ascontiguousarray(graph.kind, dtype=np.int8)
    p1 = np.ascontiguousarray(graph.p1, dtype=np.float64)
    p2 = np.ascontiguousarray(graph.p2, dtype=np.float64)
    V = int(graph.num_variables)
    marg = np.empty((V, 2), dtype=np.float64)
    deltas = np.empty(max_iterations, dtype=np.float64)
    res = OrcResult()
    st = lib().orc_run(V, len(kind), len(ev), _p(rowptr, C.c_int64), _p(ev, C.c_int32),
                       _p(kind, C.c_int8), _p(p1, C.c_double), _p(p2, C.c_double),
                       len(s_off) - 1, _p(s_off, C.c_int64), _p(s_e, C.c_int32),
                       _p(t_off, C.c_int64), _p(t_e, C.c_int32), int(max_iterations),
                       float(tolerance), int(bool(normalize)), int(threads),
                       _p(marg, C.c_double), _p(deltas, C.c_double), C.byref(res))
    if st not in (0, 2):
        raise MemoryError("oracle allocation failed")
    n = res.iterations
    return dict(marginals=marg, deltas=deltas[:n].copy(), iterations=n,
                converged=bool(res.converged), last_delta=res.last_delta,
                underflow=None if st == 0 else (res.underflow_kind, res.underflow_iteration,
                                                res.underflow_index))


# ---- restatements used by the reference arm of bench.py (sweep sets) ---------------------

class FlatGraph:
    """Plain-array factor graph (the attributes orc.run reads)."""

    def __init__(self, num_variables, rowptr, vars_, kind, p1, p2):
        self.num_variables = int(num_variables)
        self.rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        self.vars = np.ascontiguousarray(vars_, dtype=np.int32)
        self.kind = np.ascontiguousarray(kind, dtype=np.int8)
        self.p1 = np.ascontiguousarray(p1, dtype=np.float64)
        self.p2 = np.ascontiguousarray(p2, dtype=np.float64)


def clamp(graph, ids, labels) -> FlatGraph:
    """clamp_evidence applied in order (graph.py:189-200): one appended
    body-empty AND factor per observation, p1 = p2 = 1.0 (true) / 0.0 (false)."""
    ids = np.asarray(ids, dtype=np.int64)
    p = np.where(np.asarray(labels, dtype=bool), 1.0, 0.0)
    n = len(ids)
    rp = np.asarray(graph.rowptr, dtype=np.int64)
    return FlatGraph(graph.num_variables,
                     np.concatenate([rp, rp[-1] + 1 + np.arange(n, dtype=np.int64)]),
                     np.concatenate([np.asarray(graph.vars, dtype=np.int32), ids.astype(np.int32)]),
                     np.concatenate([np.asarray(graph.kind, dtype=np.int8), np.zeros(n, np.int8)]),
                     np.concatenate([np.asarray(graph.p1, dtype=np.float64), p]),
                     np.concatenate([np.asarray(graph.p2, dtype=np.float64), p]))


def parall_arrays(graph):
    """Strategy.parall().compile(graph) as arrays: one batch, s_0 = every edge
    in ascending EdgeId (schedule.py:271-272, the toposort of the empty
    relation), t_0 = every slot of a non-unary factor (schedule.py:293-312)."""
    rp = np.asarray(graph.rowptr, dtype=np.int64)
    E = int(rp[-1])
    deg = np.diff(rp)
    s_e = np.arange(E, dtype=np.int32)
    t_e = np.flatnonzero(np.repeat(deg > 1, deg)).astype(np.int32)
    return (np.array([0, E], dtype=np.int64), s_e, np.array([0, len(t_e)], dtype=np.int64), t_e)
