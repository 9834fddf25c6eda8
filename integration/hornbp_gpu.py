"""The reference-side binding: what a hornbp maintainer adds as ``hornbp/_gpu.py``.

It keeps the reference package (its FactorGraph / Schedule / EngineOptions /
InferenceResult / UnderflowError objects) and swaps only the engine:
``run(graph, schedule, options)`` is ``hornbp.engine.run`` (engine.py:531-594)
executed by ``libhbp.so`` through the C ABI of include/hornbp_gpu.h -- plain
pointers and sizes, every argument and return type declared for ctypes.

    import hornbp
    from hornbp import _gpu                       # this file
    res = _gpu.run(graph, schedule, hornbp.EngineOptions(max_iterations=1000))

Errors map to the reference's exception types: HBP_EINVAL -> ValueError,
HBP_EUNDERFLOW -> hornbp.UnderflowError with the reference's message (the
index is the reference's own, engine.py:155-165, 512-518), HBP_ECYCLE ->
hornbp.ScheduleError, anything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HBP_OK, HBP_EINVAL, HBP_EUNDERFLOW, HBP_ECUDA, HBP_ECYCLE, HBP_ENOMEM = 0, 1, 2, 3, 5, 6

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HBP_LIB_PATH") or os.path.join(
    _HERE, "..", "paper_2509_22337_b200", "_lib", "libhbp.so")

i32p, i64p, f64p, i8p = (C.POINTER(t) for t in (C.c_int32, C.c_int64, C.c_double, C.c_int8))
vp = C.c_void_p


class GraphDesc(C.Structure):  # hbp_graph_desc
    _fields_ = [("num_variables", C.c_int32), ("num_factors", C.c_int32),
                ("num_edges", C.c_int64), ("factor_rowptr", i64p), ("edge_var", i32p),
                ("factor_kind", i8p), ("p1", f64p), ("p2", f64p)]


class Options(C.Structure):  # hbp_options
    _fields_ = [("max_iterations", C.c_int32), ("normalize_messages", C.c_int32),
                ("record_history", C.c_int32), ("evidence_count", C.c_int32),
                ("tolerance", C.c_double), ("time_limit", C.c_double),
                ("precision", C.c_int32)]


class Result(C.Structure):  # hbp_result
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("last_delta", C.c_double),
                ("underflow_kind", C.c_int32), ("underflow_iteration", C.c_int32),
                ("underflow_index", C.c_int64), ("device_ms", C.c_double),
                ("total_ms", C.c_double)]


SIGNATURES = {
    "hbp_graph_create": (C.c_int32, [C.POINTER(GraphDesc), C.c_int32, C.POINTER(vp)]),
    "hbp_graph_destroy": (None, [vp]),
    "hbp_plan_create": (C.c_int32, [vp, C.c_int64, i64p, i32p, i64p, i32p, C.POINTER(vp)]),
    "hbp_plan_destroy": (None, [vp]),
    "hbp_run": (C.c_int32, [vp, C.POINTER(Options), f64p, f64p, f64p, C.POINTER(Result)]),
    "hbp_graph_history": (C.c_int32, [vp, C.c_int32, f64p]),
    "hbp_last_error": (C.c_char_p, []),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _error(status: int, what: str, res: Result | None = None):
    import hornbp
    from hornbp.schedule import ScheduleError

    msg = lib().hbp_last_error().decode()
    if status == HBP_EUNDERFLOW and res is not None:
        k, i = res.underflow_kind, int(res.underflow_index)
        if k == 1:
            text = f"variable-to-factor message degenerated to zero mass at {i} (contradictory evidence?)"
        elif k == 2:
            text = f"factor-to-variable message degenerated to zero mass at {i} (contradictory evidence?)"
        else:
            text = f"marginal of variable {i} degenerated to zero mass (contradictory evidence?)"
        return hornbp.UnderflowError(text)
    if status == HBP_EINVAL:
        return ValueError(f"{what}: {msg}")
    if status == HBP_ECYCLE:
        return ScheduleError(f"{what}: {msg}")
    if status == HBP_ENOMEM:
        return MemoryError(f"{what}: {msg}")
    return RuntimeError(f"{what}: {msg}")


def _flat(graph):
    """hornbp FactorGraph -> canonical flat arrays (factor-major edges, graph.py:146-150)."""
    F = graph.num_factors
    deg = np.fromiter((1 + len(f.body) for f in graph.factors), dtype=np.int64, count=F)
    rowptr = np.zeros(F + 1, dtype=np.int64)
    np.cumsum(deg, out=rowptr[1:])
    var = np.fromiter((v for f in graph.factors for v in (f.head, *f.body)), dtype=np.int32,
                      count=int(rowptr[-1]))
    kind = np.fromiter((1 if f.kind.value == "OR" else 0 for f in graph.factors), dtype=np.int8,
                       count=F)
    p1 = np.fromiter((f.p1 for f in graph.factors), dtype=np.float64, count=F)
    p2 = np.fromiter((f.p2 for f in graph.factors), dtype=np.float64, count=F)
    return rowptr, var, kind, p1, p2


def _batches(rowptr, batches):
    off = np.zeros(len(batches) + 1, dtype=np.int64)
    np.cumsum([len(b) for b in batches], out=off[1:])
    idx = np.fromiter((rowptr[e.factor] + e.slot for b in batches for e in b), dtype=np.int32,
                      count=int(off[-1]))
    return off, idx


def run(graph, schedule, options=None, workers: int = 1, device: int = 0):
    """hornbp.engine.run (engine.py:531-594) on the GPU; returns hornbp.InferenceResult."""
    import hornbp

    options = options or hornbp.EngineOptions()
    options.validate()
    L = lib()
    rowptr, var, kind, p1, p2 = _flat(graph)
    desc = GraphDesc(graph.num_variables, len(kind), len(var), rowptr.ctypes.data_as(i64p),
                     var.ctypes.data_as(i32p), kind.ctypes.data_as(i8p),
                     p1.ctypes.data_as(f64p), p2.ctypes.data_as(f64p))
    g = vp()
    st = L.hbp_graph_create(C.byref(desc), device, C.byref(g))
    if st != HBP_OK:
        raise _error(st, "hbp_graph_create")
    p = vp()
    try:
        s_off, s_e = _batches(rowptr, schedule.s_batches)
        t_off, t_e = _batches(rowptr, schedule.t_batches)
        st = L.hbp_plan_create(g, len(schedule.s_batches), s_off.ctypes.data_as(i64p),
                               s_e.ctypes.data_as(i32p), t_off.ctypes.data_as(i64p),
                               t_e.ctypes.data_as(i32p), C.byref(p))
        if st != HBP_OK:
            raise _error(st, "hbp_plan_create")
        opt = Options(int(options.max_iterations), int(bool(options.normalize_messages)),
                      int(bool(options.record_history)), 0, float(options.tolerance),
                      float(options.time_limit) if options.time_limit else 0.0, 0)
        V = graph.num_variables
        marg = np.empty((V, 2), dtype=np.float64)
        deltas = np.empty(int(options.max_iterations), dtype=np.float64)
        res = Result()
        st = L.hbp_run(p, C.byref(opt), marg.ctypes.data_as(f64p), deltas.ctypes.data_as(f64p),
                       None, C.byref(res))
        if st != HBP_OK:
            raise _error(st, "hbp_run", res)
        n = res.iterations
        history = None
        if options.record_history:
            h = np.empty((n, V, 2), dtype=np.float64)
            st = L.hbp_graph_history(g, n, h.ctypes.data_as(f64p))
            if st != HBP_OK:
                raise _error(st, "hbp_graph_history")
            history = [h[i].copy() for i in range(n)]
        return hornbp.InferenceResult(marginals=marg, converged=bool(res.converged),
                                      iterations=n, last_delta=float(res.last_delta),
                                      deltas=deltas[:n].tolist(), history=history)
    finally:
        if p:
            L.hbp_plan_destroy(p)
        L.hbp_graph_destroy(g)
