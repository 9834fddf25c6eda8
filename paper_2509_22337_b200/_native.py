"""ctypes binding of the C ABI in ``include/hornbp_gpu.h`` (``_lib/libhbp.so``).

This is the only way the package reaches native code; there is no Python or
CPU fallback for the engine. If the library is missing the import of the
engine fails loudly (build it with ``python -m paper_2509_22337_b200._build``
or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HBP_LIB_PATH") or os.path.join(_HERE, "_lib", "libhbp.so")

HBP_OK = 0
HBP_EINVAL = 1
HBP_EUNDERFLOW = 2
HBP_ECUDA = 3
HBP_ENCCL = 4
HBP_ECYCLE = 5
HBP_ENOMEM = 6

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
i8p = C.POINTER(C.c_int8)


class GraphDesc(C.Structure):
    _fields_ = [
        ("num_variables", C.c_int32),
        ("num_factors", C.c_int32),
        ("num_edges", C.c_int64),
        ("factor_rowptr", i64p),
        ("edge_var", i32p),
        ("factor_kind", i8p),
        ("p1", f64p),
        ("p2", f64p),
    ]


class Options(C.Structure):
    _fields_ = [
        ("max_iterations", C.c_int32),
        ("normalize_messages", C.c_int32),
        ("record_history", C.c_int32),
        ("evidence_count", C.c_int32),
        ("tolerance", C.c_double),
        ("time_limit", C.c_double),
        ("precision", C.c_int32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("last_delta", C.c_double),
        ("underflow_kind", C.c_int32),
        ("underflow_iteration", C.c_int32),
        ("underflow_index", C.c_int64),
        ("device_ms", C.c_double),
        ("total_ms", C.c_double),
    ]


class Evidence(C.Structure):
    _fields_ = [
        ("num_sets", C.c_int32),
        ("offsets", i64p),
        ("var", i32p),
        ("value", i8p),
    ]


class SetResult(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("last_delta", C.c_double),
        ("underflow_kind", C.c_int32),
        ("underflow_iteration", C.c_int32),
        ("underflow_index", C.c_int64),
    ]


class SweepOutputs(C.Structure):
    _fields_ = [
        ("sets", C.POINTER(SetResult)),
        ("deltas", f64p),
        ("marginals", f64p),
        ("marginals_on_device", C.c_int32),
        ("num_select", C.c_int32),
        ("select", i32p),
        ("p1_select", f64p),
        ("p1_on_device", C.c_int32),
        ("topk", C.c_int32),
        ("ranked", i32p),
        ("ranked_on_device", C.c_int32),
        ("device_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("wall_ms", C.c_double),
        ("launches", C.c_int32),
        ("passes", C.c_int32),
        ("compactions", C.c_int32),
    ]


class NativeError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load ``libhbp.so`` once; raise ImportError if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native engine library missing: {LIB_PATH} "
                "(run __graft_entry__.build() or python -m paper_2509_22337_b200._build)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        sigs = {
            "hbp_compile": (C.c_int32, [C.POINTER(GraphDesc), C.c_int64, i32p, i32p, i32p,
                                        C.POINTER(vp), i64p]),
            "hbp_toposort": (C.c_int32, [C.c_int64, C.c_int64, i32p, i32p, i32p, i64p]),
            "hbp_schedule_sizes": (C.c_int32, [vp, i64p, i64p, i64p]),
            "hbp_schedule_copy": (C.c_int32, [vp, i64p, i32p, i64p, i32p]),
            "hbp_schedule_destroy": (None, [vp]),
            "hbp_graph_create": (C.c_int32, [C.POINTER(GraphDesc), C.c_int32, C.POINTER(vp)]),
            "hbp_graph_destroy": (None, [vp]),
            "hbp_graph_set_stream": (C.c_int32, [vp, vp]),
            "hbp_graph_set_evidence": (C.c_int32, [vp, C.c_int32, i32p, i8p]),
            "hbp_graph_rank": (C.c_int32, [vp, C.c_int32, i32p, C.c_int32, i32p, f64p]),
            "hbp_graph_layout": (C.c_int32, [vp, i64p, i64p]),
            "hbp_graph_layout_check": (C.c_int32, [vp, i64p]),
            "hbp_plan_create": (C.c_int32, [vp, C.c_int64, i64p, i32p, i64p, i32p, C.POINTER(vp)]),
            "hbp_plan_destroy": (None, [vp]),
            "hbp_run": (C.c_int32, [vp, C.POINTER(Options), f64p, f64p, f64p, C.POINTER(Result)]),
            "hbp_graph_history": (C.c_int32, [vp, C.c_int32, f64p]),
            "hbp_run_device": (C.c_int32, [vp, C.POINTER(Options), C.POINTER(Result),
                                           C.POINTER(C.c_void_p)]),
            "hbp_pass": (C.c_int32, [vp, C.c_int32, C.c_int64, i32p, C.c_int32, f64p, f64p,
                                     f64p, f64p, i64p]),
            "hbp_marginals": (C.c_int32, [vp, f64p, f64p, f64p, i64p]),
            "hbp_sweep_create": (C.c_int32, [vp, C.c_int32, C.POINTER(vp)]),
            "hbp_sweep_capacity": (C.c_int32, [vp]),
            "hbp_sweep_run": (C.c_int32, [vp, C.POINTER(Options), C.POINTER(Evidence),
                                          C.POINTER(SweepOutputs)]),
            "hbp_sweep_destroy": (None, [vp]),
            "hbp_last_launch_count": (C.c_int64, []),
            "hbp_selftest_division": (C.c_int32, [C.c_int64, f64p, f64p, f64p, f64p]),
            "hbp_last_error": (C.c_char_p, []),
            "hbp_version": (C.c_char_p, []),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return _lib


EXPORTED = ("hbp_compile", "hbp_toposort", "hbp_schedule_sizes", "hbp_schedule_copy",
            "hbp_schedule_destroy", "hbp_graph_create", "hbp_graph_destroy", "hbp_graph_set_stream", "hbp_graph_set_evidence",
            "hbp_graph_rank", "hbp_graph_layout", "hbp_graph_layout_check",
            "hbp_plan_create", "hbp_plan_destroy", "hbp_run", "hbp_graph_history", "hbp_run_device", "hbp_pass",
            "hbp_marginals", "hbp_sweep_create", "hbp_sweep_capacity", "hbp_sweep_run",
            "hbp_sweep_destroy", "hbp_last_launch_count", "hbp_selftest_division", "hbp_last_error",
            "hbp_version")


def last_error() -> str:
    return lib().hbp_last_error().decode()


def check(status: int, what: str) -> None:
    if status != HBP_OK:
        raise NativeError(status, f"{what}: {last_error()}")


def ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


class GraphArrays:
    """Keeps the contiguous arrays alive for a GraphDesc."""

    def __init__(self, graph):
        self.rowptr = np.ascontiguousarray(graph.rowptr, dtype=np.int64)
        self.vars = np.ascontiguousarray(graph.vars, dtype=np.int32)
        self.kind = np.ascontiguousarray(graph.kind, dtype=np.int8)
        self.p1 = np.ascontiguousarray(graph.p1, dtype=np.float64)
        self.p2 = np.ascontiguousarray(graph.p2, dtype=np.float64)
        self.desc = GraphDesc(graph.num_variables, graph.num_factors, graph.num_edges,
                              ptr(self.rowptr, C.c_int64), ptr(self.vars, C.c_int32),
                              ptr(self.kind, C.c_int8), ptr(self.p1, C.c_double),
                              ptr(self.p2, C.c_double))


def compile_arrays(graph, before: np.ndarray, after: np.ndarray, rank=None):
    """Native compile: returns (s_off, s_edges, t_off, t_edges) arrays.
    Raises NativeError(HBP_ECYCLE) with .cycle_edge on a cycle."""
    L = lib()
    ga = GraphArrays(graph)
    before = np.ascontiguousarray(before, dtype=np.int32)
    after = np.ascontiguousarray(after, dtype=np.int32)
    rk = None if rank is None else np.ascontiguousarray(rank, dtype=np.int32)
    handle = C.c_void_p()
    cyc = C.c_int64(-1)
    st = L.hbp_compile(C.byref(ga.desc), len(before), ptr(before, C.c_int32), ptr(after, C.c_int32),
                       None if rk is None else ptr(rk, C.c_int32), C.byref(handle), C.byref(cyc))
    if st != HBP_OK:
        err = NativeError(st, last_error())
        err.cycle_edge = int(cyc.value)
        raise err
    try:
        k, ns, nt = C.c_int64(), C.c_int64(), C.c_int64()
        L.hbp_schedule_sizes(handle, C.byref(k), C.byref(ns), C.byref(nt))
        s_off = np.empty(k.value + 1, dtype=np.int64)
        t_off = np.empty(k.value + 1, dtype=np.int64)
        s_e = np.empty(ns.value, dtype=np.int32)
        t_e = np.empty(nt.value, dtype=np.int32)
        L.hbp_schedule_copy(handle, ptr(s_off, C.c_int64), ptr(s_e, C.c_int32),
                            ptr(t_off, C.c_int64), ptr(t_e, C.c_int32))
    finally:
        L.hbp_schedule_destroy(handle)
    return s_off, s_e, t_off, t_e


def toposort(num_edges: int, before: np.ndarray, after: np.ndarray) -> np.ndarray:
    L = lib()
    before = np.ascontiguousarray(before, dtype=np.int32)
    after = np.ascontiguousarray(after, dtype=np.int32)
    out = np.empty(num_edges, dtype=np.int32)
    cyc = C.c_int64(-1)
    st = L.hbp_toposort(num_edges, len(before), ptr(before, C.c_int32), ptr(after, C.c_int32),
                        ptr(out, C.c_int32), C.byref(cyc))
    if st != HBP_OK:
        err = NativeError(st, last_error())
        err.cycle_edge = int(cyc.value)
        raise err
    return out
