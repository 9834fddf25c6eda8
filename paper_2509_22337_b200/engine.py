"""Inference engine: the reference's ``hornbp.engine`` API on the B200 executor.

``run(graph, schedule, options, workers)`` keeps the reference signature and
result type (engine.py:531-594). Underneath, a graph is laid out on the device
once (``hbp_graph_create``), a schedule becomes a device-resident level
program once (``hbp_plan_create``), and every ``run`` is a single persistent
kernel launch that iterates to convergence on the device
(``csrc/engine.cu``). Both are cached per (graph, schedule) object, the
reference's "compile once, run many" contract (storage.py:31-34).

The single-pass functions (``update_vtof_batch``, ``update_ftov_batch``,
``update_{and,or}_{body,head}``, ``compute_marginals``,
``closed_form_message``) operate on a host ``MessageStore`` like the
reference; each call ships the store to the device, runs one pass of the
same message kernels, and scatters the results back.

There is no CPU fallback: without the native library the package fails to
import the engine, and without a GPU every device call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native
from .graph import EdgeId, Factor, FactorGraph, FactorKind, KIND_OR
from .schedule import Schedule
from .storage import MessageStore, StorageError, initialize

MIN_MESSAGE_SUM = 1e-300

_native.lib()  # fail loudly at import if the engine library is missing


class UnderflowError(RuntimeError):
    """A message or marginal degenerated to total mass zero
    (usually contradictory evidence on connected variables).

    Beyond the reference's message, raised instances carry ``kind`` (1
    variable-to-factor, 2 factor-to-variable, 3 marginal), ``iteration`` (0
    for the single-pass API) and ``index``: the reference's own report --
    the vtof store position, the ftov store position, or the variable id of
    ``rows[argmin(total)]`` in the first failing pass (engine.py:155-165,
    :512-518)."""

    kind: int = 0
    iteration: int = 0
    index: int = -1


def _underflow_error(kind: int, index: int, iteration: int = 0) -> UnderflowError:
    """The reference's UnderflowError text (engine.py:159-164, :515-518)."""
    if kind == 1:
        msg = f"variable-to-factor message degenerated to zero mass at {index} (contradictory evidence?)"
    elif kind == 2:
        msg = f"factor-to-variable message degenerated to zero mass at {index} (contradictory evidence?)"
    else:
        msg = f"marginal of variable {index} degenerated to zero mass (contradictory evidence?)"
    exc = UnderflowError(msg)
    exc.kind, exc.index, exc.iteration = int(kind), int(index), int(iteration)
    return exc


class OpCounter:
    """Counts elementwise multiplications executed by the message kernels."""

    __slots__ = ("count",)

    def __init__(self):
        self.count = 0

    def add(self, n: int) -> None:
        self.count += int(n)


@dataclass
class EngineOptions:
    max_iterations: int = 1000
    tolerance: float = 1e-9
    normalize_messages: bool = True
    time_limit: Optional[float] = None
    record_history: bool = False
    # extension (not in the reference): "fp64" -- bitwise with the reference --
    # or "fp32" messages for run_many (marginals within 1e-5 of fp64)
    precision: str = "fp64"

    def validate(self) -> None:
        if self.precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.tolerance < 0:
            raise ValueError("tolerance must be nonnegative")
        if self.time_limit is not None and self.time_limit <= 0:
            raise ValueError("time_limit must be positive")


@dataclass
class InferenceResult:
    marginals: np.ndarray  # (num_variables, 2): P(X=0), P(X=1)
    converged: bool
    iterations: int
    last_delta: float
    deltas: list[float] = field(default_factory=list)
    history: Optional[list[np.ndarray]] = None
    # additions (not in the reference): device time of the iteration loop and
    # the bench numerator sum |s_i| + |t_i| (cli.py:337-339)
    device_ms: Optional[float] = None
    updates_per_iteration: Optional[int] = None


# ---- device handles ----------------------------------------------------------------------

_device_index = int(os.environ.get("HBP_DEVICE", "0"))
_cache_lock = threading.Lock()
_GRAPHS: "OrderedDict[int, tuple[weakref.ref, _DeviceGraph]]" = OrderedDict()
_MAX_CACHED_GRAPHS = 6


def set_device(index: int) -> None:
    """CUDA device used for new device graphs (one process per GPU)."""
    global _device_index
    _device_index = int(index)


def get_device() -> int:
    return _device_index


def _raise_status(status: int, what: str, result: Optional[_native.Result] = None,
                  graph: Optional[FactorGraph] = None):
    msg = _native.last_error()
    if status == _native.HBP_EUNDERFLOW and result is not None:
        raise _underflow_error(result.underflow_kind, int(result.underflow_index),
                               result.underflow_iteration)
    if status in (_native.HBP_EINVAL, _native.HBP_ECYCLE):
        raise ValueError(f"{what}: {msg}")
    if status == _native.HBP_ENOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


class _GraphHandle:
    """Owns one hbp_graph. Plans and sweeps hold this (not the _DeviceGraph
    that caches them), so the ownership graph has no cycle: dropping a
    _DeviceGraph frees its plans, sweeps and device memory at once, by
    reference count, instead of at some later cyclic-GC pass."""

    def __init__(self, arrays, num_variables: int, num_edges: int, device: int):
        self.num_variables = num_variables
        self.num_edges = num_edges
        self.device = device
        h = C.c_void_p()
        st = _native.lib().hbp_graph_create(C.byref(arrays.desc), device, C.byref(h))
        if st != _native.HBP_OK:
            _raise_status(st, "hbp_graph_create")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _native.lib().hbp_graph_destroy(h)
            except Exception:  # interpreter shutdown: the module may be gone
                pass
            self.handle = None


class _Plan:
    def __init__(self, dg: "_GraphHandle", arrays):
        s_off, s_e, t_off, t_e = arrays
        self.dg = dg
        self.updates = int(len(s_e) + len(t_e))
        self.num_batches = len(s_off) - 1
        h = C.c_void_p()
        st = _native.lib().hbp_plan_create(
            dg.handle, len(s_off) - 1, _native.ptr(np.ascontiguousarray(s_off), C.c_int64),
            _native.ptr(np.ascontiguousarray(s_e, dtype=np.int32), C.c_int32),
            _native.ptr(np.ascontiguousarray(t_off), C.c_int64),
            _native.ptr(np.ascontiguousarray(t_e, dtype=np.int32), C.c_int32), C.byref(h))
        if st != _native.HBP_OK:
            _raise_status(st, "hbp_plan_create")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _native.lib().hbp_plan_destroy(h)
            except Exception:  # interpreter shutdown: the module may be gone
                pass
            self.handle = None

    def options(self, options: EngineOptions) -> _native.Options:
        return _native.Options(int(options.max_iterations), int(bool(options.normalize_messages)),
                               int(bool(options.record_history)), 0, float(options.tolerance),
                               float(options.time_limit) if options.time_limit else 0.0,
                               1 if options.precision == "fp32" else 0)

    def run(self, options: EngineOptions, graph: FactorGraph) -> InferenceResult:
        V = self.dg.num_variables
        opt = self.options(options)
        marg = np.empty((V, 2), dtype=np.float64)
        deltas = np.empty(options.max_iterations, dtype=np.float64)
        res = _native.Result()
        st = _native.lib().hbp_run(self.handle, C.byref(opt), _native.ptr(marg, C.c_double),
                                   _native.ptr(deltas, C.c_double), None, C.byref(res))
        if st != _native.HBP_OK:
            _raise_status(st, "hbp_run", res, graph)
        n = res.iterations
        hist = None
        if options.record_history:  # sized by the iterations run (engine.py:574-575)
            hist = np.empty((n, V, 2), dtype=np.float64)
            st = _native.lib().hbp_graph_history(self.dg.handle, n, _native.ptr(hist, C.c_double))
            if st != _native.HBP_OK:
                _raise_status(st, "hbp_graph_history")
        return InferenceResult(
            marginals=marg, converged=bool(res.converged), iterations=n,
            last_delta=float(res.last_delta), deltas=deltas[:n].tolist(),
            history=None if hist is None else [hist[i].copy() for i in range(n)],
            device_ms=float(res.device_ms), updates_per_iteration=self.updates)


    def run_device(self, options: EngineOptions, graph: FactorGraph) -> _native.Result:
        """Run with the marginals left on the device (hbp_run_device)."""
        opt = self.options(options)
        res = _native.Result()
        st = _native.lib().hbp_run_device(self.handle, C.byref(opt), C.byref(res), None)
        if st != _native.HBP_OK:
            _raise_status(st, "hbp_run_device", res, graph)
        return res


class _Sweep:
    def __init__(self, dg: "_GraphHandle", capacity: int):
        self.dg = dg
        h = C.c_void_p()
        st = _native.lib().hbp_sweep_create(dg.handle, int(capacity), C.byref(h))
        if st != _native.HBP_OK:
            _raise_status(st, "hbp_sweep_create")
        self.handle = h
        self.capacity = int(_native.lib().hbp_sweep_capacity(h))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _native.lib().hbp_sweep_destroy(h)
            except Exception:  # interpreter shutdown: the module may be gone
                pass
            self.handle = None


class _DeviceGraph:
    """Device layout of one FactorGraph plus its compiled plans."""

    def __init__(self, graph: FactorGraph, device: int):
        self.arrays = _native.GraphArrays(graph)
        self.num_variables = graph.num_variables
        self.num_edges = graph.num_edges
        self.device = device
        self.h = _GraphHandle(self.arrays, graph.num_variables, graph.num_edges, device)
        self.handle = self.h.handle
        self._plans: "OrderedDict[int, tuple[weakref.ref, _Plan]]" = OrderedDict()
        self._sweeps: dict = {}

    def plan(self, schedule: Schedule, graph: FactorGraph) -> _Plan:
        key = id(schedule)
        hit = self._plans.get(key)
        if hit is not None and hit[0]() is schedule:
            self._plans.move_to_end(key)
            return hit[1]
        p = _Plan(self.h, schedule.arrays(graph))
        self._plans[key] = (weakref.ref(schedule), p)
        while len(self._plans) > 8:
            self._plans.popitem(last=False)
        return p

    def set_stream(self, stream) -> None:
        """Run this graph's device work on an external stream (an int handle,
        or anything with ``cuda_stream``, e.g. a torch.cuda.Stream); None =
        the graph's own stream."""
        handle = getattr(stream, "cuda_stream", stream)
        st = _native.lib().hbp_graph_set_stream(self.handle, C.c_void_p(handle or None))
        if st != _native.HBP_OK:
            _raise_status(st, "hbp_graph_set_stream")

    def set_evidence(self, variables, values) -> None:
        """Clamp ``variables`` to ``values`` for the following runs
        (hbp_graph_set_evidence); empty clears."""
        var = np.ascontiguousarray(np.asarray(variables, dtype=np.int32))
        val = np.ascontiguousarray(np.asarray(values, dtype=np.int8))
        st = _native.lib().hbp_graph_set_evidence(self.handle, len(var), _native.ptr(var, C.c_int32),
                                                   _native.ptr(val, C.c_int8))
        if st != _native.HBP_OK:
            _raise_status(st, "hbp_graph_set_evidence")

    def rank(self, select: np.ndarray, topk: int) -> tuple[np.ndarray, np.ndarray]:
        """Top-k of ``select`` (ascending ids) by the last run's P1, variables
        with evidence excluded (hbp_graph_rank)."""
        sel = np.ascontiguousarray(select, dtype=np.int32)
        out = np.empty(topk, dtype=np.int32)
        p1 = np.empty(topk, dtype=np.float64)
        st = _native.lib().hbp_graph_rank(self.handle, len(sel), _native.ptr(sel, C.c_int32),
                                          int(topk), _native.ptr(out, C.c_int32),
                                          _native.ptr(p1, C.c_double))
        if st != _native.HBP_OK:
            _raise_status(st, "hbp_graph_rank")
        return out, p1

    def sweep(self, capacity: int = 0) -> "_Sweep":
        """Multi-evidence sweep buffers for this graph (cached per capacity)."""
        sw = self._sweeps.get(capacity)
        if sw is None:
            self._sweeps.clear()  # one set of sweep buffers per graph
            sw = _Sweep(self.h, capacity)
            self._sweeps[capacity] = sw
        return sw

    def parall_updates(self, graph: FactorGraph) -> int:
        """sum |s_0| + |t_0| of the PARALL schedule: every edge plus every
        slot of a non-unary factor (schedule.py:293-312)."""
        if getattr(self, "_parall_updates", None) is None:  # per graph, once
            deg = np.diff(np.asarray(graph.rowptr, dtype=np.int64))
            self._parall_updates = int(graph.num_edges + deg[deg > 1].sum())
        return self._parall_updates

    def __del__(self):
        # plans and sweeps first (they hold self.h); the graph goes with the
        # last reference to self.h
        self._sweeps = {}
        self._plans = OrderedDict()


def device_graph(graph: FactorGraph) -> _DeviceGraph:
    """Cached device layout for ``graph`` on the current device."""
    key = id(graph)
    with _cache_lock:
        hit = _GRAPHS.get(key)
        if hit is not None and hit[0]() is graph and hit[1].device == _device_index:
            _GRAPHS.move_to_end(key)
            return hit[1]
    if graph.num_edges == 0:
        raise StorageError("graph has no edges")
    dg = _DeviceGraph(graph, _device_index)
    with _cache_lock:
        _GRAPHS[key] = (weakref.ref(graph, lambda _r, k=key: _GRAPHS.pop(k, None)), dg)
        while len(_GRAPHS) > _MAX_CACHED_GRAPHS:
            _GRAPHS.popitem(last=False)
    return dg


def clear_device_cache() -> None:
    with _cache_lock:
        _GRAPHS.clear()


def _resolve_workers(workers: int) -> int:
    """``workers`` is accepted for signature compatibility; results never
    depend on it (engine.py:28) and the device ignores it."""
    if workers < 0:
        raise ValueError("workers must be nonnegative")
    return workers or (os.cpu_count() or 1)


# ---- run ----------------------------------------------------------------------------------

def run(graph: FactorGraph, schedule: Schedule, options: Optional[EngineOptions] = None,
        workers: int = 1) -> InferenceResult:
    """Iterate the schedule until marginals stop moving or budgets run out
    (engine.py:531-594): per iteration every batch refreshes its
    variable-to-factor then its factor-to-variable messages; converged iff
    max |dP1| < tolerance after an iteration."""
    options = options or EngineOptions()
    options.validate()
    _resolve_workers(workers)
    if options.precision != "fp64":
        return _run_fp32(graph, schedule, options)
    dg = device_graph(graph)
    return dg.plan(schedule, graph).run(options, graph)


def _run_fp32(graph: FactorGraph, schedule: Schedule, options: EngineOptions) -> InferenceResult:
    """The optional fp32 mode for a single graph: message
    storage in fp32, arithmetic and marginals in fp64, through the sweep
    kernel's fp32 instance with one (empty) evidence set. PARALL schedules
    only -- the fp32 storage lives in the sweep kernel, which runs the
    synchronous schedule. Marginals are within 1e-5 of the fp64 run
    (north star), not bitwise."""
    from .sweep import run_many

    s_off, s_e, t_off, t_e = schedule.arrays(graph)
    rp = np.asarray(graph.rowptr, dtype=np.int64)
    nonunary = int((np.diff(rp)[np.diff(rp) > 1]).sum())
    if len(s_off) != 2 or len(s_e) != graph.num_edges or len(t_e) != nonunary:
        raise ValueError("fp32 mode runs PARALL schedules only (the fp32 message storage is the "
                         "sweep kernel's)")
    if options.record_history:
        raise ValueError("record_history is not supported in fp32 mode")
    r = run_many(graph, [[]], None, options,
                 marginals=True, deltas=True)
    if r.errors and r.errors[0] is not None:
        raise r.errors[0]
    return InferenceResult(marginals=r.marginals[0], converged=bool(r.converged[0]),
                           iterations=int(r.iterations[0]), last_delta=float(r.last_delta[0]),
                           deltas=list(r.deltas[0]), history=None, device_ms=r.kernel_ms,
                           updates_per_iteration=int(r.updates_per_iteration[0]))


# ---- single-pass API on a host store ------------------------------------------------------

def _store_pass(store: MessageStore, direction: int, targets: np.ndarray, normalize: bool) -> None:
    dg = device_graph(store.graph)
    t = np.ascontiguousarray(targets, dtype=np.int32)
    for name in ("vtof0", "vtof1", "ftov0", "ftov1"):
        arr = getattr(store, name)
        if not (arr.flags.c_contiguous and arr.dtype == np.float64):
            setattr(store, name, np.ascontiguousarray(arr, dtype=np.float64))
    where = C.c_int64(-1)
    st = _native.lib().hbp_pass(dg.handle, direction, len(t), _native.ptr(t, C.c_int32),
                                int(bool(normalize)), _native.ptr(store.vtof0, C.c_double),
                                _native.ptr(store.vtof1, C.c_double),
                                _native.ptr(store.ftov0, C.c_double),
                                _native.ptr(store.ftov1, C.c_double), C.byref(where))
    if st == _native.HBP_EUNDERFLOW:
        raise _underflow_error(1 if direction == 0 else 2, int(where.value))
    if st != _native.HBP_OK:
        _raise_status(st, "hbp_pass")


def _count_vtof(store: MessageStore, idx: np.ndarray, counter: Optional[OpCounter]) -> None:
    """The reference's count (engine.py:181-182): 2 multiplies per lane of the
    product scan, whose lanes cover every slot of the target's row (the own
    slot multiplies by 1.0) -- 2 x row length per target."""
    if counter is not None:
        d = store.av_end[idx] - store.av_start[idx]
        counter.add(int((2 * d).sum()))


def _count_ftov(store: MessageStore, idx: np.ndarray, counter: Optional[OpCounter]) -> None:
    """The reference's count per factor-to-variable target with factor row
    length d: body targets 4d (engine.py:224-225) + 1 (:258-259, :292-293),
    head targets 2d (:246-247) + 3 (:277-278, :311-312)."""
    if counter is not None:
        ft = store.vtof_to_ftov[idx]
        d = store.af_end[ft] - store.af_start[ft]
        head = store.af_head[ft]
        n = np.where(head, 2 * d + 3, 4 * d + 1)
        counter.add(int(n.sum()))


def update_vtof_batch(store: MessageStore, edges: Sequence[EdgeId], normalize: bool = True,
                      workers: int = 1, counter: Optional[OpCounter] = None) -> None:
    """Recompute the named variable-to-factor messages (engine.py:413-428)."""
    if not len(edges):
        return
    idx = store.vtof_indices(list(edges))
    _count_vtof(store, idx, counter)
    _store_pass(store, 0, idx, normalize)


def update_ftov_batch(store: MessageStore, edges: Sequence[EdgeId], normalize: bool = True,
                      workers: int = 1, counter: Optional[OpCounter] = None) -> None:
    """Recompute the named factor-to-variable messages (engine.py:431-446);
    the device groups them by (kind, head/body, degree) itself."""
    if not len(edges):
        return
    idx = store.vtof_indices(list(edges))
    _count_ftov(store, idx, counter)
    _store_pass(store, 1, idx, normalize)


def split_ftov_batch(graph: FactorGraph, batch: Sequence[EdgeId]):
    """(AND body, AND head, OR body, OR head) routing of a batch (engine.py:357-377)."""
    groups: tuple[list, list, list, list] = ([], [], [], [])
    for edge in batch:
        graph.check_edge(edge)
        is_or = int(graph.kind[edge[0]]) == KIND_OR
        groups[2 * is_or + (edge[1] == 0)].append(edge)
    return groups


def _routed_update(store, edges, kind: FactorKind, head: bool, normalize, counter) -> None:
    if not len(edges):
        return
    graph = store.graph
    want = 1 if kind is FactorKind.OR else 0
    for edge in edges:
        graph.check_edge(edge)
        if int(graph.kind[edge[0]]) != want or (edge[1] == 0) != head:
            where = "head" if head else "body"
            raise ValueError(f"edge {EdgeId(*edge)} is not a {kind.value} {where} target")
    update_ftov_batch(store, edges, normalize, counter=counter)


def update_and_body(store, edges, normalize=True, workers=1, counter=None) -> None:
    """Messages from AND factors toward body variables."""
    _routed_update(store, edges, FactorKind.AND, False, normalize, counter)


def update_and_head(store, edges, normalize=True, workers=1, counter=None) -> None:
    """Messages from AND factors toward their head variable."""
    _routed_update(store, edges, FactorKind.AND, True, normalize, counter)


def update_or_body(store, edges, normalize=True, workers=1, counter=None) -> None:
    """Messages from OR factors toward body variables."""
    _routed_update(store, edges, FactorKind.OR, False, normalize, counter)


def update_or_head(store, edges, normalize=True, workers=1, counter=None) -> None:
    """Messages from OR factors toward their head variable."""
    _routed_update(store, edges, FactorKind.OR, True, normalize, counter)


def compute_marginals(store: MessageStore) -> np.ndarray:
    """(P0, P1) per variable from the store's ftov buffers (engine.py:500-528)."""
    dg = device_graph(store.graph)
    out = np.empty((store.graph.num_variables, 2), dtype=np.float64)
    f0 = np.ascontiguousarray(store.ftov0, dtype=np.float64)
    f1 = np.ascontiguousarray(store.ftov1, dtype=np.float64)
    bad = C.c_int64(-1)
    st = _native.lib().hbp_marginals(dg.handle, _native.ptr(f0, C.c_double),
                                     _native.ptr(f1, C.c_double), _native.ptr(out, C.c_double),
                                     C.byref(bad))
    if st == _native.HBP_EUNDERFLOW:
        raise _underflow_error(3, int(bad.value))
    if st != _native.HBP_OK:
        _raise_status(st, "hbp_marginals")
    return out


def closed_form_message(kind: FactorKind, p1: float, p2: float,
                        incoming: Sequence[Optional[tuple[float, float]]], target_slot: int,
                        counter: Optional[OpCounter] = None) -> tuple[float, float]:
    """One unnormalised factor-to-variable message through the device kernels
    (engine.py:597-628); ``incoming`` is indexed by slot, head first."""
    degree = len(incoming)
    if not 0 <= target_slot < degree:
        raise ValueError("target slot out of range")
    factor = Factor(kind, 0, tuple(range(1, degree)), p1, p2)
    store = initialize(FactorGraph(degree, [factor]))
    for slot in range(degree):
        if slot == target_slot:
            continue
        store.vtof0[slot], store.vtof1[slot] = incoming[slot]
    edge = EdgeId(0, target_slot)
    update_ftov_batch(store, [edge], normalize=False, counter=counter)
    i = store.ftov_index(edge)
    return float(store.ftov0[i]), float(store.ftov1[i])
