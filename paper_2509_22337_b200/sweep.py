"""Multi-evidence sweep: many evidence / feedback sets over one graph.

The reference answers "what would the ranking be under feedback set j?" one
set at a time: ``clamp_evidence`` per observed alarm, ``Strategy.compile`` on
the clamped graph, ``run`` from uniform (``ranking.py:94-135``,
``graph.py:189-200``, ``engine.py:531``). ``run_many`` answers it for many
sets at once on the device: under PARALL, set j's result is bitwise identical
to ``run(G_j, Strategy.parall().compile(G_j), options)`` with ``G_j`` the base
graph clamped to set j's observations in order (csrc/sweep.cu explains why a
shared CSR with per-set evidence codes is exact). Each set stops at its own
convergence iteration.

Other strategies have no shared-CSR form for every clamp pattern (an explicit
SEQFIX order cannot even be recompiled after a clamp, schedule.py:184-185),
so ``run_many`` materialises the clamped graph per set and runs it on the
single-graph device executor -- the reference's own semantics, still on the
GPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _native
from .engine import EngineOptions, UnderflowError, _underflow_error, device_graph, run
from .graph import FactorGraph, GraphError, clamp_evidence
from .schedule import Strategy


@dataclass
class SweepResult:
    """Per-set outputs of ``run_many`` (set j in row j)."""

    iterations: np.ndarray                 # (n,) int32
    converged: np.ndarray                  # (n,) bool
    last_delta: np.ndarray                 # (n,) float64
    deltas: Optional[list[list[float]]]    # per set, like InferenceResult.deltas
    marginals: Optional[np.ndarray]        # (n, V, 2) float64 (P0, P1)
    p1_select: Optional[np.ndarray]        # (n, len(select)) float64
    ranked: Optional[np.ndarray]           # (n, topk) int32, -1 padded
    select: Optional[np.ndarray]           # the selection (ascending variable ids)
    errors: list[Optional[UnderflowError]] = field(default_factory=list)
    updates_per_iteration: Optional[np.ndarray] = None  # (n,) sum|s_i| + |t_i| of G_j
    device_ms: Optional[float] = None      # stream time of the sweep (all passes)
    kernel_ms: Optional[float] = None      # persistent sweep kernel(s) only
    launches: int = 0
    passes: int = 0
    compactions: int = 0                   # straggler compactions (staged kernel)

    def __len__(self) -> int:
        return len(self.iterations)

    def total_updates(self) -> int:
        """Edge-message updates over all sets (cli.py:337-344 per set)."""
        return int(np.dot(self.updates_per_iteration.astype(np.int64),
                          self.iterations.astype(np.int64)))


def _host_empty(shape, dtype) -> np.ndarray:
    """Output array in page-locked host memory when torch's caching pinned
    allocator is available (device-to-host copies run at full PCIe/C2C rate
    and the buffers are reused across calls); plain numpy otherwise."""
    try:
        import torch

        if torch.cuda.is_available():
            t = torch.empty(shape, dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True)
            return t.numpy()
    except (ImportError, RuntimeError, AttributeError):
        pass
    return np.empty(shape, dtype=dtype)


class EvidenceCSR:
    """Evidence sets in CSR form: set j is var[offsets[j]:offsets[j+1]] with
    observed values val[...] (nonzero = true). ``run_many`` takes it as is --
    no per-set Python conversion -- e.g. when the same sets are swept
    repeatedly (build it once with ``EvidenceCSR.from_sets``)."""

    def __init__(self, offsets, var, val):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.var = np.ascontiguousarray(var, dtype=np.int32)
        self.val = np.ascontiguousarray(np.asarray(val) != 0, dtype=np.int8)
        if (self.offsets.ndim != 1 or len(self.offsets) < 1 or self.offsets[0] != 0
                or np.any(np.diff(self.offsets) < 0) or self.offsets[-1] != len(self.var)
                or len(self.val) != len(self.var)):
            raise ValueError("bad evidence CSR")

    @classmethod
    def from_sets(cls, graph: FactorGraph, evidence_sets) -> "EvidenceCSR":
        return cls(*_normalise_sets(graph, evidence_sets))

    def __len__(self) -> int:
        return len(self.offsets) - 1

    def __getitem__(self, key):
        """A slice of sets is an EvidenceCSR (re-based offsets, views of the
        arrays); an integer is set j as a list of (variable, observed) pairs."""
        if isinstance(key, slice):
            lo, hi, step = key.indices(len(self))
            if step != 1:
                raise ValueError("EvidenceCSR slices must be contiguous")
            hi = max(lo, hi)
            a, b = int(self.offsets[lo]), int(self.offsets[hi])
            return EvidenceCSR(self.offsets[lo:hi + 1] - a, self.var[a:b], self.val[a:b])
        j = int(key)
        if j < 0:
            j += len(self)
        if not 0 <= j < len(self):
            raise IndexError("evidence set index out of range")
        a, b = int(self.offsets[j]), int(self.offsets[j + 1])
        return [(int(v), bool(o)) for v, o in zip(self.var[a:b].tolist(), self.val[a:b].tolist())]


def _normalise_sets(graph: FactorGraph, evidence_sets) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Evidence sets -> (offsets, var, value). A set is an iterable of
    (variable, observed) pairs or an (ids, labels) pair of arrays (zipped,
    so the shorter one bounds it); an EvidenceCSR is taken as is."""
    if isinstance(evidence_sets, EvidenceCSR):
        v = evidence_sets.var
        bad = (v < 0) | (v >= graph.num_variables)
        if bad.any():
            raise GraphError(f"variable {int(v[int(np.argmax(bad))])} out of range")
        return evidence_sets.offsets, evidence_sets.var, evidence_sets.val
    vs: list[np.ndarray] = []
    os_: list[np.ndarray] = []
    for ev in evidence_sets:
        if isinstance(ev, tuple) and len(ev) == 2 and all(isinstance(x, np.ndarray) for x in ev):
            n = min(len(ev[0]), len(ev[1]))
            v = ev[0][:n].ravel()
            o = ev[1][:n].ravel()
        else:
            pairs = list(ev)
            v = np.fromiter((int(p[0]) for p in pairs), dtype=np.int64, count=len(pairs))
            o = np.fromiter((bool(p[1]) for p in pairs), dtype=bool, count=len(pairs))
        vs.append(v)
        os_.append(o)
    offsets = np.zeros(len(vs) + 1, dtype=np.int64)
    if vs:
        np.cumsum([len(v) for v in vs], out=offsets[1:])
    var = np.concatenate(vs).astype(np.int64) if vs else np.zeros(0, dtype=np.int64)
    val = np.concatenate(os_).astype(bool) if os_ else np.zeros(0, dtype=bool)
    bad = (var < 0) | (var >= graph.num_variables)
    if bad.any():
        raise GraphError(f"variable {int(var[int(np.argmax(bad))])} out of range")
    return offsets, var.astype(np.int32), val.astype(np.int8)




def _is_parall(strategy) -> bool:
    return strategy is None or getattr(strategy, "kind", None) == "PARALL"


def run_many(graph: FactorGraph, evidence_sets: Iterable, strategy: Optional[Strategy] = None,
             options: Optional[EngineOptions] = None, *, marginals: bool = True,
             deltas: bool = True, select: Optional[Sequence[int]] = None, topk: int = 0,
             capacity: int = 0, device_out: Optional[dict] = None) -> SweepResult:
    """Run every evidence set from uniform messages; see the module docstring.

    select / topk: also return P1 of the selected variables (ascending ids)
    and, if topk > 0, the top-k of the selection ranked like
    ``rank_alarms(marginals, alarms, already_labeled=set's variables)``.
    device_out: optional {"marginals"|"p1_select"|"ranked": tensor} device
    buffers (anything with ``data_ptr()``) on the graph's GPU that receive
    those outputs instead of host arrays (used by the multi-GPU gather).
    """
    options = options or EngineOptions()
    options.validate()
    if options.record_history:
        raise ValueError("record_history is not supported by run_many")
    off, var, val = _normalise_sets(graph, evidence_sets)
    n = len(off) - 1
    sel = None if select is None else np.ascontiguousarray(np.asarray(select, dtype=np.int32))
    if sel is not None and len(sel) > 1 and np.any(np.diff(sel) <= 0):
        raise ValueError("select must be strictly ascending variable ids")
    if topk and sel is None:
        raise ValueError("topk needs a selection (the alarm variables)")
    if not _is_parall(strategy):
        if options.precision != "fp64":
            raise ValueError("fp32 mode needs the PARALL sweep")
        return _run_materialised(graph, off, var, val, strategy, options, marginals, deltas, sel,
                                 topk)
    device_out = device_out or {}
    dg = device_graph(graph)
    sw = dg.sweep(capacity)
    V = graph.num_variables
    res = (_native.SetResult * max(1, n))()
    outs = _native.SweepOutputs()
    outs.sets = C.cast(res, C.POINTER(_native.SetResult))
    dl = np.zeros((n, options.max_iterations), dtype=np.float64) if deltas else None
    outs.deltas = None if dl is None else _native.ptr(dl, C.c_double)
    mg = None
    if "marginals" in device_out:
        outs.marginals = C.cast(C.c_void_p(device_out["marginals"].data_ptr()), _native.f64p)
        outs.marginals_on_device = 1
    elif marginals:
        mg = _host_empty((n, V, 2), np.float64)
        outs.marginals = _native.ptr(mg, C.c_double)
    p1 = rk = None
    if sel is not None:
        outs.num_select = len(sel)
        outs.select = _native.ptr(sel, C.c_int32)
        if "p1_select" in device_out:
            outs.p1_select = C.cast(C.c_void_p(device_out["p1_select"].data_ptr()), _native.f64p)
            outs.p1_on_device = 1
        else:
            p1 = _host_empty((n, len(sel)), np.float64)
            outs.p1_select = _native.ptr(p1, C.c_double)
        if topk:
            outs.topk = int(topk)
            if "ranked" in device_out:
                outs.ranked = C.cast(C.c_void_p(device_out["ranked"].data_ptr()), _native.i32p)
                outs.ranked_on_device = 1
            else:
                rk = _host_empty((n, topk), np.int32)
                outs.ranked = _native.ptr(rk, C.c_int32)
    ev = _native.Evidence(n, _native.ptr(off, C.c_int64), _native.ptr(var, C.c_int32),
                          _native.ptr(val, C.c_int8))
    opt = _native.Options(int(options.max_iterations), int(bool(options.normalize_messages)), 0,
                          0, float(options.tolerance),
                          float(options.time_limit) if options.time_limit else 0.0,
                          1 if options.precision == "fp32" else 0)
    st = _native.lib().hbp_sweep_run(sw.handle, C.byref(opt), C.byref(ev), C.byref(outs))
    if st != _native.HBP_OK:
        if st == _native.HBP_EINVAL:
            raise ValueError(f"hbp_sweep_run: {_native.last_error()}")
        raise RuntimeError(f"hbp_sweep_run: {_native.last_error()}")
    # the per-set records as one numpy view (no per-set ctypes access)
    rec = np.frombuffer(res, dtype=_SET_RESULT, count=max(1, n))[:n]
    its = rec["iterations"].astype(np.int32)
    uk = rec["underflow_kind"]
    errors: list[Optional[UnderflowError]] = [None] * n
    for j in np.flatnonzero(uk):
        errors[j] = _underflow_error(int(uk[j]), int(rec["underflow_index"][j]),
                                     int(rec["underflow_iteration"][j]))
    base_upd = dg.parall_updates(graph)
    return SweepResult(
        iterations=its,
        converged=rec["converged"] != 0,
        last_delta=rec["last_delta"].astype(np.float64),
        deltas=None if dl is None else [dl[j, :its[j]].tolist() for j in range(n)],
        marginals=mg, p1_select=p1, ranked=rk, select=sel, errors=errors,
        updates_per_iteration=base_upd + np.diff(off),
        device_ms=float(outs.device_ms), kernel_ms=float(outs.kernel_ms),
        launches=int(outs.launches), passes=int(outs.passes),
        compactions=int(outs.compactions))


# numpy layout of _native.SetResult (hbp_set_result)
_SET_RESULT = np.dtype({"names": [f[0] for f in _native.SetResult._fields_],
                        "formats": [np.int32, np.int32, np.float64, np.int32, np.int32, np.int64],
                        "offsets": [getattr(_native.SetResult, f[0]).offset
                                    for f in _native.SetResult._fields_],
                        "itemsize": C.sizeof(_native.SetResult)})


def _run_materialised(graph, off, var, val, strategy, options, want_marg, want_deltas, sel, topk):
    """Non-PARALL strategies: clamp + compile + run per set on the device."""
    from .ranking import AlarmSet, rank_alarms

    n = len(off) - 1
    its, conv, last, dls, margs, p1s, rks, errs, upd = [], [], [], [], [], [], [], [], []
    for j in range(n):
        cur = graph
        for v, o in zip(var[off[j]:off[j + 1]].tolist(), val[off[j]:off[j + 1]].tolist()):
            cur = clamp_evidence(cur, int(v), bool(o))
        sched = strategy.compile(cur)
        upd.append(sched.updates_per_iteration())
        try:
            r = run(cur, sched, options)
        except UnderflowError as exc:
            its.append(0), conv.append(False), last.append(np.nan), dls.append([])
            margs.append(np.full((graph.num_variables, 2), np.nan))
            errs.append(exc)
            if sel is not None:
                p1s.append(np.full(len(sel), np.nan))
                rks.append(np.full(topk, -1, dtype=np.int32))
            continue
        its.append(r.iterations), conv.append(r.converged), last.append(r.last_delta)
        dls.append(r.deltas), margs.append(r.marginals), errs.append(None)
        if sel is not None:
            p1s.append(r.marginals[sel, 1])
            if topk:
                alarms = AlarmSet(tuple(sel.tolist()), tuple([False] * len(sel)))
                ranked = rank_alarms(r.marginals, alarms, var[off[j]:off[j + 1]].tolist())[:topk]
                rks.append(np.array(ranked + [-1] * (topk - len(ranked)), dtype=np.int32))
    return SweepResult(
        iterations=np.array(its, dtype=np.int32), converged=np.array(conv, dtype=bool),
        last_delta=np.array(last, dtype=np.float64), deltas=dls if want_deltas else None,
        marginals=np.stack(margs) if want_marg and n else None,
        p1_select=np.stack(p1s) if sel is not None and n else None,
        ranked=np.stack(rks) if topk and n else None, select=sel, errors=errs,
        updates_per_iteration=np.array(upd, dtype=np.int64))
