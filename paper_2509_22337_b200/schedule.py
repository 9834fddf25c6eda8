"""Update strategies -> dependency-analysed batches (drop-in for hornbp/schedule.py).

The user-facing objects (``Strategy``, ``UpdatePoset``, ``Schedule``) keep the
reference's names, constructors, error types and semantics. The work is done
by the native compiler (``csrc/compiler.cpp`` via ``hbp_compile``): the
ordering relation travels as two int32 arrays of canonical edge indices, the
batches come back as CSR arrays, and the ``EdgeId`` tuple-of-tuples the
reference exposes are only materialised if a caller reads them. The engine
consumes the arrays directly, so compiling PARALL or canonical SEQFIX at ftp
scale never builds per-edge Python objects.

Batch identity with the reference (``compile_schedule``, schedule.py:335) is
pinned by tests/test_schedule.py on the BASELINE configurations and on random
posets.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _native
from .graph import EdgeId, FactorGraph, GraphError

STRATEGY_NAMES = ("PARALL", "SEQFIX", "TOPO", "CUSTOM")


class ScheduleError(ValueError):
    """Invalid strategy, ordering relation, or schedule."""


def _neighbor_indices(graph: FactorGraph, e: int) -> np.ndarray:
    """Canonical indices of N_E(e): edges (a*, v*) with v* another variable of
    e's factor a and a* != a (Def. 4; schedule.py:35-52)."""
    rp, ved = graph._var_csr()
    fac = int(np.searchsorted(graph.rowptr, e, side="right") - 1)
    lo, hi = int(graph.rowptr[fac]), int(graph.rowptr[fac + 1])
    out = []
    for q in range(lo, hi):
        if q == e:
            continue
        v = int(graph.vars[q])
        row = ved[rp[v]:rp[v + 1]]
        row_f = np.searchsorted(graph.rowptr, row, side="right") - 1
        out.append(row[row_f != fac])
    return np.concatenate(out) if out else np.empty(0, dtype=np.int64)


def edge_neighbors(graph: FactorGraph, edge: EdgeId) -> set[EdgeId]:
    """Edges whose factor-to-variable messages feed this edge's update."""
    graph.check_edge(edge)
    return set(graph.edges_at(_neighbor_indices(graph, graph.edge_index(edge))))


class UpdatePoset:
    """Strict partial order over a graph's edges, given by covering pairs.

    Same contract as the reference (schedule.py:55-155): self pairs are
    rejected, duplicates dropped, cycles raise ScheduleError at construction,
    ``rank`` is the total-order shortcut for fixed sequences.
    """

    def __init__(self, graph: FactorGraph, pairs: Iterable[tuple[EdgeId, EdgeId]],
                 rank: Optional[dict] = None):
        pairs = list(pairs)
        if pairs:
            arr = np.asarray([(b[0], b[1], a[0], a[1]) for b, a in pairs], dtype=np.int64)
            before = graph.edge_indices(arr[:, :2])
            after = graph.edge_indices(arr[:, 2:])
        else:
            before = after = np.empty(0, dtype=np.int64)
        rank_arr = None
        if rank is not None:
            rank_arr = np.empty(graph.num_edges, dtype=np.int64)
            keys = list(rank.keys())
            rank_arr[graph.edge_indices(keys)] = np.fromiter(rank.values(), dtype=np.int64,
                                                             count=len(keys))
        self._setup(graph, before, after, rank_arr)

    @classmethod
    def _from_indices(cls, graph, before, after, rank=None) -> "UpdatePoset":
        self = cls.__new__(cls)
        self._setup(graph, np.asarray(before, dtype=np.int64), np.asarray(after, dtype=np.int64),
                    None if rank is None else np.asarray(rank, dtype=np.int64))
        return self

    def _setup(self, graph, before, after, rank) -> None:
        self.graph = graph
        if len(before):
            same = before == after
            if same.any():
                e = graph.edge_at(int(before[np.flatnonzero(same)[0]]))
                raise ScheduleError(f"edge {e} cannot precede itself")
            key = before * graph.num_edges + after
            _, first = np.unique(key, return_index=True)
            keep = np.sort(first)
            before, after = before[keep], after[keep]
        self._before = before.astype(np.int32)
        self._after = after.astype(np.int32)
        self._rank = None if rank is None else rank.astype(np.int32)
        self._pairs = None
        self._pred = None
        try:
            self._order = _native.toposort(graph.num_edges, self._before, self._after)
        except _native.NativeError as exc:
            if exc.status != _native.HBP_ECYCLE:
                raise
            stuck = graph.edge_at(exc.cycle_edge)
            raise ScheduleError(f"ordering relation has a cycle through edge {stuck}") from None
        self._pos = None

    @property
    def pairs(self) -> tuple[tuple[EdgeId, EdgeId], ...]:
        if self._pairs is None:
            b = self.graph.edges_at(self._before)
            a = self.graph.edges_at(self._after)
            self._pairs = tuple(zip(b, a))
        return self._pairs

    def sorted_edges(self) -> list[EdgeId]:
        return self.graph.edges_at(self._order)

    @property
    def has_order(self) -> bool:
        return len(self._before) > 0

    def precedes(self, before: EdgeId, after: EdgeId) -> bool:
        """Whether ``before < after`` in the transitive closure."""
        b = self.graph.edge_index(before)
        a = self.graph.edge_index(after)
        return self._precedes_idx(b, a)

    def _precedes_idx(self, b: int, a: int) -> bool:
        if b == a:
            return False
        if self._rank is not None:
            return bool(self._rank[b] < self._rank[a])
        if self._pred is None:
            n = self.graph.num_edges
            order = np.argsort(self._after, kind="stable")
            self._pred_ptr = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(np.bincount(self._after, minlength=n), out=self._pred_ptr[1:])
            self._pred = self._before[order]
            self._pos = np.empty(n, dtype=np.int64)
            self._pos[self._order] = np.arange(n)
        # any path b -> ... -> a stays inside [pos(b), pos(a)] of the topo order
        lo = self._pos[b]
        if lo >= self._pos[a]:
            return False
        seen = {a}
        stack = [a]
        while stack:
            x = stack.pop()
            for y in self._pred[self._pred_ptr[x]:self._pred_ptr[x + 1]].tolist():
                if y == b:
                    return True
                if y not in seen and self._pos[y] > lo:
                    seen.add(y)
                    stack.append(y)
        return False


def delta(poset: UpdatePoset, e1: EdgeId, e2: EdgeId) -> int:
    """1 iff updating e1 reads e2's current-iteration value (schedule.py:158-167)."""
    poset.graph.check_edge(e1)
    poset.graph.check_edge(e2)
    if e2 in edge_neighbors(poset.graph, e1) and poset.precedes(e2, e1):
        return 1
    return 0


def parall_poset(graph: FactorGraph) -> UpdatePoset:
    return UpdatePoset._from_indices(graph, [], [])


def seqfix_poset(graph: FactorGraph, order: Optional[Sequence[EdgeId]] = None) -> UpdatePoset:
    """Chain over a fixed sequence, canonical order if omitted (schedule.py:175-188)."""
    n = graph.num_edges
    if order is None:
        seq = np.arange(n, dtype=np.int64)
    else:
        seq = graph.edge_indices(list(order)) if len(order) else np.empty(0, dtype=np.int64)
        if len(seq) != n or not np.array_equal(np.sort(seq), np.arange(n)):
            raise ScheduleError("SEQFIX order must be a permutation of all edges")
    rank = np.empty(n, dtype=np.int64)
    rank[seq] = np.arange(n)
    return UpdatePoset._from_indices(graph, seq[:-1], seq[1:], rank)


def topo_poset(graph: FactorGraph) -> UpdatePoset:
    """Two-phase tree order: leaves-to-root then root-to-leaves (schedule.py:191-251).
    Requires a forest; a cycle raises ScheduleError naming the closing edge."""
    nv = graph.num_variables
    nodes = nv + graph.num_factors
    fac = graph.edge_factor()
    var = graph.vars.astype(np.int64)
    nbr: list[list[tuple[int, int]]] = [[] for _ in range(nodes)]
    for e, (v, f) in enumerate(zip(var.tolist(), fac.tolist())):
        nbr[v].append((nv + f, e))
        nbr[nv + f].append((v, e))
    depth = [-1] * nodes
    for root in range(nv):
        if depth[root] != -1:
            continue
        depth[root] = 0
        parent: dict[int, int] = {}
        queue = deque([root])
        while queue:
            node = queue.popleft()
            for other, e in nbr[node]:
                if depth[other] == -1:
                    depth[other] = depth[node] + 1
                    parent[other] = e
                    queue.append(other)
                elif parent.get(node) != e:
                    raise ScheduleError(
                        f"graph has a cycle through edge {graph.edge_at(e)}; "
                        "TOPO requires a tree-structured graph")
    dep = np.asarray(depth, dtype=np.int64)
    dv = dep[var]
    df = dep[nv + fac]
    idx = np.arange(graph.num_edges)
    inward = idx[dv < df]
    outward = idx[dv >= df]
    inward = inward[np.lexsort((inward, -df[inward]))]
    outward = outward[np.lexsort((outward, dv[outward]))]
    linear = np.concatenate([inward, outward])
    position = np.empty(graph.num_edges, dtype=np.int64)
    position[linear] = np.arange(len(linear))
    before, after = [], []
    for e in linear.tolist():
        nb = _neighbor_indices(graph, e)
        nb = nb[position[nb] < position[e]]
        before.extend(nb.tolist())
        after.extend([e] * len(nb))
    return UpdatePoset._from_indices(graph, before, after)


def custom_poset(graph: FactorGraph, pairs: Iterable[tuple[EdgeId, EdgeId]]) -> UpdatePoset:
    return UpdatePoset(graph, pairs)


class Schedule:
    """Compiled plan: aligned factor-to-variable (s) / variable-to-factor (t)
    batches. Constructible from EdgeId tuples like the reference dataclass
    (schedule.py:315-332); compiled schedules carry CSR arrays of canonical
    edge indices and build the tuples lazily."""

    __slots__ = ("_s", "_t", "_arr", "_rowptr", "_graph_ref", "__weakref__")

    def __init__(self, s_batches, t_batches):
        self._s = tuple(tuple(EdgeId(*e) for e in b) for b in s_batches)
        self._t = tuple(tuple(EdgeId(*e) for e in b) for b in t_batches)
        self._arr = None
        self._rowptr = None
        self._graph_ref = None

    @classmethod
    def _from_arrays(cls, graph: FactorGraph, s_off, s_edges, t_off, t_edges) -> "Schedule":
        self = cls.__new__(cls)
        self._s = None
        self._t = None
        self._arr = (np.asarray(s_off, dtype=np.int64), np.asarray(s_edges, dtype=np.int32),
                     np.asarray(t_off, dtype=np.int64), np.asarray(t_edges, dtype=np.int32))
        self._rowptr = graph.rowptr
        self._graph_ref = graph
        return self

    def _materialize(self, which: int):
        off, edges = self._arr[2 * which], self._arr[2 * which + 1]
        rp = self._rowptr
        f = np.searchsorted(rp, edges, side="right") - 1
        ids = list(map(EdgeId, f.tolist(), (edges - rp[f]).tolist()))
        o = off.tolist()
        return tuple(tuple(ids[o[i]:o[i + 1]]) for i in range(len(o) - 1))

    @property
    def s_batches(self) -> tuple[tuple[EdgeId, ...], ...]:
        if self._s is None:
            self._s = self._materialize(0)
        return self._s

    @property
    def t_batches(self) -> tuple[tuple[EdgeId, ...], ...]:
        if self._t is None:
            self._t = self._materialize(1)
        return self._t

    @property
    def num_batches(self) -> int:
        return len(self._arr[0]) - 1 if self._arr is not None else len(self._s)

    def batch_index(self) -> dict[EdgeId, int]:
        index: dict[EdgeId, int] = {}
        for i, batch in enumerate(self.s_batches):
            for edge in batch:
                index[edge] = i
        return index

    def batch_sizes(self) -> list[int]:
        if self._arr is not None:
            return np.diff(self._arr[0]).tolist()
        return [len(b) for b in self._s]

    def updates_per_iteration(self) -> int:
        """sum |s_i| + sum |t_i|, the bench metric's numerator (cli.py:337-339)."""
        if self._arr is not None:
            return int(len(self._arr[1]) + len(self._arr[3]))
        return sum(map(len, self._s)) + sum(map(len, self._t))

    def arrays(self, graph: FactorGraph):
        """(s_off, s_edges, t_off, t_edges) as canonical indices of ``graph``.
        Schedules compiled for a graph stay valid for graphs that only append
        factors (clamp_evidence keeps every existing edge index)."""
        if self._arr is not None:
            rp = self._rowptr
            if graph.rowptr is rp or (len(graph.rowptr) >= len(rp)
                                      and np.array_equal(graph.rowptr[:len(rp)], rp)):
                return self._arr
        arrs = []
        for batches in (self.s_batches, self.t_batches):
            off = np.zeros(len(batches) + 1, dtype=np.int64)
            np.cumsum([len(b) for b in batches], out=off[1:])
            flat = [e for b in batches for e in b]
            idx = graph.edge_indices(flat) if flat else np.empty(0, dtype=np.int64)
            arrs += [off, idx.astype(np.int32)]
        return tuple(arrs)

    def __eq__(self, other) -> bool:
        if not isinstance(other, Schedule):
            return NotImplemented
        return self.s_batches == other.s_batches and self.t_batches == other.t_batches

    def __hash__(self) -> int:
        return hash((self.s_batches, self.t_batches))

    def __repr__(self) -> str:
        return f"Schedule(num_batches={self.num_batches}, sizes={self.batch_sizes()[:8]}...)"


def _compile_poset(graph: FactorGraph, poset: UpdatePoset) -> Schedule:
    try:
        arrs = _native.compile_arrays(graph, poset._before, poset._after, poset._rank)
    except _native.NativeError as exc:
        if exc.status == _native.HBP_ECYCLE:
            raise ScheduleError(
                f"ordering relation has a cycle through edge {graph.edge_at(exc.cycle_edge)}") from None
        raise
    return Schedule._from_arrays(graph, *arrs)


def dependency_analysis(poset: UpdatePoset) -> list[list[EdgeId]]:
    """Alg. 2 batches (schedule.py:261-290), computed natively."""
    return [list(b) for b in _compile_poset(poset.graph, poset).s_batches]


def group_var_to_factor(graph: FactorGraph, s_batches: Sequence[Sequence[EdgeId]]
                        ) -> list[list[EdgeId]]:
    """Alg. 3 companion batches (schedule.py:293-312)."""
    out = []
    for batch in s_batches:
        if not batch:
            out.append([])
            continue
        idx = graph.edge_indices(list(batch))
        fac = np.searchsorted(graph.rowptr, idx, side="right") - 1
        slots = []
        for f in np.unique(fac).tolist():
            own = set(idx[fac == f].tolist())
            lo, hi = int(graph.rowptr[f]), int(graph.rowptr[f + 1])
            slots.extend(q for q in range(lo, hi) if len(own) > 1 or q not in own)
        out.append(graph.edges_at(sorted(slots)))
    return out


def compile_schedule(graph: FactorGraph, poset: UpdatePoset) -> Schedule:
    return _compile_poset(graph, poset)


def verify_batches(poset: UpdatePoset, s_batches: Sequence[Sequence[EdgeId]]
                   ) -> list[tuple[EdgeId, EdgeId]]:
    """Theorem-2 check (schedule.py:344-362): every ordered feeding message
    must sit in an earlier batch. Returns the violating (edge, dependency)."""
    graph = poset.graph
    batch_of = np.full(graph.num_edges, -1, dtype=np.int64)
    placed = []
    for i, batch in enumerate(s_batches):
        if batch:
            idx = graph.edge_indices(list(batch))
            batch_of[idx] = i
            placed.append(idx)
    bad = []
    for idx in placed:
        for e in idx.tolist():
            i = batch_of[e]
            for o in _neighbor_indices(graph, e).tolist():
                if batch_of[o] >= i and poset._precedes_idx(o, e):
                    bad.append((graph.edge_at(e), graph.edge_at(o)))
    return bad


def _parse_edge_token(token: str, lineno: int) -> EdgeId:
    parts = token.split(":")
    if len(parts) != 2:
        raise ScheduleError(f"line {lineno}: expected <factor>:<slot>, got {token!r}")
    try:
        return EdgeId(int(parts[0]), int(parts[1]))
    except ValueError:
        raise ScheduleError(f"line {lineno}: bad edge token {token!r}") from None


@dataclass(frozen=True)
class Strategy:
    """Named update strategy (schedule.py:375-475)."""

    kind: str
    order: Optional[tuple[EdgeId, ...]] = None
    pairs: Optional[tuple[tuple[EdgeId, EdgeId], ...]] = None

    def __post_init__(self):
        if self.kind not in STRATEGY_NAMES:
            raise ScheduleError(f"unknown strategy {self.kind!r}")

    @classmethod
    def parall(cls) -> "Strategy":
        return cls("PARALL")

    @classmethod
    def seqfix(cls, order: Optional[Sequence[EdgeId]] = None) -> "Strategy":
        return cls("SEQFIX", order=tuple(order) if order is not None else None)

    @classmethod
    def topo(cls) -> "Strategy":
        return cls("TOPO")

    @classmethod
    def custom(cls, pairs: Iterable[tuple[EdgeId, EdgeId]]) -> "Strategy":
        return cls("CUSTOM", pairs=tuple(pairs))

    @classmethod
    def from_name(cls, name: str) -> "Strategy":
        name = name.upper()
        if name == "CUSTOM":
            raise ScheduleError("CUSTOM strategy needs a strategy file")
        if name not in STRATEGY_NAMES:
            raise ScheduleError(f"unknown strategy {name!r}")
        return cls(name)

    @classmethod
    def from_text(cls, text: str) -> "Strategy":
        """``strategy X`` then ``edge f:s`` (SEQFIX) / ``before f:s f:s`` (CUSTOM)."""
        kind: Optional[str] = None
        order: list[EdgeId] = []
        pairs: list[tuple[EdgeId, EdgeId]] = []
        for lineno, raw in enumerate(text.splitlines(), start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if kind is None:
                if len(tok) != 2 or tok[0] != "strategy":
                    raise ScheduleError(
                        f"line {lineno}: expected 'strategy <PARALL|SEQFIX|TOPO|CUSTOM>'")
                if tok[1] not in STRATEGY_NAMES:
                    raise ScheduleError(f"line {lineno}: unknown strategy {tok[1]!r}")
                kind = tok[1]
            elif tok[0] == "edge":
                if kind != "SEQFIX":
                    raise ScheduleError(f"line {lineno}: 'edge' lines need strategy SEQFIX")
                if len(tok) != 2:
                    raise ScheduleError(f"line {lineno}: expected 'edge <factor>:<slot>'")
                order.append(_parse_edge_token(tok[1], lineno))
            elif tok[0] == "before":
                if kind != "CUSTOM":
                    raise ScheduleError(f"line {lineno}: 'before' lines need strategy CUSTOM")
                if len(tok) != 3:
                    raise ScheduleError(
                        f"line {lineno}: expected 'before <factor>:<slot> <factor>:<slot>'")
                pairs.append((_parse_edge_token(tok[1], lineno), _parse_edge_token(tok[2], lineno)))
            else:
                raise ScheduleError(f"line {lineno}: unknown directive {tok[0]!r}")
        if kind is None:
            raise ScheduleError("strategy file is empty")
        if kind == "SEQFIX":
            return cls.seqfix(order if order else None)
        if kind == "CUSTOM":
            return cls.custom(pairs)
        return cls(kind)

    def build_poset(self, graph: FactorGraph) -> UpdatePoset:
        if self.kind == "PARALL":
            return parall_poset(graph)
        if self.kind == "SEQFIX":
            return seqfix_poset(graph, self.order)
        if self.kind == "TOPO":
            return topo_poset(graph)
        return custom_poset(graph, self.pairs or ())

    def compile(self, graph: FactorGraph) -> Schedule:
        return compile_schedule(graph, self.build_poset(graph))
