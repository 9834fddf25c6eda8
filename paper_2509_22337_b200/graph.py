"""Binary AND/OR factor graphs, held as flat arrays.

Drop-in for the reference data model (``hornbp/graph.py:38-200``): the same
``FactorGraph`` / ``Factor`` / ``EdgeId`` / ``FactorKind`` names, validation
rules and error types, the FASTFG text format (``graph.py:203-287``), the
clause/tuple/input DAG conversion (``graph.py:290-417``) and evidence
clamping (``graph.py:189-200``).

The representation is different. A graph is four flat arrays in canonical
factor-major edge order, which is exactly the order the device layout and
the strategy compiler consume:

* ``kind[F]`` (int8, 0 = AND, 1 = OR), ``p1[F]``, ``p2[F]`` (float64)
* ``rowptr[F+1]`` (int64): factor ``f`` owns canonical edges
  ``rowptr[f] .. rowptr[f+1]-1``; slot 0 is the head
* ``vars[E]`` (int32): the variable at each canonical edge

A canonical edge index is also the reference's variable-to-factor buffer
position (``storage.py:45-52``), so ``EdgeId(f, s)`` <-> ``rowptr[f] + s``.
``Factor`` objects and the per-variable adjacency are materialised lazily,
only when a caller asks for them; building an ftp-scale graph therefore
costs array operations, not 211k Python objects.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Iterator, NamedTuple, Optional, Sequence

import numpy as np

KIND_AND = 0
KIND_OR = 1


class GraphError(ValueError):
    """Invalid factor graph structure or parameters."""


class FormatError(GraphError):
    """Malformed input text; carries the 1-based line number."""

    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line


class FactorKind(Enum):
    AND = "AND"
    OR = "OR"


_KIND_CODE = {FactorKind.AND: KIND_AND, FactorKind.OR: KIND_OR}
_CODE_KIND = (FactorKind.AND, FactorKind.OR)


class EdgeId(NamedTuple):
    """Edge named by (factor index, slot); slot 0 is the head variable."""

    factor: int
    slot: int

    def __str__(self) -> str:
        return f"{self.factor}:{self.slot}"


@dataclass(frozen=True)
class Factor:
    kind: FactorKind
    head: int
    body: tuple[int, ...]
    p1: float
    p2: float

    @property
    def arity(self) -> int:
        return len(self.body)

    @property
    def degree(self) -> int:
        return len(self.body) + 1

    def variables(self) -> tuple[int, ...]:
        return (self.head,) + self.body


def _factor_problem(index: int, kind: int, head: int, body, p1: float, p2: float,
                    num_variables: int) -> Optional[str]:
    """First violated rule for one factor, in the reference's check order
    (``graph.py:121-140``); None when the factor is valid."""
    label = f"factor {index}"
    for var in (head,) + tuple(body):
        if not 0 <= var < num_variables:
            return f"{label}: variable {var} out of range"
    if head in body:
        return f"{label}: head variable repeated in body"
    if len(set(body)) != len(body):
        return f"{label}: duplicate body variable"
    for name, p in (("p1", p1), ("p2", p2)):
        if not 0.0 <= p <= 1.0:
            return f"{label}: {name}={p} outside [0, 1]"
    if not body:
        if kind == KIND_OR:
            return f"{label}: OR factor with empty body has no meaning"
        if p1 != p2:
            return (f"{label}: body-empty factor requires p1 == p2 "
                    f"(got {p1}, {p2})")
    return None


class FactorGraph:
    """Immutable bipartite graph of binary variables and AND/OR factors.

    ``FactorGraph(num_variables, factors, names=None)`` accepts ``Factor``
    objects exactly like the reference; :meth:`from_arrays` builds one
    straight from the flat arrays (the fast path used by the generator,
    the parsers and :func:`clamp_evidence`).
    """

    __slots__ = ("num_variables", "names", "kind", "p1", "p2", "rowptr", "vars",
                 "_factors", "_adjacency", "_var_rowptr", "_var_edges",
                 "__weakref__")

    def __init__(self, num_variables: int, factors: Sequence[Factor],
                 names: Optional[Sequence[str]] = None):
        factors = tuple(factors)
        n = len(factors)
        kind = np.empty(n, dtype=np.int8)
        p1 = np.empty(n, dtype=np.float64)
        p2 = np.empty(n, dtype=np.float64)
        rowptr = np.zeros(n + 1, dtype=np.int64)
        flat: list[int] = []
        for i, f in enumerate(factors):
            kind[i] = _KIND_CODE[f.kind]
            p1[i] = f.p1
            p2[i] = f.p2
            flat.append(f.head)
            flat.extend(f.body)
            rowptr[i + 1] = len(flat)
        self._init(num_variables, kind, p1, p2, rowptr,
                   np.asarray(flat, dtype=np.int64), names)
        self._factors = factors

    @classmethod
    def from_arrays(cls, num_variables: int, kind, p1, p2, rowptr, vars_,
                    names: Optional[Sequence[str]] = None) -> "FactorGraph":
        self = cls.__new__(cls)
        self._init(num_variables, np.asarray(kind, dtype=np.int8),
                   np.asarray(p1, dtype=np.float64), np.asarray(p2, dtype=np.float64),
                   np.asarray(rowptr, dtype=np.int64), np.asarray(vars_, dtype=np.int64),
                   names)
        return self

    def _init(self, num_variables, kind, p1, p2, rowptr, flat, names) -> None:
        if num_variables < 0:
            raise GraphError("variable count must be nonnegative")
        if names is not None and len(names) != num_variables:
            raise GraphError("names table must have one entry per variable")
        self.num_variables = int(num_variables)
        self.names = tuple(names) if names else None
        self._factors = None
        self._adjacency = None
        self._var_rowptr = None
        self._var_edges = None
        self._validate(kind, p1, p2, rowptr, flat)
        self.kind = kind
        self.p1 = p1
        self.p2 = p2
        self.rowptr = rowptr
        self.vars = flat.astype(np.int32)
        for arr in (self.kind, self.p1, self.p2, self.rowptr, self.vars):
            arr.flags.writeable = False

    def _validate(self, kind, p1, p2, rowptr, flat) -> None:
        """Vectorised form of the reference checks; on failure, re-derive the
        first offending factor's message in the reference's order."""
        n = len(kind)
        nv = self.num_variables
        deg = np.diff(rowptr)
        bad = np.zeros(n, dtype=bool)
        if len(flat):
            owner = np.repeat(np.arange(n), deg)
            out = (flat < 0) | (flat >= nv)
            if out.any():
                bad[owner[out]] = True
            # head or body repeated within a factor: sort each row, look for
            # equal neighbours (row id as the major key).
            order = np.lexsort((flat, owner))
            so, sf = owner[order], flat[order]
            dup = (so[1:] == so[:-1]) & (sf[1:] == sf[:-1])
            if dup.any():
                bad[so[1:][dup]] = True
        bad |= ~((p1 >= 0.0) & (p1 <= 1.0)) | ~((p2 >= 0.0) & (p2 <= 1.0))
        empty = deg == 1
        bad |= empty & ((kind == KIND_OR) | (p1 != p2))
        bad |= deg < 1
        if bad.any():
            i = int(np.flatnonzero(bad)[0])
            lo, hi = int(rowptr[i]), int(rowptr[i + 1])
            if hi <= lo:
                raise GraphError(f"factor {i}: no head variable")
            msg = _factor_problem(i, int(kind[i]), int(flat[lo]),
                                  tuple(int(v) for v in flat[lo + 1:hi]),
                                  float(p1[i]), float(p2[i]), nv)
            raise GraphError(msg or f"factor {i}: invalid")
        if nv:
            seen = np.zeros(nv, dtype=bool)
            seen[flat] = True
            if not seen.all():
                raise GraphError(f"variable {int(np.flatnonzero(~seen)[0])} appears in no factor")

    # ---- reference-compatible surface -------------------------------------------------
    @property
    def num_factors(self) -> int:
        return len(self.kind)

    @property
    def num_edges(self) -> int:
        return len(self.vars)

    @property
    def factors(self) -> tuple[Factor, ...]:
        if self._factors is None:
            rp = self.rowptr.tolist()
            fl = self.vars.tolist()
            kinds = self.kind.tolist()
            p1 = self.p1.tolist()
            p2 = self.p2.tolist()
            self._factors = tuple(
                Factor(_CODE_KIND[kinds[i]], fl[rp[i]], tuple(fl[rp[i] + 1:rp[i + 1]]),
                       p1[i], p2[i])
                for i in range(len(kinds)))
        return self._factors

    def _var_csr(self) -> tuple[np.ndarray, np.ndarray]:
        """Per-variable rows of canonical edge indices, ordered by (factor,
        slot) -- the reference's adjacency order (``graph.py:105-118``)."""
        if self._var_rowptr is None:
            counts = np.bincount(self.vars, minlength=self.num_variables)
            rp = np.zeros(self.num_variables + 1, dtype=np.int64)
            np.cumsum(counts, out=rp[1:])
            self._var_rowptr = rp
            self._var_edges = np.argsort(self.vars, kind="stable").astype(np.int64)
        return self._var_rowptr, self._var_edges

    @property
    def adjacency(self) -> tuple[tuple[tuple[int, int], ...], ...]:
        if self._adjacency is None:
            rp, ed = self._var_csr()
            fac = self.edge_factor()
            slot = ed - self.rowptr[fac[ed]]
            pairs = list(zip(fac[ed].tolist(), slot.tolist()))
            rpl = rp.tolist()
            self._adjacency = tuple(tuple(pairs[rpl[v]:rpl[v + 1]])
                                    for v in range(self.num_variables))
        return self._adjacency

    def edge_factor(self) -> np.ndarray:
        """Factor index of every canonical edge."""
        return np.repeat(np.arange(self.num_factors, dtype=np.int64), np.diff(self.rowptr))

    def edge_slot(self) -> np.ndarray:
        return np.arange(self.num_edges, dtype=np.int64) - np.repeat(self.rowptr[:-1], np.diff(self.rowptr))

    def edges(self) -> Iterator[EdgeId]:
        rp = self.rowptr.tolist()
        for fi in range(self.num_factors):
            for slot in range(rp[fi + 1] - rp[fi]):
                yield EdgeId(fi, slot)

    def edge_list(self) -> list[EdgeId]:
        return list(self.edges())

    def edge_index(self, edge: EdgeId) -> int:
        """Canonical index (= reference vtof position) of an edge."""
        self.check_edge(edge)
        return int(self.rowptr[edge[0]]) + int(edge[1])

    def edge_indices(self, edges) -> np.ndarray:
        """Vectorised :meth:`edge_index`; raises GraphError on bad edges."""
        if len(edges) == 0:
            return np.empty(0, dtype=np.int64)
        arr = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        f, s = arr[:, 0], arr[:, 1]
        if f.min() < 0 or f.max() >= self.num_factors:
            bad = int(np.flatnonzero((f < 0) | (f >= self.num_factors))[0])
            raise GraphError(f"edge {f[bad]}:{s[bad]}: factor index out of range")
        deg = self.rowptr[f + 1] - self.rowptr[f]
        if s.min() < 0 or np.any(s >= deg):
            bad = int(np.flatnonzero((s < 0) | (s >= deg))[0])
            raise GraphError(f"edge {f[bad]}:{s[bad]}: slot out of range")
        return self.rowptr[f] + s

    def edge_at(self, index: int) -> EdgeId:
        f = int(np.searchsorted(self.rowptr, index, side="right") - 1)
        return EdgeId(f, int(index - self.rowptr[f]))

    def edges_at(self, indices) -> list[EdgeId]:
        idx = np.asarray(indices, dtype=np.int64)
        f = np.searchsorted(self.rowptr, idx, side="right") - 1
        return [EdgeId(a, b) for a, b in zip(f.tolist(), (idx - self.rowptr[f]).tolist())]

    def variable_of(self, edge: EdgeId) -> int:
        if not 0 <= edge[0] < self.num_factors:
            raise GraphError(f"edge {EdgeId(*edge)}: factor index out of range")
        lo, hi = int(self.rowptr[edge[0]]), int(self.rowptr[edge[0] + 1])
        if not 0 <= edge[1] < hi - lo:
            raise GraphError(f"edge {EdgeId(*edge)}: slot out of range")
        return int(self.vars[lo + edge[1]])

    def check_edge(self, edge: EdgeId) -> EdgeId:
        if not 0 <= edge[0] < self.num_factors:
            raise GraphError(f"edge {EdgeId(*edge)}: factor index out of range")
        if not 0 <= edge[1] < int(self.rowptr[edge[0] + 1] - self.rowptr[edge[0]]):
            raise GraphError(f"edge {EdgeId(*edge)}: slot out of range")
        return edge

    def degree_of_variable(self, var: int) -> int:
        rp, _ = self._var_csr()
        return int(rp[var + 1] - rp[var])

    def name_of(self, var: int) -> str:
        return self.names[var] if self.names is not None else str(var)

    def to_fastfg(self) -> str:
        """FASTFG serialisation, byte-identical to the reference's
        (``graph.py:177-186``: ``repr`` of the probabilities)."""
        rp = self.rowptr.tolist()
        fl = self.vars.tolist()
        kinds = self.kind.tolist()
        p1 = self.p1.tolist()
        p2 = self.p2.tolist()
        names = ("AND", "OR")
        out = ["FASTFG 1", f"vars {self.num_variables}"]
        for i in range(len(kinds)):
            body = ",".join(map(str, fl[rp[i] + 1:rp[i + 1]]))
            out.append(f"factor {names[kinds[i]]} {p1[i]!r} {p2[i]!r} "
                       f"head={fl[rp[i]]} body={body}")
        return "\n".join(out) + "\n"


def clamp_evidence(graph: FactorGraph, variable: int, observed: bool) -> FactorGraph:
    """New graph with ``variable`` pinned: one appended body-empty AND factor
    with p1 = p2 = 1.0 (true) or 0.0 (false); existing edge ids unchanged
    (``graph.py:189-200``)."""
    if not 0 <= variable < graph.num_variables:
        raise GraphError(f"variable {variable} out of range")
    p = 1.0 if observed else 0.0
    out = FactorGraph.__new__(FactorGraph)
    out.num_variables = graph.num_variables
    out.names = graph.names
    out._factors = None if graph._factors is None else graph._factors + (
        Factor(FactorKind.AND, variable, (), p, p),)
    out._adjacency = None
    out._var_rowptr = None
    out._var_edges = None
    out.kind = np.append(graph.kind, np.int8(KIND_AND))
    out.p1 = np.append(graph.p1, p)
    out.p2 = np.append(graph.p2, p)
    out.rowptr = np.append(graph.rowptr, graph.rowptr[-1] + 1)
    out.vars = np.append(graph.vars, np.int32(variable))
    for arr in (out.kind, out.p1, out.p2, out.rowptr, out.vars):
        arr.flags.writeable = False
    return out


# ---- FASTFG ---------------------------------------------------------------------------

def parse_fastfg(text: str) -> FactorGraph:
    """Parse ``FASTFG 1`` / ``vars N`` / ``factor KIND p1 p2 head=v body=v,..``
    lines (``graph.py:203-287``), with the same FormatError line numbers."""
    header_ok = False
    nv: Optional[int] = None
    kinds: list[int] = []
    p1s: list[float] = []
    p2s: list[float] = []
    rowptr = [0]
    flat: list[int] = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        if not header_ok:
            if tok != ["FASTFG", "1"]:
                raise FormatError(lineno, "expected header 'FASTFG 1'")
            header_ok = True
            continue
        if nv is None:
            if len(tok) != 2 or tok[0] != "vars":
                raise FormatError(lineno, "expected 'vars <N>'")
            try:
                nv = int(tok[1])
            except ValueError:
                raise FormatError(lineno, f"bad variable count {tok[1]!r}") from None
            if nv < 0:
                raise FormatError(lineno, "variable count must be nonnegative")
            continue
        kind, pa, pb, head, body = _factor_tokens(lineno, tok, nv)
        kinds.append(kind)
        p1s.append(pa)
        p2s.append(pb)
        flat.append(head)
        flat.extend(body)
        rowptr.append(len(flat))
    if not header_ok:
        raise FormatError(1, "missing 'FASTFG 1' header")
    if nv is None:
        raise FormatError(1, "missing 'vars <N>' line")
    try:
        return FactorGraph.from_arrays(nv, kinds, p1s, p2s, rowptr, flat)
    except GraphError as exc:
        raise GraphError(f"invalid graph: {exc}") from exc


def _factor_tokens(lineno: int, tok: list[str], nv: int):
    if len(tok) != 6 or tok[0] != "factor":
        raise FormatError(lineno, "expected 'factor <AND|OR> <p1> <p2> head=<v> body=<v,...>'")
    try:
        kind = _KIND_CODE[FactorKind(tok[1])]
    except ValueError:
        raise FormatError(lineno, f"unknown factor kind {tok[1]!r}") from None
    probs = []
    for t in tok[2:4]:
        try:
            p = float(t)
        except ValueError:
            raise FormatError(lineno, f"bad probability {t!r}") from None
        if not 0.0 <= p <= 1.0:
            raise FormatError(lineno, f"probability {t} outside [0, 1]")
        probs.append(p)
    if not tok[4].startswith("head="):
        raise FormatError(lineno, "expected head=<v>")
    if not tok[5].startswith("body="):
        raise FormatError(lineno, "expected body=<v,...>")

    def index(t: str) -> int:
        try:
            v = int(t)
        except ValueError:
            raise FormatError(lineno, f"bad variable index {t!r}") from None
        if not 0 <= v < nv:
            raise FormatError(lineno, f"variable index {v} out of range (vars {nv})")
        return v

    head = index(tok[4][5:])
    body = [index(t) for t in tok[5][5:].split(",") if t != ""]
    if head in body:
        raise FormatError(lineno, f"head variable {head} repeated in body")
    if len(set(body)) != len(body):
        raise FormatError(lineno, "duplicate body variable")
    return kind, probs[0], probs[1], head, body


# ---- clause / tuple / input DAGs ------------------------------------------------------

@dataclass(frozen=True)
class DagNode:
    id: str
    role: str  # "clause", "tuple" or "input"
    prob: Optional[float] = None


DEFAULT_CLAUSE_PROB = 0.999


def from_bayesian_dag(nodes: Sequence[DagNode],
                      dag_edges: Sequence[tuple[str, str]]) -> FactorGraph:
    """One variable and one factor per DAG node (``graph.py:302-358``):
    input -> AND prior (p, p); clause -> AND(p, 0) over its premises;
    tuple -> OR(1, 0) over its deriving clauses. Premise order = edge order."""
    pos: dict[str, int] = {}
    for node in nodes:
        if node.role not in ("clause", "tuple", "input"):
            raise GraphError(f"node {node.id}: unknown role {node.role!r}")
        if node.id in pos:
            raise GraphError(f"node {node.id}: declared twice")
        if node.role == "tuple" and node.prob is not None:
            raise GraphError(f"node {node.id}: tuple nodes take no probability")
        pos[node.id] = len(pos)
    n = len(nodes)
    parents: list[list[int]] = [[] for _ in range(n)]
    children: list[list[int]] = [[] for _ in range(n)]
    for src, dst in dag_edges:
        for end in (src, dst):
            if end not in pos:
                raise GraphError(f"edge {src} -> {dst}: unknown node {end!r}")
        parents[pos[dst]].append(pos[src])
        children[pos[src]].append(pos[dst])
    _require_acyclic(nodes, parents, children)

    kind = np.empty(n, dtype=np.int8)
    p1 = np.empty(n)
    p2 = np.empty(n)
    rowptr = [0]
    flat: list[int] = []
    for i, node in enumerate(nodes):
        p = DEFAULT_CLAUSE_PROB if node.prob is None else node.prob
        par = parents[i]
        if node.role == "input":
            if par:
                raise GraphError(f"node {node.id}: input node has premises")
            kind[i], p1[i], p2[i] = KIND_AND, p, p
        elif node.role == "clause":
            if not par:
                raise GraphError(f"node {node.id}: clause node has no premises; use role input")
            kind[i], p1[i], p2[i] = KIND_AND, p, 0.0
        else:
            if not par:
                raise GraphError(f"node {node.id}: tuple node has no deriving clause")
            kind[i], p1[i], p2[i] = KIND_OR, 1.0, 0.0
        flat.append(i)
        flat.extend(par)
        rowptr.append(len(flat))
    return FactorGraph.from_arrays(n, kind, p1, p2, rowptr, flat, [x.id for x in nodes])


def _require_acyclic(nodes, parents, children) -> None:
    indeg = [len(p) for p in parents]
    stack = [i for i, d in enumerate(indeg) if d == 0]
    done = 0
    while stack:
        i = stack.pop()
        done += 1
        for j in children[i]:
            indeg[j] -= 1
            if indeg[j] == 0:
                stack.append(j)
    if done != len(nodes):
        stuck = next(i for i, d in enumerate(indeg) if d > 0)
        raise GraphError(f"input DAG has a cycle through node {nodes[stuck].id}")


def parse_dag(text: str) -> FactorGraph:
    """``node <id> <role> [p=<prob>]`` / ``edge <from> <to>`` lines
    (``graph.py:379-417``)."""
    nodes: list[DagNode] = []
    links: list[tuple[str, str]] = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        if tok[0] == "node":
            if len(tok) not in (3, 4):
                raise FormatError(lineno, "expected 'node <id> <role> [p=<prob>]'")
            prob = None
            if len(tok) == 4:
                if not tok[3].startswith("p="):
                    raise FormatError(lineno, "expected p=<prob>")
                try:
                    prob = float(tok[3][2:])
                except ValueError:
                    raise FormatError(lineno, f"bad probability {tok[3][2:]!r}") from None
                if not 0.0 <= prob <= 1.0:
                    raise FormatError(lineno, f"probability {prob} outside [0, 1]")
            nodes.append(DagNode(tok[1], tok[2], prob))
        elif tok[0] == "edge":
            if len(tok) != 3:
                raise FormatError(lineno, "expected 'edge <from> <to>'")
            links.append((tok[1], tok[2]))
        else:
            raise FormatError(lineno, f"unknown directive {tok[0]!r}")
    try:
        return from_bayesian_dag(nodes, links)
    except GraphError as exc:
        if isinstance(exc, FormatError):
            raise
        raise GraphError(f"invalid DAG: {exc}") from exc
