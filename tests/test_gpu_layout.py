"""The device-built layout (csrc/layout_dev.cu) against the
host builder (csrc/layout.cpp), array by array, and the MessageStore
transpose it must reproduce (storage.py:36-94)."""

import ctypes as C

import numpy as np
import pytest

from builders import hub_graph, random_graph
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import EngineOptions, Strategy, _native, initialize
from paper_2509_22337_b200 import workloads as W

pytestmark = pytest.mark.gpu


def layout_mismatches(g) -> int:
    P.engine.clear_device_cache()
    dg = P.engine.device_graph(g)
    bad = C.c_int64(-1)
    st = _native.lib().hbp_graph_layout_check(dg.handle, C.byref(bad))
    assert st == _native.HBP_OK, _native.last_error()
    return bad.value


@pytest.mark.parametrize("name", ["weblech", "hedc", "avrora", "ftp"])
def test_device_layout_equals_host_layout_workloads(name):
    g, _ = W.graph(name)
    assert layout_mismatches(g) == 0


def test_device_layout_equals_host_layout_random_and_long_rows():
    rng = np.random.default_rng(404)
    for _ in range(40):
        g = random_graph(rng, max_vars=30, max_factors=30, max_body=6, or_prob=0.5)
        assert layout_mismatches(g) == 0
    for hub, wide in [(5, 5), (45, 44), (300, 120)]:
        assert layout_mismatches(hub_graph(rng, hub_degree=hub, wide_body=wide)) == 0


def test_device_layout_reference_transpose():
    g, _ = W.graph("hedc")
    P.engine.clear_device_cache()
    dg = P.engine.device_graph(g)
    V, E = g.num_variables, g.num_edges
    rp = np.empty(V + 1, dtype=np.int64)
    f2v = np.empty(E, dtype=np.int64)
    assert _native.lib().hbp_graph_layout(dg.handle, _native.ptr(rp, C.c_int64),
                                          _native.ptr(f2v, C.c_int64)) == _native.HBP_OK
    store = initialize(g)
    assert np.array_equal(rp, np.asarray(store.rowptr_ftov))
    assert np.array_equal(f2v, np.asarray(store.ftov_to_vtof))


def test_parall_plan_without_host_layout_is_bitwise():
    """run() with PARALL takes the device shape test (no host layout); a
    levelled schedule on the same fresh graph builds the host layout lazily.
    Both must equal the oracle path's results."""
    g, _ = W.graph("avrora")
    opts = EngineOptions(1000, 1e-9)
    P.engine.clear_device_cache()
    a = P.run(g, Strategy.parall().compile(g), opts)
    s = Strategy.seqfix().compile(g)
    b = P.run(g, s, opts)
    P.engine.clear_device_cache()
    b2 = P.run(g, s, opts)  # host layout first this time
    a2 = P.run(g, Strategy.parall().compile(g), opts)
    assert a.marginals.tobytes() == a2.marginals.tobytes() and a.iterations == a2.iterations
    assert b.marginals.tobytes() == b2.marginals.tobytes() and b.iterations == b2.iterations


def _create(V, rowptr, evar, kind):
    rowptr = np.asarray(rowptr, dtype=np.int64)
    evar = np.asarray(evar, dtype=np.int32)
    kind = np.asarray(kind, dtype=np.int8)
    F = len(rowptr) - 1
    p = np.full(max(F, 1), 0.5)
    desc = _native.GraphDesc(V, F, int(len(evar)), _native.ptr(rowptr, C.c_int64),
                             _native.ptr(evar, C.c_int32), _native.ptr(kind, C.c_int8),
                             _native.ptr(p, C.c_double), _native.ptr(p, C.c_double))
    h = C.c_void_p()
    st = _native.lib().hbp_graph_create(C.byref(desc), 0, C.byref(h))
    if st == _native.HBP_OK:
        _native.lib().hbp_graph_destroy(h)
        return None
    return st, _native.last_error()


@pytest.mark.parametrize("case,want", [
    ((3, [0, 2, 2], [0, 1], [0, 0]), "factor 1: degree must be in [1, 65535]"),
    ((3, [0, 2, 3], [0, 1, 2], [0, 7]), "factor 1: bad kind"),
    ((3, [0, 2, 3], [0, 1, 5], [0, 0]), "edge variable out of range"),
    ((4, [0, 2, 3], [0, 1, 2], [0, 1]), "variable 3 appears in no factor"),
    ((3, [0, 2, 4], [0, 1, 2], [0, 1]), "factor_rowptr does not span the edge array"),
])
def test_device_layout_rejects_like_the_host_builder(case, want):
    """hbp_graph_create validates on the device; the errors are the host
    builder's (layout.cpp), in its order."""
    err = _create(*case)
    assert err is not None and err[0] == _native.HBP_EINVAL
    assert want in err[1], err[1]
