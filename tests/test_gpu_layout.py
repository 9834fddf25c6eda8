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
