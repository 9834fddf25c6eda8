"""Host MessageStore mirror: reference layout goldens and invariants."""

import numpy as np
import pytest

from builders import example_graph, random_graph
from paper_2509_22337_b200 import EdgeId, Factor, FactorGraph, FactorKind
from paper_2509_22337_b200.storage import StorageError, edge_indices, initialize


def test_row_pointers_and_uniform():
    s = initialize(example_graph())
    assert s.rowptr_vtof.tolist() == [0, 1, 2, 5]
    assert s.rowptr_ftov.tolist() == [0, 2, 4, 5]
    for b in (s.vtof0, s.vtof1, s.ftov0, s.ftov1):
        assert (b == 1.0).all() and len(b) == 5
    with pytest.raises(StorageError):
        initialize(FactorGraph(0, []))


def test_bijection_roundtrip_and_duality():
    g = example_graph()
    s = initialize(g)
    assert edge_indices(s, EdgeId(0, 0)) == (0, 0)
    for e in g.edges():
        vt, ft = edge_indices(s, e)
        assert s.edge_at_vtof(vt) == e and s.edge_at_ftov(ft) == e
        assert s.av_excl[vt] == ft and s.af_excl[ft] == vt
    assert (s.af_head == (s.af_excl == s.af_v0)).all()


@pytest.mark.needs_ref
def test_layout_identical_to_reference(hornbp_ref):
    rng = np.random.default_rng(2)
    R = hornbp_ref
    from hornbp.storage import initialize as rinit
    for _ in range(20):
        g = random_graph(rng, max_vars=10, max_factors=10)
        rg = R.FactorGraph(g.num_variables, [R.Factor(R.FactorKind(f.kind.value), f.head, f.body, f.p1, f.p2)
                                             for f in g.factors])
        a, b = initialize(g), rinit(rg)
        for name in ("rowptr_vtof", "vtof_var", "vtof_factor", "rowptr_ftov", "ftov_to_vtof",
                     "vtof_to_ftov", "ftov_var", "av_start", "av_end", "av_excl", "af_start",
                     "af_end", "af_excl", "af_v0", "af_p1", "af_p2", "af_kind", "af_head"):
            assert np.array_equal(getattr(a, name), getattr(b, name)), name
