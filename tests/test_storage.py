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


@pytest.mark.needs_ref
def test_op_counter_matches_reference(hornbp_ref):
    """OpCounter counts what the reference's passes count (engine.py:181-182,
    224-225, 246-247, 258-259, 277-278, 292-293, 311-312), per batch, on
    random graphs: the counting is host-side, so this runs on CPU."""
    R = hornbp_ref
    from hornbp.storage import initialize as rinit
    from paper_2509_22337_b200 import OpCounter
    from paper_2509_22337_b200.engine import _count_ftov, _count_vtof

    rng = np.random.default_rng(11)
    for _ in range(25):
        g = random_graph(rng, max_vars=12, max_factors=12, max_body=6)
        rg = R.FactorGraph(g.num_variables, [R.Factor(R.FactorKind(f.kind.value), f.head, f.body, f.p1, f.p2)
                                             for f in g.factors])
        sched = R.Strategy.parall().compile(rg)
        s_batch, t_batch = sched.s_batches[0], sched.t_batches[0]
        rs = rinit(rg)
        want_v, want_f = R.OpCounter(), R.OpCounter()
        R.update_vtof_batch(rs, t_batch, counter=want_v)
        R.update_ftov_batch(rs, s_batch, counter=want_f)
        st = initialize(g)
        got_v, got_f = OpCounter(), OpCounter()
        _count_vtof(st, st.vtof_indices(list(t_batch)), got_v)
        _count_ftov(st, st.vtof_indices(list(s_batch)), got_f)
        assert (got_v.count, got_f.count) == (want_v.count, want_f.count)
