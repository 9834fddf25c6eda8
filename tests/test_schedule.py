"""Strategy compiler: batch identity with the reference, Theorem 2, goldens."""

import numpy as np
import pytest

from builders import example_graph, random_graph, random_poset, random_tree
from conftest import sched_sha
from paper_2509_22337_b200 import EdgeId, Factor, FactorGraph, FactorKind
from paper_2509_22337_b200 import workloads as W
from paper_2509_22337_b200.schedule import (Schedule, ScheduleError, Strategy, UpdatePoset,
                                            compile_schedule, delta, dependency_analysis,
                                            edge_neighbors, group_var_to_factor, parall_poset,
                                            seqfix_poset, topo_poset, verify_batches)

A1_V1, A2_V2, A3_V3, A3_V1, A3_V2 = EdgeId(0, 0), EdgeId(1, 0), EdgeId(2, 0), EdgeId(2, 1), EdgeId(2, 2)
ORDER = [A1_V1, A2_V2, A3_V1, A3_V2, A3_V3]


def test_edge_neighbors():
    g = example_graph()
    assert edge_neighbors(g, A3_V1) == {A2_V2}
    assert edge_neighbors(g, A1_V1) == set()
    assert edge_neighbors(g, A3_V3) == {A1_V1, A2_V2}


def test_posets():
    g = example_graph()
    p = parall_poset(g)
    assert p.pairs == () and not p.has_order
    s = seqfix_poset(g, ORDER)
    for i, a in enumerate(ORDER):
        for b in ORDER[i + 1:]:
            assert s.precedes(a, b) and not s.precedes(b, a)
    with pytest.raises(ScheduleError):
        seqfix_poset(g, [A1_V1, A2_V2])
    with pytest.raises(ScheduleError):
        seqfix_poset(g, ORDER[:-1] + [A1_V1])
    with pytest.raises(ScheduleError, match="cycle"):
        UpdatePoset(g, [(A1_V1, A2_V2), (A2_V2, A1_V1)])
    with pytest.raises(ScheduleError, match="precede itself"):
        UpdatePoset(g, [(A1_V1, A1_V1)])


def test_batch_goldens():
    g = example_graph()
    assert [sorted(b) for b in dependency_analysis(parall_poset(g))] == [g.edge_list()]
    assert [sorted(b) for b in dependency_analysis(seqfix_poset(g, ORDER))] == [
        sorted([A1_V1, A2_V2]), sorted([A3_V1, A3_V2, A3_V3])]
    two = FactorGraph(2, [Factor(FactorKind.AND, 0, (), .7, .7), Factor(FactorKind.AND, 1, (), .6, .6)])
    assert len(dependency_analysis(seqfix_poset(two))) == 1


def test_fully_chained_order_singletons():
    g = FactorGraph(5, [Factor(FactorKind.AND, 2, (0, 1), .9, 0.), Factor(FactorKind.AND, 3, (0, 1), .8, 0.),
                        Factor(FactorKind.AND, 4, (2, 3), .7, 0.)])
    order = [EdgeId(2, 1), EdgeId(0, 2), EdgeId(1, 1), EdgeId(0, 0), EdgeId(2, 2), EdgeId(1, 2),
             EdgeId(0, 1), EdgeId(1, 0), EdgeId(2, 0)]
    batches = dependency_analysis(seqfix_poset(g, order))
    assert len(batches) == 9 and all(len(b) == 1 for b in batches)


def test_group_var_to_factor():
    g = example_graph()
    assert group_var_to_factor(g, [[A3_V1]]) == [sorted([A3_V3, A3_V2])]
    assert group_var_to_factor(g, [[A1_V1, A2_V2]]) == [[]]
    assert group_var_to_factor(g, [[A3_V1, A3_V2, A3_V3]]) == [sorted([A3_V3, A3_V1, A3_V2])]


def test_delta_indicator():
    g = example_graph()
    s = seqfix_poset(g, ORDER)
    assert delta(s, A3_V3, A1_V1) == 1
    assert delta(s, A1_V1, A3_V3) == 0
    assert delta(parall_poset(g), A3_V3, A1_V1) == 0


def test_compiled_t_batches_match_group_var_to_factor():
    rng = np.random.default_rng(3)
    for _ in range(10):
        g = random_graph(rng, max_vars=8, max_factors=8)
        sched = compile_schedule(g, random_poset(rng, g))
        assert [list(t) for t in sched.t_batches] == group_var_to_factor(g, sched.s_batches)


def test_theorem2_and_partition_on_random_posets():
    rng = np.random.default_rng(5)
    for _ in range(25):
        g = random_graph(rng, max_vars=10, max_factors=10)
        poset = random_poset(rng, g)
        sched = compile_schedule(g, poset)
        flat = [e for b in sched.s_batches for e in b]
        assert sorted(flat) == g.edge_list()
        assert verify_batches(poset, sched.s_batches) == []


def test_topo_on_trees_and_cycle_error():
    rng = np.random.default_rng(9)
    for _ in range(10):
        g = random_tree(rng)
        sched = Strategy.topo().compile(g)
        assert verify_batches(topo_poset(g), sched.s_batches) == []
    loop = FactorGraph(2, [Factor(FactorKind.AND, 0, (1,), .9, 0.), Factor(FactorKind.AND, 1, (0,), .9, 0.)])
    with pytest.raises(ScheduleError, match="cycle"):
        Strategy.topo().compile(loop)


def test_strategy_text():
    s = Strategy.from_text("strategy SEQFIX\nedge 0:0\nedge 1:0\nedge 2:1\nedge 2:2\nedge 2:0\n")
    assert s.kind == "SEQFIX" and s.order == tuple(ORDER)
    c = Strategy.from_text("# c\nstrategy CUSTOM\nbefore 0:0 2:0\n")
    assert c.pairs == ((A1_V1, A3_V3),)
    assert Strategy.from_text("strategy PARALL\n") == Strategy.parall()
    for bad in ["", "strategy NOPE\n", "strategy PARALL\nedge 0:0\n", "strategy SEQFIX\nedge 0\n",
                "strategy CUSTOM\nbefore 0:0\n", "strategy SEQFIX\nwhat\n"]:
        with pytest.raises(ScheduleError):
            Strategy.from_text(bad)
    with pytest.raises(ScheduleError):
        Strategy.from_name("CUSTOM")
    assert Strategy.from_name("topo").kind == "TOPO"


def test_schedule_from_tuples_equals_compiled():
    g = example_graph()
    sched = Strategy.seqfix(ORDER).compile(g)
    again = Schedule(sched.s_batches, sched.t_batches)
    assert again == sched and again.num_batches == 2
    for a, b in zip(again.arrays(g), sched.arrays(g)):
        assert np.array_equal(a, b)
    assert sched.batch_sizes() == [2, 3]


@pytest.mark.parametrize("key", ["C1", "C2", "C2-canonical", "C4-PARALL", "C4-SEQFIX"])
def test_baseline_schedules_match_reference(key, golden):
    w = W.build(key.replace("C1-tol", "C1"))
    sched = w.strategy.compile(w.graph)
    want = golden["runs"][key]
    assert sched.num_batches == want["k"]
    assert sched.updates_per_iteration() == want["updates_per_iteration"]
    assert sched_sha(sched.arrays(w.graph)) == want["sched_sha"]


@pytest.mark.needs_ref
def test_random_posets_identical_to_reference(hornbp_ref):
    """Batch-for-batch equality with hornbp.compile_schedule (CUSTOM, TOPO, SEQFIX)."""
    rng = np.random.default_rng(123)
    R = hornbp_ref
    for trial in range(40):
        g = random_graph(rng, max_vars=12, max_factors=12, or_prob=0.5)
        rg = R.FactorGraph(g.num_variables, [R.Factor(R.FactorKind(f.kind.value), f.head, f.body, f.p1, f.p2)
                                             for f in g.factors])
        poset = random_poset(rng, g)
        rposet = R.UpdatePoset(rg, [(R.EdgeId(*a), R.EdgeId(*b)) for a, b in poset.pairs])
        mine = compile_schedule(g, poset)
        ref = R.compile_schedule(rg, rposet)
        assert mine.s_batches == ref.s_batches and mine.t_batches == ref.t_batches
        perm = [g.edge_list()[i] for i in rng.permutation(g.num_edges)]
        assert Strategy.seqfix(perm).compile(g).s_batches == R.Strategy.seqfix(perm).compile(rg).s_batches
        t = random_tree(rng, max_vars=9)
        rt = R.FactorGraph(t.num_variables, [R.Factor(R.FactorKind(f.kind.value), f.head, f.body, f.p1, f.p2)
                                             for f in t.factors])
        assert Strategy.topo().compile(t).s_batches == R.Strategy.topo().compile(rt).s_batches
