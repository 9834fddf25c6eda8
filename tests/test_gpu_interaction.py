"""GPU parity of the device-resident interaction loop (F1): the trace equals
the reference loop's (ranking.py:94-135) -- clamp + compile + run each round --
replayed on the C oracle with real clamped graphs: same alarms, labels and
p_true bits, for PARALL and canonical SEQFIX."""

import numpy as np
import pytest

from oracle import orc
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import EngineOptions, Strategy, clamp_evidence, rank_alarms
from paper_2509_22337_b200 import workloads as W

pytestmark = pytest.mark.gpu


def replay(g, alarms, strategy, opts, trace):
    cur, labeled = g, []
    for rnd in trace.rounds:
        s = strategy.compile(cur)
        o = orc.run(cur, s.arrays(cur), opts.max_iterations, opts.tolerance, threads=8)
        top = rank_alarms(o["marginals"], alarms, labeled)[0]
        assert top == rnd.alarm
        assert o["marginals"][top, 1] == rnd.p_true
        lab = alarms.label_of(top)
        assert lab == rnd.label
        cur = clamp_evidence(cur, top, lab)
        labeled.append(top)


@pytest.mark.parametrize("strategy", [Strategy.parall(), Strategy.seqfix()], ids=["PARALL", "SEQFIX"])
def test_loop_weblech_full_trace(strategy):
    g, alarms = W.graph("weblech")
    opts = EngineOptions(1000, 1e-9)
    trace = P.interaction_loop(g, alarms, strategy, opts)
    assert sum(trace.label_sequence) == alarms.num_true
    replay(g, alarms, strategy, opts, trace)


@pytest.mark.parametrize("name,strategy,rounds", [
    ("hedc", Strategy.parall(), 25), ("hedc", Strategy.seqfix(), 10), ("ftp", Strategy.parall(), 6)])
def test_loop_prefix_matches_reference_semantics(name, strategy, rounds):
    g, alarms = W.graph(name)
    opts = EngineOptions(1000, 1e-9)
    trace = P.interaction_loop(g, alarms, strategy, opts, max_rounds=rounds)
    assert len(trace.rounds) == rounds
    replay(g, alarms, strategy, opts, trace)


def test_loop_matches_host_path():
    """Device path == the generic host path (clamp + compile + run per round),
    which CUSTOM strategies take; an empty CUSTOM relation compiles to PARALL's
    single batch."""
    g, alarms = W.graph("weblech")
    opts = EngineOptions(1000, 1e-9)
    a = P.interaction_loop(g, alarms, Strategy.parall(), opts)
    b = P.interaction_loop(g, alarms, Strategy.custom([]), opts)
    assert [(r.alarm, r.label, r.p_true) for r in a.rounds] == \
           [(r.alarm, r.label, r.p_true) for r in b.rounds]


def test_evidence_run_equals_clamped_graph_run():
    g, alarms = W.graph("hedc")
    ids, labels = W.evidence_set(alarms, 5)
    cur = W.clamped_graph(g, ids, labels)
    opts = EngineOptions(1000, 1e-9)
    for strat in (Strategy.parall(), Strategy.seqfix()):
        want = P.run(cur, strat.compile(cur), opts)
        dg = P.engine.device_graph(g)
        plan = dg.plan(strat.compile(g), g)
        dg.set_evidence(ids, labels.astype(np.int8))
        try:
            got = plan.run(opts, g)
        finally:
            dg.set_evidence([], [])
        assert got.iterations == want.iterations
        assert got.marginals.tobytes() == want.marginals.tobytes()
        assert got.deltas == want.deltas


def test_explicit_seqfix_order_fails_like_the_reference():
    """An explicit SEQFIX order is no longer a permutation of the clamped
    graph's edges, so the reference's second round raises (schedule.py:184-185)."""
    g, alarms = W.graph("weblech")
    with pytest.raises(P.ScheduleError):
        P.interaction_loop(g, alarms, Strategy.seqfix(g.edge_list()), EngineOptions(1000, 1e-9))
