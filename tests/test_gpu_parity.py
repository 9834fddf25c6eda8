"""GPU parity: the CUDA engine against the reference (golden fixtures) and the
C oracle, bit for bit. Run on the B200 box: pytest -m gpu."""

import itertools
import os

import numpy as np
import pytest

from builders import example_graph, random_graph, random_poset, random_tree
from conftest import ROOT, sha
from oracle import orc
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import (EdgeId, EngineOptions, Factor, FactorGraph, FactorKind, OpCounter,
                                   Strategy, UnderflowError, clamp_evidence, closed_form_message,
                                   compute_marginals, initialize, rank_alarms, update_and_body,
                                   update_and_head, update_ftov_batch, update_vtof_batch)
from paper_2509_22337_b200 import workloads as W

pytestmark = pytest.mark.gpu

P3 = 0.997002999


def device_vs_oracle(g, sched, opts):
    res = P.run(g, sched, opts)
    o = orc.run(g, sched.arrays(g), opts.max_iterations, opts.tolerance, opts.normalize_messages, threads=4)
    return res, o


# ---- BASELINE configurations vs the reference's golden outputs -----------------------------

@pytest.mark.parametrize("key", ["C1", "C1-tol", "C2", "C2-canonical", "C3", "C4-PARALL", "C4-SEQFIX"])
def test_baseline_bitwise(key, golden):
    w = W.build(key.replace("-tol", ""))
    want = golden["runs"][key]
    max_it, tol = want["max_iterations"], want["tolerance"]
    sched = w.strategy.compile(w.graph)
    res = P.run(w.graph, sched, EngineOptions(max_iterations=max_it, tolerance=tol))
    assert res.iterations == want["iterations"]
    assert res.converged == want["converged"]
    assert [float(d).hex() for d in res.deltas] == want["deltas"]
    assert sha(res.marginals) == want["marginals_sha"]
    o = orc.run(w.graph, sched.arrays(w.graph), max_it, tol, threads=8)
    assert res.marginals.tobytes() == o["marginals"].tobytes()


def test_c1_full_marginal_arrays():
    w = W.build("C1")
    res = P.run(w.graph, w.strategy.compile(w.graph), EngineOptions(100, 0.0))
    ref = np.load(os.path.join(ROOT, "tests", "golden", "weblech_c1.npz"))
    assert res.marginals.tobytes() == ref["marginals"].tobytes()
    assert np.asarray(res.deltas).tobytes() == ref["deltas"].tobytes()


def test_c3_residual_order_matches_reference(golden):
    g, _ = W.graph("avrora")
    assert sha(W.residual_order(g).astype(np.int64)) == golden["runs"]["C3"]["order_sha"]


def test_c4_topk_ranking_identical(golden):
    w = W.build("C4-PARALL")
    res = P.run(w.graph, w.strategy.compile(w.graph), EngineOptions(1000, 1e-9))
    ranked = rank_alarms(res.marginals, w.alarms)
    assert ranked[:10] == golden["runs"]["C4-PARALL"]["top10"]
    assert sha(np.asarray(ranked[:100], dtype=np.int64)) == golden["runs"]["C4-PARALL"]["top100_sha"]


@pytest.mark.parametrize("j", [0, 1, 2, 3])
def test_c5_evidence_sets(j, golden):
    g, alarms = W.graph("ftp")
    ids, labels = W.evidence_set(alarms, j)
    cur = W.clamped_graph(g, ids, labels)
    res = P.run(cur, Strategy.parall().compile(cur), EngineOptions(1000, 1e-9))
    want = golden["sweep"][str(j)]
    assert res.iterations == want["iterations"]
    assert sha(res.marginals) == want["marginals_sha"]
    ranked = rank_alarms(res.marginals, alarms, ids.tolist())
    assert ranked[:10] == want["top10"]
    assert sha(np.asarray(ranked[:100], dtype=np.int64)) == want["top100_sha"]


# ---- random graphs vs the oracle ----------------------------------------------------------

def test_random_graphs_bitwise_vs_oracle():
    rng = np.random.default_rng(2024)
    for trial in range(120):
        g = random_graph(rng, max_vars=14, max_factors=14, max_body=4, or_prob=0.5)
        kind = trial % 4
        if kind == 0:
            sched = Strategy.parall().compile(g)
        elif kind == 1:
            sched = P.compile_schedule(g, random_poset(rng, g))
        elif kind == 2:
            perm = rng.permutation(g.num_edges)
            sched = Strategy.seqfix(g.edges_at(perm)).compile(g)
        else:
            sched = Strategy.seqfix().compile(g)
        opts = EngineOptions(max_iterations=int(rng.integers(1, 40)),
                             tolerance=float(rng.choice([0.0, 1e-9, 1e-5])),
                             normalize_messages=bool(trial % 5 != 2))
        o = orc.run(g, sched.arrays(g), opts.max_iterations, opts.tolerance, opts.normalize_messages)
        if o["underflow"] is not None:
            with pytest.raises(UnderflowError) as ei:
                P.run(g, sched, opts)
            assert (ei.value.kind, ei.value.iteration, ei.value.index) == o["underflow"], trial
            continue
        res = P.run(g, sched, opts)
        assert res.iterations == o["iterations"], trial
        assert res.converged == o["converged"]
        assert res.marginals.tobytes() == o["marginals"].tobytes(), trial
        assert np.asarray(res.deltas).tobytes() == o["deltas"].tobytes()


def test_trees_all_strategies_bitwise_and_exact():
    rng = np.random.default_rng(6)
    for _ in range(15):
        g = random_tree(rng, max_vars=10)
        exact = enumerate_marginals(g)
        for strat in (Strategy.parall(), Strategy.topo(), Strategy.seqfix()):
            sched = strat.compile(g)
            res, o = device_vs_oracle(g, sched, EngineOptions(max_iterations=200))
            assert res.marginals.tobytes() == o["marginals"].tobytes()
            assert res.converged
            assert np.allclose(res.marginals, exact, atol=1e-8)


def test_bitwise_independent_of_grid_size():
    """HBP_GRID forces the CTA count: the work moves between CTAs, the bits
    do not (PARALL whole-node phases and fused levels alike)."""
    for key in ("C2", "C4-PARALL"):
        w = W.build(key)
        sched = w.strategy.compile(w.graph)
        a = P.run(w.graph, sched, EngineOptions(1000, 1e-9))
        os.environ["HBP_GRID"] = "37"
        try:
            P.engine.clear_device_cache()
            b = P.run(w.graph, sched, EngineOptions(1000, 1e-9))
        finally:
            os.environ.pop("HBP_GRID")
            P.engine.clear_device_cache()
        assert a.iterations == b.iterations
        assert a.marginals.tobytes() == b.marginals.tobytes()


# ---- run-loop contracts (engine.py:531-594) -----------------------------------------------

def test_example_graph_converges_to_p_cubed():
    g = example_graph()
    order = [EdgeId(0, 0), EdgeId(1, 0), EdgeId(2, 1), EdgeId(2, 2), EdgeId(2, 0)]
    for strat in (Strategy.parall(), Strategy.seqfix(order), Strategy.topo()):
        res = P.run(g, strat.compile(g))
        assert res.converged
        assert res.marginals[2, 1] == pytest.approx(P3, abs=1e-9)


def test_first_iteration_fixed_order_vs_flooding():
    g = example_graph()
    order = [EdgeId(0, 0), EdgeId(1, 0), EdgeId(2, 1), EdgeId(2, 2), EdgeId(2, 0)]
    one = EngineOptions(max_iterations=1, tolerance=0.0)
    assert P.run(g, Strategy.seqfix(order).compile(g), one).marginals[2, 1] == pytest.approx(P3, abs=1e-12)
    assert P.run(g, Strategy.parall().compile(g), one).marginals[2, 1] == pytest.approx(0.24975, abs=1e-12)


def test_contracts():
    g = example_graph()
    s = Strategy.parall().compile(g)
    with pytest.raises(ValueError):
        P.run(g, s, EngineOptions(max_iterations=0))
    r = P.run(g, s, EngineOptions(max_iterations=1))
    assert not r.converged and r.iterations == 1 and len(r.deltas) == 1
    r = P.run(g, s, EngineOptions(max_iterations=3, tolerance=0.0, record_history=True))
    assert len(r.history) == 3 and r.history[-1][2, 1] == r.marginals[2, 1]
    r = P.run(g, s, EngineOptions(max_iterations=100000, tolerance=0.0, time_limit=1e-9))
    assert not r.converged and r.iterations < 100000
    with pytest.raises(UnderflowError, match="marginal of variable 0"):
        bad = clamp_evidence(clamp_evidence(g, 0, True), 0, False)
        P.run(bad, Strategy.parall().compile(bad))


def test_history_matches_oracle_prefixes():
    rng = np.random.default_rng(8)
    g = random_graph(rng, max_vars=9, max_factors=9)
    s = Strategy.parall().compile(g)
    r = P.run(g, s, EngineOptions(max_iterations=6, tolerance=0.0, record_history=True))
    for i, h in enumerate(r.history, start=1):
        o = orc.run(g, s.arrays(g), i, 0.0)
        assert h.tobytes() == o["marginals"].tobytes()


def test_history_sized_by_iterations_run():
    """record_history keeps only the iterations that run (engine.py:574-575):
    a huge max_iterations at ftp scale must not allocate max_iterations x V;
    a run longer than the device's history budget re-runs with an exact
    buffer, and every recorded row is that iteration's marginals."""
    w = W.build("C4-PARALL")
    s = w.strategy.compile(w.graph)
    r = P.run(w.graph, s, EngineOptions(max_iterations=10_000_000, tolerance=1e-9,
                                        record_history=True))
    assert r.converged and len(r.history) == r.iterations == 23
    assert r.history[-1].tobytes() == r.marginals.tobytes()
    r2 = P.run(w.graph, s, EngineOptions(max_iterations=90, tolerance=0.0, record_history=True))
    assert len(r2.history) == 90  # beyond the 256 MiB budget (79 ftp iterations): re-run
    r3 = P.run(w.graph, s, EngineOptions(max_iterations=40, tolerance=0.0))
    assert r2.history[39].tobytes() == r3.marginals.tobytes()
    assert r2.history[22].tobytes() == r.marginals.tobytes()


def test_normalization_toggle_close():
    rng = np.random.default_rng(8)
    for _ in range(10):
        g = random_graph(rng, max_vars=5, max_factors=4)
        s = Strategy.parall().compile(g)
        a = P.run(g, s, EngineOptions(max_iterations=8, tolerance=0.0))
        b = P.run(g, s, EngineOptions(max_iterations=8, tolerance=0.0, normalize_messages=False))
        assert np.allclose(a.marginals, b.marginals, atol=1e-9)


def test_marginal_rows_sum_to_exactly_one():
    w = W.build("C4-PARALL")
    r = P.run(w.graph, w.strategy.compile(w.graph))
    assert np.all(r.marginals.sum(axis=1) == 1.0)


# ---- single-pass API on a host store --------------------------------------------------------

def naive_message(kind, p1, p2, incoming, target):
    """Brute-force sum over the factor table (independent of the closed forms)."""
    d = len(incoming)
    out = [0.0, 0.0]
    for bits in itertools.product((0, 1), repeat=d):
        body = bits[1:]
        cond = (all(body) if kind is FactorKind.AND else any(body)) if body else kind is FactorKind.AND
        ph = p1 if cond else p2
        val = ph if bits[0] else 1.0 - ph
        for s in range(d):
            if s != target:
                val *= incoming[s][bits[s]]
        out[bits[target]] += val
    return out


def enumerate_marginals(g):
    n = g.num_variables
    sums = np.zeros(n)
    tot = 0.0
    for a in range(1 << n):
        w = 1.0
        for f in g.factors:
            body = [(a >> v) & 1 for v in f.body]
            cond = (all(body) if f.kind is FactorKind.AND else any(body)) if body else f.kind is FactorKind.AND
            ph = f.p1 if cond else f.p2
            w *= ph if (a >> f.head) & 1 else 1.0 - ph
        tot += w
        for v in range(n):
            if (a >> v) & 1:
                sums[v] += w
    out = np.empty((n, 2))
    out[:, 1] = sums / tot
    out[:, 0] = 1.0 - out[:, 1]
    return out


def test_closed_form_frozen_values():
    assert closed_form_message(FactorKind.AND, 0.999, 0.0, [None, (0.5, 0.5), (0.5, 0.5)], 0) == \
        pytest.approx((0.75025, 0.24975), abs=1e-15)
    assert closed_form_message(FactorKind.OR, 1.0, 0.0, [(0.0, 1.0), None, (0.3, 0.7)], 1) == \
        pytest.approx((0.7, 1.0), abs=1e-15)
    assert closed_form_message(FactorKind.OR, 1.0, 0.0, [None, (0.5, 0.5), (0.5, 0.5)], 0) == \
        pytest.approx((0.25, 0.75), abs=1e-15)
    assert closed_form_message(FactorKind.AND, 0.999, 0.999, [None], 0) == pytest.approx((0.001, 0.999))
    assert closed_form_message(FactorKind.AND, 1.0, 1.0, [None], 0) == pytest.approx((0.0, 1.0))
    assert closed_form_message(FactorKind.AND, 0.999, 0.0, [(1.0, 1.0), None, (0.5, 0.5)], 1) == \
        pytest.approx((1.0, 1.0))


@pytest.mark.parametrize("kind", [FactorKind.AND, FactorKind.OR])
@pytest.mark.parametrize("head", [True, False])
def test_closed_form_vs_naive_table(kind, head):
    rng = np.random.default_rng(77 + 2 * (kind is FactorKind.OR) + head)
    for _ in range(60):
        arity = int(rng.integers(0 if head else 1, 9))
        if kind is FactorKind.OR and arity == 0:
            arity = 1
        p1 = float(rng.uniform(0, 1))
        p2 = p1 if arity == 0 else float(rng.uniform(0, 1))
        tgt = 0 if head else int(rng.integers(1, arity + 1))
        inc = [(float(rng.uniform(.05, 1)), float(rng.uniform(.05, 1))) for _ in range(arity + 1)]
        got = closed_form_message(kind, p1, p2, inc, tgt)
        want = naive_message(kind, p1, p2, inc, tgt)
        gs, ws = sum(got), sum(want)
        assert got[1] / gs == pytest.approx(want[1] / ws, rel=1e-12, abs=1e-13)


def test_multiply_count_linear():
    for arity in (1, 2, 8, 64, 256):
        inc = [(0.4, 0.6)] * (arity + 1)
        c = OpCounter()
        closed_form_message(FactorKind.AND, 0.9, 0.05, inc, 1, c)
        assert c.count <= 4 * arity + 8
        c = OpCounter()
        closed_form_message(FactorKind.OR, 0.9, 0.05, inc, 0, c)
        assert c.count <= 4 * arity + 8


def test_vtof_pass_products():
    g = FactorGraph(1, [Factor(FactorKind.AND, 0, (), .5, .5)] * 3)
    s = initialize(g)
    s.ftov0[:] = [0.2, 0.5, 9.0]
    s.ftov1[:] = [0.8, 0.5, 9.0]
    update_vtof_batch(s, [EdgeId(2, 0)], normalize=False)
    assert s.vtof0[2] == pytest.approx(0.1) and s.vtof1[2] == pytest.approx(0.4)
    g1 = FactorGraph(1, [Factor(FactorKind.AND, 0, (), 0.9, 0.9)])
    s1 = initialize(g1)
    s1.ftov0[0], s1.ftov1[0] = 0.3, 0.7
    update_vtof_batch(s1, [EdgeId(0, 0)], normalize=False)
    assert (s1.vtof0[0], s1.vtof1[0]) == (1.0, 1.0)


def test_ftov_batch_mixed_vs_naive():
    rng = np.random.default_rng(12)
    g = random_graph(rng, max_vars=8, max_factors=8, or_prob=0.5)
    s = initialize(g)
    s.vtof0[:] = rng.uniform(0.05, 1.0, size=g.num_edges)
    s.vtof1[:] = rng.uniform(0.05, 1.0, size=g.num_edges)
    v0, v1 = s.vtof0.copy(), s.vtof1.copy()
    update_ftov_batch(s, g.edge_list(), normalize=False)
    for e in g.edges():
        f = g.factors[e.factor]
        inc = [(v0[g.edge_index(EdgeId(e.factor, k))], v1[g.edge_index(EdgeId(e.factor, k))])
               for k in range(f.degree)]
        want = naive_message(f.kind, f.p1, f.p2, inc, e.slot)
        got = (s.ftov0[s.ftov_index(e)], s.ftov1[s.ftov_index(e)])
        assert got[1] / sum(got) == pytest.approx(want[1] / sum(want), rel=1e-12)


def test_routing_validation_and_marginals():
    g = example_graph()
    s = initialize(g)
    with pytest.raises(ValueError, match="head"):
        update_and_head(s, [EdgeId(2, 1)])
    with pytest.raises(ValueError, match="body"):
        update_and_body(s, [EdgeId(0, 0)])
    update_and_head(s, [EdgeId(0, 0)])
    assert np.all(compute_marginals(initialize(g)) == 0.5)
    rng = np.random.default_rng(4)
    g = random_graph(rng)
    s = initialize(g)
    s.ftov0[:] = rng.uniform(0.01, 1.0, size=g.num_edges)
    s.ftov1[:] = rng.uniform(0.01, 1.0, size=g.num_edges)
    m = compute_marginals(s)
    assert np.all(m.sum(axis=1) == 1.0)


def test_interaction_loop_matches_oracle_replay():
    rng = np.random.default_rng(33)
    g, alarms = W.graph("weblech")
    trace = P.interaction_loop(g, alarms, Strategy.parall(), EngineOptions(1000, 1e-9))
    # replay with the oracle
    cur, labeled = g, []
    for rnd in trace.rounds:
        s = Strategy.parall().compile(cur)
        o = orc.run(cur, s.arrays(cur), 1000, 1e-9)
        top = rank_alarms(o["marginals"], alarms, labeled)[0]
        assert top == rnd.alarm and o["marginals"][top, 1] == rnd.p_true
        lab = alarms.label_of(top)
        cur = clamp_evidence(cur, top, lab)
        labeled.append(top)
    assert sum(trace.label_sequence) == alarms.num_true


def test_shared_reciprocal_division_is_ddiv_rn():
    """div2_rn (one reciprocal refinement for both normalisations) vs __ddiv_rn."""
    import ctypes as C
    from paper_2509_22337_b200 import _native

    rng = np.random.default_rng(99)
    n = 1 << 20
    a = np.concatenate([rng.uniform(0, 1, n // 4), rng.uniform(0, 1, n // 4) * 2.0 ** rng.integers(-1074, 1023, n // 4),
                        np.abs(rng.standard_normal(n // 4)) * 1e-300, rng.uniform(0.5, 2.0, n // 4)])
    b = np.concatenate([rng.uniform(0, 1, n // 4) + a[: n // 4], 2.0 ** rng.integers(-1074, 1024, n // 4) * rng.uniform(1, 2, n // 4),
                        np.abs(rng.standard_normal(n // 4)) * 1e-290, rng.uniform(1e-308, 1e-300, n // 4)])
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 1.0, 3.0])
    a = np.concatenate([a, np.repeat(special, len(special))])
    b = np.concatenate([b, np.tile(special, len(special))])
    fast = np.empty(2 * len(a))
    ref = np.empty(2 * len(a))
    st = _native.lib().hbp_selftest_division(len(a), _native.ptr(a, C.c_double), _native.ptr(b, C.c_double),
                                             _native.ptr(fast, C.c_double), _native.ptr(ref, C.c_double))
    assert st == 0, _native.last_error()
    assert fast.tobytes() == ref.tobytes()


def test_long_rows_bitwise_vs_oracle():
    """Variable rows of 40+ slots and a 41-slot clause: the slot-per-thread
    heavy paths of the single-graph executor, all strategies."""
    from builders import hub_graph
    rng = np.random.default_rng(123)
    for trial in range(4):
        g = hub_graph(rng)
        for strat in (Strategy.parall(), Strategy.seqfix()):
            sched = strat.compile(g)
            opts = EngineOptions(max_iterations=60, tolerance=1e-12)
            res, o = device_vs_oracle(g, sched, opts)
            assert res.iterations == o["iterations"]
            assert res.marginals.tobytes() == o["marginals"].tobytes(), (trial, strat.kind)
            assert np.asarray(res.deltas).tobytes() == o["deltas"].tobytes()


@pytest.mark.parametrize("grouping", ["1", "0"])
def test_grouping_modes_bitwise_identical(grouping, monkeypatch):
    """HBP_GROUPING (the grouping A/B of profiles/r1_grouping_ab.md) only moves
    work between threads: slot items in degree order (1) or in EdgeId order
    (0) give the default node-grouped plan's bits."""
    rng = np.random.default_rng(99)
    graphs = [W.graph("hedc")[0]] + [random_graph(rng, max_vars=20, max_factors=20, max_body=5)
                                     for _ in range(6)]
    for g in graphs:
        for strat in (Strategy.parall(), Strategy.seqfix()):
            opts = EngineOptions(60, 1e-9)
            monkeypatch.delenv("HBP_GROUPING", raising=False)
            P.engine.clear_device_cache()
            ref = P.run(g, strat.compile(g), opts)
            monkeypatch.setenv("HBP_GROUPING", grouping)
            P.engine.clear_device_cache()
            got = P.run(g, strat.compile(g), opts)
            assert got.iterations == ref.iterations
            assert got.marginals.tobytes() == ref.marginals.tobytes()
            assert np.asarray(got.deltas).tobytes() == np.asarray(ref.deltas).tobytes()
    P.engine.clear_device_cache()


def test_more_phases_than_the_shared_memory_phase_cache():
    """avrora under a random-permutation SEQFIX compiles to 660 levels = 1,320
    phases, past the kernel's 1,024-entry shared-memory phase cache (the rest
    are read from global memory): still bitwise equal to the oracle."""
    g, _ = W.graph("avrora")
    rng = np.random.default_rng(5)
    order = [g.edge_at(int(i)) for i in rng.permutation(g.num_edges)]
    sched = Strategy.seqfix(order).compile(g)
    assert 2 * sched.num_batches > 1024
    res, o = device_vs_oracle(g, sched, EngineOptions(max_iterations=50, tolerance=1e-6))
    assert res.iterations == o["iterations"] and res.converged == o["converged"]
    assert res.marginals.tobytes() == o["marginals"].tobytes()
    assert np.asarray(res.deltas).tobytes() == o["deltas"].tobytes()


def _compile_any(rng, g, mode):
    if mode == 0:
        return Strategy.parall().compile(g)
    if mode == 1:
        return Strategy.seqfix().compile(g)
    if mode == 2:
        return Strategy.seqfix(g.edges_at(rng.permutation(g.num_edges))).compile(g)
    return P.compile_schedule(g, random_poset(rng, g))


def test_underflow_attribution_bitwise_vs_oracle():
    """UnderflowError names the reference's message or variable: the first
    failing pass of the first failing iteration, rows[argmin(total)] in the
    reference's stable descending-row-length order (engine.py:155-165,
    :512-518) -- (kind, iteration, index) equal to the oracle's, which
    tests/test_oracle.py pins to hornbp itself."""
    from builders import contradictory_graph

    rng = np.random.default_rng(505)
    raised, kinds = 0, set()
    for trial in range(360):
        g = contradictory_graph(rng)
        sched = _compile_any(rng, g, trial % 4)
        opts = EngineOptions(max_iterations=int(rng.integers(1, 25)), tolerance=1e-9,
                             normalize_messages=trial % 7 != 3)
        o = orc.run(g, sched.arrays(g), opts.max_iterations, opts.tolerance, opts.normalize_messages)
        if o["underflow"] is None:
            res = P.run(g, sched, opts)
            assert res.iterations == o["iterations"], trial
            assert res.marginals.tobytes() == o["marginals"].tobytes(), trial
            continue
        with pytest.raises(UnderflowError) as ei:
            P.run(g, sched, opts)
        got = (ei.value.kind, ei.value.iteration, ei.value.index)
        assert got == o["underflow"], (trial, got, o["underflow"])
        raised += 1
        kinds.add(got[0])
    assert raised >= 200 and kinds == {1, 2, 3}, (raised, kinds)


def test_underflow_attribution_with_evidence_codes():
    """interaction_loop's device evidence (hbp_graph_set_evidence) reports the
    clamped graph's positions: the clamp slots lengthen their variables'
    rows and shift later ftov rows (graph.py:189-200, storage.py:55-63)."""
    from builders import contradictory_graph

    rng = np.random.default_rng(606)
    raised = 0
    for trial in range(120):
        g = contradictory_graph(rng, n_clamps=0)
        pairs = [(int(rng.integers(0, g.num_variables)), bool(rng.integers(0, 2)))
                 for _ in range(int(rng.integers(1, 6)))]
        strategy = Strategy.parall() if trial % 2 == 0 else Strategy.seqfix()
        cur = g
        for v, o_ in pairs:
            cur = clamp_evidence(cur, v, o_)
        sched = strategy.compile(cur)
        o = orc.run(cur, sched.arrays(cur), 30, 1e-9)
        dg = P.engine.device_graph(g)
        plan = dg.plan(strategy.compile(g), g)
        dg.set_evidence([v for v, _ in pairs], [o_ for _, o_ in pairs])
        try:
            if o["underflow"] is None:
                res = plan.run(EngineOptions(30, 1e-9), g)
                assert res.marginals.tobytes() == o["marginals"].tobytes(), trial
                continue
            with pytest.raises(UnderflowError) as ei:
                plan.run(EngineOptions(30, 1e-9), g)
        finally:
            dg.set_evidence([], [])
        assert (ei.value.kind, ei.value.iteration, ei.value.index) == o["underflow"], trial
        raised += 1
    assert raised >= 40, raised


def _plan_info(g, sched):
    import ctypes as C
    lib = P._native.lib()
    f = lib.hbp_debug_plan_info
    f.restype = None
    f.argtypes = [C.c_void_p] + [C.POINTER(C.c_int32)] * 4
    plan = P.engine.device_graph(g).plan(sched, g)
    nph, grid, thr, nfused = (C.c_int32() for _ in range(4))
    f(plan.handle, C.byref(nph), C.byref(grid), C.byref(thr), C.byref(nfused))
    return nph.value, nfused.value


def test_level_fusion_plans():
    """Levels whose factor-side writes no other factor of the level reads
    run as one phase (layout.cpp emit_fused): every level >= 1 of ftp's
    canonical SEQFIX (475 of 476), about half of hedc's random order."""
    w = W.build("C4-SEQFIX")
    sched = w.strategy.compile(w.graph)
    nph, nfused = _plan_info(w.graph, sched)
    assert sched.num_batches == 476 and nfused == 475 and nph == 2 + 475, (nph, nfused)
    w = W.build("C2")
    nph, nfused = _plan_info(w.graph, w.strategy.compile(w.graph))
    assert 90 <= nfused < 224 and nph == 2 * 224 - nfused, (nph, nfused)


def test_level_fusion_bitwise_identical_to_two_phase(monkeypatch):
    """HBP_FUSE=0 runs every level as two phases: same bits, iterations and
    deltas as the fused plan, on every schedule family."""
    rng = np.random.default_rng(4242)
    graphs = [W.graph("hedc")[0]] + [random_graph(rng, max_vars=40, max_factors=40, max_body=6)
                                     for _ in range(12)]
    for i, g in enumerate(graphs):
        for mode in (1, 2, 3):
            sched = _compile_any(rng, g, mode)
            opts = EngineOptions(60, 1e-9)
            monkeypatch.delenv("HBP_FUSE", raising=False)
            P.engine.clear_device_cache()
            ref = P.run(g, sched, opts)
            monkeypatch.setenv("HBP_FUSE", "0")
            P.engine.clear_device_cache()
            got = P.run(g, sched, opts)
            assert got.iterations == ref.iterations, (i, mode)
            assert got.marginals.tobytes() == ref.marginals.tobytes(), (i, mode)
            assert np.asarray(got.deltas).tobytes() == np.asarray(ref.deltas).tobytes()
    P.engine.clear_device_cache()


def test_small_levels_on_a_cluster_bitwise(monkeypatch):
    """HBP_CSIZE=2/4 runs the small levels on a thread-block cluster of that
    many CTAs (cluster barrier between them) instead of CTA 0 alone: same bits,
    iterations and deltas (fused and unfused plans)."""
    rng = np.random.default_rng(99)
    graphs = [W.graph("hedc")[0]] + [random_graph(rng, max_vars=40, max_factors=40, max_body=6)
                                     for _ in range(6)]
    for i, g in enumerate(graphs):
        for mode in (1, 2, 3):
            sched = _compile_any(rng, g, mode)
            opts = EngineOptions(60, 1e-9)
            for fuse in (None, "0"):
                out = []
                for cs in (None, "2", "4"):
                    for k, v in (("HBP_CSIZE", cs), ("HBP_FUSE", fuse)):
                        if v is None:
                            monkeypatch.delenv(k, raising=False)
                        else:
                            monkeypatch.setenv(k, v)
                    P.engine.clear_device_cache()
                    out.append(P.run(g, sched, opts))
                for got in out[1:]:
                    assert got.iterations == out[0].iterations, (i, mode, fuse)
                    assert got.marginals.tobytes() == out[0].marginals.tobytes(), (i, mode, fuse)
                    assert np.asarray(got.deltas).tobytes() == np.asarray(out[0].deltas).tobytes()
    monkeypatch.delenv("HBP_CSIZE", raising=False)
    monkeypatch.delenv("HBP_FUSE", raising=False)
    P.engine.clear_device_cache()


def _pslot(g, sched):
    import ctypes as C
    f = P._native.lib().hbp_debug_plan_pslot
    f.restype = C.c_int32
    f.argtypes = [C.c_void_p]
    return f(P.engine.device_graph(g).plan(sched, g).handle)


def test_pslot_bitwise_identical_to_two_phase(monkeypatch):
    """PARALL runs as one phase per iteration (lbp_pslot: vtof messages
    recomputed per factor slot from the variable rows, double-buffered ftov);
    HBP_PSLOT=0 keeps the two-phase kernel. Same bits, iterations, deltas and
    history, with and without normalisation and device evidence codes."""
    rng = np.random.default_rng(777)
    used = 0
    graphs = [W.graph("weblech")[0], W.graph("hedc")[0]] + [
        random_graph(rng, max_vars=60, max_factors=60, max_body=7) for _ in range(16)]
    for i, g in enumerate(graphs):
        sched = Strategy.parall().compile(g)
        for norm in (True, False):
            opts = EngineOptions(int(rng.integers(1, 80)), 1e-9, normalize_messages=norm,
                                 record_history=True)
            ev = None
            if i % 3 == 1:
                vs = np.sort(rng.choice(g.num_variables, size=min(3, g.num_variables), replace=False))
                ev = (vs, rng.integers(0, 2, size=len(vs)).astype(bool))
            out = []
            for env in (None, "0"):
                if env is None:
                    monkeypatch.delenv("HBP_PSLOT", raising=False)
                else:
                    monkeypatch.setenv("HBP_PSLOT", env)
                P.engine.clear_device_cache()
                dg = P.engine.device_graph(g)
                # eligible: no node of degree > 32 (a factor = a lane group of a warp)
                small = (np.bincount(np.asarray(g.vars)).max() <= 32
                         and np.diff(np.asarray(g.rowptr)).max() <= 32)
                assert _pslot(g, sched) == (1 if env is None and small else 0), i
                used += env is None and small
                if ev is not None:
                    dg.set_evidence(*ev)
                try:
                    out.append(P.run(g, sched, opts))
                except UnderflowError as e:
                    out.append((e.kind, e.iteration, e.index))
            a, b = out
            if isinstance(a, tuple) or isinstance(b, tuple):
                assert a == b, (i, norm)
                continue
            assert a.iterations == b.iterations and a.converged == b.converged, (i, norm)
            assert a.marginals.tobytes() == b.marginals.tobytes(), (i, norm)
            assert np.asarray(a.deltas).tobytes() == np.asarray(b.deltas).tobytes(), (i, norm)
            assert len(a.history) == len(b.history)
            for x, y in zip(a.history, b.history):
                assert np.asarray(x).tobytes() == np.asarray(y).tobytes(), (i, norm)
    assert used >= 20, used
    monkeypatch.delenv("HBP_PSLOT", raising=False)
    P.engine.clear_device_cache()


def test_pslot_cluster_barrier_bitwise(monkeypatch):
    """lbp_pslot on at most 8 CTAs runs as one thread-block cluster whose
    iteration barrier is the hardware cluster barrier; HBP_PSLOT_CLUSTER=0
    keeps the global-memory counter barrier. Forced grids of 2..8 CTAs
    (HBP_GRID) and C1 weblech's own grid: same bits and iterations either
    way, and the same as the two-phase kernel."""
    rng = np.random.default_rng(4242)
    graphs = [W.graph("weblech")[0]] + [
        random_graph(rng, max_vars=60, max_factors=60, max_body=7) for _ in range(8)]
    for i, g in enumerate(graphs):
        sched = Strategy.parall().compile(g)
        for grid in ((None,) if i == 0 else (2, 5, 8)):
            opts = EngineOptions(int(rng.integers(1, 120)), 1e-9, record_history=(i % 2 == 0))
            out = []
            for env in ({}, {"HBP_PSLOT_CLUSTER": "0"}, {"HBP_PSLOT": "0"}):
                for k in ("HBP_PSLOT_CLUSTER", "HBP_PSLOT", "HBP_GRID"):
                    monkeypatch.delenv(k, raising=False)
                for k, v in env.items():
                    monkeypatch.setenv(k, v)
                if grid is not None:
                    monkeypatch.setenv("HBP_GRID", str(grid))
                P.engine.clear_device_cache()
                try:
                    out.append(P.run(g, sched, opts))
                except UnderflowError as e:
                    out.append((e.kind, e.iteration, e.index))
            for b in out[1:]:
                a = out[0]
                if isinstance(a, tuple) or isinstance(b, tuple):
                    assert a == b, (i, grid)
                    continue
                assert a.iterations == b.iterations and a.converged == b.converged, (i, grid)
                assert a.marginals.tobytes() == b.marginals.tobytes(), (i, grid)
                assert np.asarray(a.deltas).tobytes() == np.asarray(b.deltas).tobytes(), (i, grid)
                assert (a.history is None) == (b.history is None), (i, grid)
                for x, y in zip(a.history or [], b.history or []):
                    assert np.asarray(x).tobytes() == np.asarray(y).tobytes(), (i, grid)
    for k in ("HBP_PSLOT_CLUSTER", "HBP_PSLOT", "HBP_GRID"):
        monkeypatch.delenv(k, raising=False)
    P.engine.clear_device_cache()


def test_fp32_run_within_1e5_of_fp64():
    """run(..., EngineOptions(precision="fp32")): fp32
    message storage, fp64 arithmetic -- marginals within the north star's
    1e-5 of the fp64 run; PARALL only."""
    cases = [(W.build("C4-PARALL").graph, 1e-9), (W.build("C1").graph, 1e-9)]
    rng = np.random.default_rng(77)
    cases += [(random_graph(rng, max_vars=30, max_factors=30, max_body=5), 1e-9) for _ in range(10)]
    for g, tol in cases:
        sched = Strategy.parall().compile(g)
        a = P.run(g, sched, EngineOptions(500, tol))
        b = P.run(g, sched, EngineOptions(500, tol, precision="fp32"))
        assert np.abs(a.marginals - b.marginals).max() <= 1e-5
        # iteration counts may differ: fp32-stored messages can settle into
        # ~1e-8 oscillations that never meet a 1e-9 tolerance
        assert len(b.deltas) == b.iterations
    g = W.build("C2").graph
    with pytest.raises(ValueError):
        P.run(g, Strategy.seqfix().compile(g), EngineOptions(50, 1e-9, precision="fp32"))


def test_device_ranking_beyond_one_window():
    """The device top-k streams candidates through a 16,384-entry window
    (lbp_kernels.cuh topk_stream): a selection of every ftp variable
    (211,175) ranks exactly like the host (-P1, id) order, ties included, for
    the single graph and for sweep sets."""
    g = W.build("C4-PARALL").graph
    sched = Strategy.parall().compile(g)
    res = P.run(g, sched, EngineOptions(1000, 1e-9))
    sel = np.arange(g.num_variables, dtype=np.int32)
    order = np.lexsort((sel, -res.marginals[:, 1]))
    for k in (1, 100, 5000):
        got, p1 = P.engine.device_graph(g).rank(sel, k)
        assert got.tolist() == order[:k].tolist(), k
        assert p1.tobytes() == res.marginals[order[:k], 1].tobytes()
    _, alarms = W.graph("ftp")
    sets = [W.evidence_set(alarms, j) for j in range(2)]
    r = P.run_many(g, sets, None, EngineOptions(1000, 1e-9), marginals=True, deltas=False,
                   select=sel, topk=300)
    for j in range(2):
        lab = set(int(v) for v in sets[j][0])
        keep = np.array([v not in lab for v in sel])
        o = np.lexsort((sel, -r.marginals[j][:, 1]))
        want = [int(v) for v in o if keep[v]][:300]
        assert r.ranked[j].tolist() == want
