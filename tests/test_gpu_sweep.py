"""GPU parity of the multi-evidence sweep (csrc/sweep.cu) against the
reference semantics: set j == run(clamp_evidence(G, set j), PARALL), bit for
bit, checked through the C oracle and the reference's golden C5 sets."""

import numpy as np
import pytest

from builders import random_graph
from conftest import sha
from oracle import orc
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import (EngineOptions, Factor, FactorGraph, FactorKind, Strategy,
                                   clamp_evidence, rank_alarms)
from paper_2509_22337_b200 import workloads as W

pytestmark = pytest.mark.gpu


def clamp_all(g, pairs):
    for v, o in pairs:
        g = clamp_evidence(g, int(v), bool(o))
    return g


def oracle_set(g, pairs, opts):
    cur = clamp_all(g, pairs)
    sched = Strategy.parall().compile(cur)
    return orc.run(cur, sched.arrays(cur), opts.max_iterations, opts.tolerance,
                   opts.normalize_messages, threads=4), sched


def random_sets(rng, V, n, max_size=8, allow_dup=False):
    sets = []
    for _ in range(n):
        k = int(rng.integers(0, max_size + 1))
        vs = rng.choice(V, size=min(k, V), replace=allow_dup)
        sets.append([(int(v), bool(rng.integers(0, 2))) for v in vs])
    return sets


def check_against_oracle(g, sets, opts, res):
    for j, pairs in enumerate(sets):
        o, sched = oracle_set(g, pairs, opts)
        if o["underflow"] is not None:
            e = res.errors[j]
            assert e is not None, j
            assert (e.kind, e.iteration, e.index) == o["underflow"], (j, e, o["underflow"])
            continue
        assert res.errors[j] is None, (j, res.errors[j])
        assert res.iterations[j] == o["iterations"], j
        assert bool(res.converged[j]) == o["converged"], j
        assert res.marginals[j].tobytes() == o["marginals"].tobytes(), j
        assert np.asarray(res.deltas[j]).tobytes() == o["deltas"].tobytes(), j
        assert res.updates_per_iteration[j] == sched.updates_per_iteration()


@pytest.mark.parametrize("name", ["weblech", "hedc"])
def test_sweep_bitwise_vs_oracle_baseline_graphs(name):
    g, alarms = W.graph(name)
    rng = np.random.default_rng(11)
    sets = random_sets(rng, g.num_variables, 40)
    sets[0] = []  # no evidence == plain run
    opts = EngineOptions(1000, 1e-9)
    res = P.run_many(g, sets, Strategy.parall(), opts)
    check_against_oracle(g, sets, opts, res)
    plain = P.run(g, Strategy.parall().compile(g), opts)
    assert res.marginals[0].tobytes() == plain.marginals.tobytes()


def test_sweep_random_graphs_all_options():
    rng = np.random.default_rng(77)
    for trial in range(30):
        g = random_graph(rng, max_vars=14, max_factors=14, max_body=4, or_prob=0.5)
        sets = random_sets(rng, g.num_variables, int(rng.integers(1, 70)), max_size=4,
                           allow_dup=trial % 3 == 0)
        opts = EngineOptions(max_iterations=int(rng.integers(1, 40)),
                             tolerance=float(rng.choice([0.0, 1e-9, 1e-5])),
                             normalize_messages=bool(trial % 5 != 2))
        res = P.run_many(g, sets, None, opts)
        check_against_oracle(g, sets, opts, res)


def test_sweep_contradictory_evidence_is_a_per_set_underflow():
    g, _ = W.graph("weblech")
    v = 5
    sets = [[(v, True)], [(v, True), (v, False)], []]
    res = P.run_many(g, sets)
    assert res.errors[0] is None and res.errors[2] is None
    assert isinstance(res.errors[1], P.UnderflowError)
    o, _ = oracle_set(g, sets[1], EngineOptions())
    assert o["underflow"] is not None and o["underflow"][0] == 3  # marginal, like the reference
    e = res.errors[1]
    assert (e.kind, e.iteration, e.index) == o["underflow"]


def test_sweep_underflow_attribution_vs_oracle():
    """Per-set UnderflowError of the sweep == the reference's report for
    run(clamp_evidence(G, set j), PARALL), on contradictory random graphs."""
    from builders import contradictory_graph

    rng = np.random.default_rng(707)
    raised = 0
    for trial in range(25):
        g = contradictory_graph(rng, n_clamps=0)
        sets = random_sets(rng, g.num_variables, 40, max_size=5, allow_dup=True)
        opts = EngineOptions(max_iterations=30, tolerance=1e-9,
                             normalize_messages=trial % 5 != 2)
        res = P.run_many(g, sets, None, opts)
        check_against_oracle(g, sets, opts, res)
        raised += sum(e is not None for e in res.errors)
    assert raised >= 200, raised


def test_sweep_passes_equal_single_pass():
    g, _ = W.graph("hedc")
    rng = np.random.default_rng(5)
    sets = random_sets(rng, g.num_variables, 70)
    a = P.run_many(g, sets, capacity=32)
    cap = P.engine.device_graph(g).sweep(32).capacity  # rounded to the kernel's set unit
    assert a.passes == -(-len(sets) // cap) > 1
    b = P.run_many(g, sets, capacity=128)
    assert b.passes == 1
    assert a.marginals.tobytes() == b.marginals.tobytes()
    assert (a.iterations == b.iterations).all()


def test_sweep_selection_and_device_ranking():
    g, alarms = W.graph("avrora")
    rng = np.random.default_rng(9)
    ids = np.asarray(alarms.alarms)
    labels = np.asarray(alarms.labels)
    sets = []
    for j in range(24):
        pick = np.sort(rng.choice(len(ids), 8, replace=False))
        sets.append(list(zip(ids[pick].tolist(), labels[pick].tolist())))
    sel = np.sort(ids)
    res = P.run_many(g, sets, select=sel, topk=50)
    for j, pairs in enumerate(sets):
        assert res.p1_select[j].tobytes() == res.marginals[j][sel, 1].tobytes()
        want = rank_alarms(res.marginals[j], alarms, [v for v, _ in pairs])[:50]
        assert res.ranked[j].tolist() == want, j


def test_sweep_golden_c5_sets(golden):
    g, alarms = W.graph("ftp")
    sets = [W.evidence_set(alarms, j) for j in range(4)]
    sel = np.sort(np.asarray(alarms.alarms))
    res = P.run_many(g, sets, Strategy.parall(), EngineOptions(1000, 1e-9), select=sel, topk=100)
    for j in range(4):
        want = golden["sweep"][str(j)]
        assert res.iterations[j] == want["iterations"]
        assert sha(res.marginals[j]) == want["marginals_sha"]
        ranked = res.ranked[j].tolist()
        assert ranked[:10] == want["top10"]
        assert sha(np.asarray(ranked[:100], dtype=np.int64)) == want["top100_sha"]


def test_sweep_time_limit_and_max_iterations():
    g, _ = W.graph("hedc")
    sets = [[], [(1, True)]]
    res = P.run_many(g, sets, options=EngineOptions(max_iterations=3, tolerance=0.0))
    assert list(res.iterations) == [3, 3] and not res.converged.any()
    res = P.run_many(g, sets, options=EngineOptions(max_iterations=1000, tolerance=0.0,
                                                   time_limit=1e-6))
    assert (res.iterations >= 1).all() and (res.iterations < 1000).all()


def test_sweep_non_parall_strategy_materialises():
    g, _ = W.graph("weblech")
    sets = [[(3, True)], [(7, False), (9, True)]]
    res = P.run_many(g, sets, Strategy.seqfix(), EngineOptions(1000, 1e-9))
    for j, pairs in enumerate(sets):
        cur = clamp_all(g, pairs)
        r = P.run(cur, Strategy.seqfix().compile(cur), EngineOptions(1000, 1e-9))
        assert res.marginals[j].tobytes() == r.marginals.tobytes()


def test_sweep_long_rows_heavy_chunks():
    """Rows longer than a staged chunk (32 rows) take the heavy path (rows read
    from global memory); bitwise against the oracle, evidence on the hub."""
    from builders import hub_graph
    rng = np.random.default_rng(321)
    g = hub_graph(rng, hub_degree=45, wide_body=44)
    sets = [[], [(0, True)], [(0, False), (3, True)], [(g.num_variables - 2, True)]] + \
        random_sets(rng, g.num_variables, 40, max_size=3)
    opts = EngineOptions(max_iterations=80, tolerance=1e-12)
    res = P.run_many(g, sets, None, opts)
    check_against_oracle(g, sets, opts, res)


@pytest.mark.parametrize("name,n,min_compactions", [("weblech", 300, 2), ("hedc", 160, 1),
                                                    ("hedc", 640, 2)])
def test_sweep_compaction_every_set_bitwise(name, n, min_compactions):
    """Many sets with spread-out convergence: the staged kernel packs the
    stragglers into fewer tiles mid-run, repeatedly (each compaction into its
    own region of the alternate buffers) -- every set, stopped before, between
    or after them, must still equal the oracle bit for bit."""
    g, alarms = W.graph(name)
    rng = np.random.default_rng(2025)
    ids = np.asarray(alarms.alarms)
    labels = np.asarray(alarms.labels)
    sets = []
    for j in range(n):
        k = int(rng.integers(0, min(10, len(ids)) + 1))
        pick = rng.choice(len(ids), k, replace=False)
        sets.append(list(zip(ids[pick].tolist(), labels[pick].tolist())))
    opts = EngineOptions(1000, 1e-9)
    sel = np.sort(ids)
    res = P.run_many(g, sets, None, opts, select=sel, topk=min(20, len(sel)))
    assert res.compactions >= min_compactions, res.compactions
    check_against_oracle(g, sets, opts, res)
    for j, pairs in enumerate(sets):
        assert res.p1_select[j].tobytes() == res.marginals[j][sel, 1].tobytes()
        want = rank_alarms(res.marginals[j], alarms, [v for v, _ in pairs])[:min(20, len(sel))]
        assert res.ranked[j][:len(want)].tolist() == want, j


def test_sweep_ftp_many_sets_vs_oracle():
    """48 C5-style ftp sets (PARALL, tol 1e-9), every set against the oracle."""
    g, alarms = W.graph("ftp")
    sets = [W.evidence_set(alarms, j) for j in range(100, 148)]
    opts = EngineOptions(1000, 1e-9)
    res = P.run_many(g, sets, None, opts)
    for j, (ids, labels) in enumerate(sets):
        o, _ = oracle_set(g, list(zip(ids.tolist(), labels.tolist())), opts)
        assert res.iterations[j] == o["iterations"], j
        assert res.marginals[j].tobytes() == o["marginals"].tobytes(), j


@pytest.mark.parametrize("name,n", [("hedc", 64), ("ftp", 16)])
def test_sweep_fp32_mode_within_1e5_of_fp64(name, n):
    """Optional fp32 mode (north star: marginals within 1e-5 of the fp64
    reference): fp32 message storage, fp64 arithmetic and marginals, in the
    same staged kernel."""
    g, alarms = W.graph(name)
    sets = [W.evidence_set(alarms, j, size=min(8, len(alarms))) for j in range(n)]
    opts64 = EngineOptions(1000, 1e-9)
    opts32 = EngineOptions(1000, 1e-9, precision="fp32")
    r64 = P.run_many(g, sets, None, opts64)
    r32 = P.run_many(g, sets, None, opts32)
    assert r32.converged.all()
    assert np.abs(r32.marginals - r64.marginals).max() < 1e-5
    assert (np.abs(r32.iterations - r64.iterations) <= 3).all()
    for j in range(min(4, n)):  # and against the oracle directly
        ids, labels = sets[j]
        o, _ = oracle_set(g, list(zip(ids.tolist(), labels.tolist())), opts64)
        assert np.abs(r32.marginals[j] - o["marginals"]).max() < 1e-5


def test_fp32_is_parall_only():
    g, _ = W.graph("weblech")
    with pytest.raises(ValueError):
        P.run(g, Strategy.seqfix().compile(g), EngineOptions(precision="fp32"))
    with pytest.raises(ValueError):
        P.run_many(g, [[]], Strategy.seqfix(), EngineOptions(precision="fp32"))


def test_sweep_fp32_mode_with_compaction():
    """fp32 message storage through a straggler compaction (many sets of
    spread-out convergence): still within the 1e-5 bar of the fp64 sweep,
    identical top-20 rankings."""
    g, alarms = W.graph("weblech")
    rng = np.random.default_rng(7)
    ids = np.asarray(alarms.alarms)
    labels = np.asarray(alarms.labels)
    sets = []
    for j in range(300):
        k = int(rng.integers(0, min(10, len(ids)) + 1))
        pick = rng.choice(len(ids), k, replace=False)
        sets.append(list(zip(ids[pick].tolist(), labels[pick].tolist())))
    sel = np.sort(ids)
    topk = min(20, len(sel))
    r64 = P.run_many(g, sets, None, EngineOptions(1000, 1e-9), select=sel, topk=topk)
    r32 = P.run_many(g, sets, None, EngineOptions(1000, 1e-9, precision="fp32"), select=sel,
                     topk=topk)
    assert r32.compactions >= 1
    assert np.abs(r32.marginals - r64.marginals).max() < 1e-5
    assert np.abs(r32.p1_select - r64.p1_select).max() < 1e-5
    same = sum(r32.ranked[j].tolist() == r64.ranked[j].tolist() for j in range(len(sets)))
    assert same >= 0.99 * len(sets)


def test_sweep_empty_and_csr_inputs():
    """Zero sets (list or CSR) give empty results; an EvidenceCSR with a
    duplicated observation equals the same sets in list form, bit for bit."""
    g, _ = W.graph("weblech")
    r = P.run_many(g, [])
    assert len(r.iterations) == 0 and r.marginals.shape == (0, g.num_variables, 2)
    assert len(P.run_many(g, P.EvidenceCSR([0], [], [])).iterations) == 0
    a = P.run_many(g, P.EvidenceCSR([0, 0, 2], [5, 5], [1, 1]))
    b = P.run_many(g, [[], [(5, True), (5, True)]])
    assert a.marginals.tobytes() == b.marginals.tobytes()
    assert list(a.iterations) == list(b.iterations) and a.errors == b.errors == [None, None]


def test_ranking_keeps_alarms_with_p1_exactly_zero():
    """An unlabeled alarm whose P1 is exactly 0.0 (derived only through a
    false-clamped tuple by a deterministic OR, synth.py's p1=1, p2=0) is still
    ranked -- last, by id -- like rank_alarms (ranking.py:83-91)."""
    from paper_2509_22337_b200 import AlarmSet

    g = FactorGraph(4, [Factor(FactorKind.AND, 0, (), 0.5, 0.5),
                        Factor(FactorKind.OR, 1, (0,), 1.0, 0.0),
                        Factor(FactorKind.OR, 3, (0,), 1.0, 0.0),
                        Factor(FactorKind.AND, 2, (), 0.3, 0.3)])
    alarms = AlarmSet((0, 1, 2, 3), (False, False, True, False))
    sets = [[(0, False)], [(0, False), (2, True)], []]
    sel = np.arange(4)
    res = P.run_many(g, sets, select=sel, topk=4)
    for j, pairs in enumerate(sets):
        assert res.marginals[j].shape == (4, 2)
        want = rank_alarms(res.marginals[j], alarms, [v for v, _ in pairs])
        got = [v for v in res.ranked[j].tolist() if v >= 0]
        assert got == want, (j, got, want)
    assert res.marginals[0][1, 1] == 0.0 and 1 in res.ranked[0].tolist()
    # the single-graph device ranking (interaction_loop's argmax) as well
    dg = P.engine.device_graph(g)
    plan = dg.plan(Strategy.parall().compile(g), g)
    dg.set_evidence([0, 2], [0, 1])
    try:
        plan.run(EngineOptions(), g)
        top, p1 = dg.rank(np.array([1, 2, 3], dtype=np.int32), 1)
        assert top[0] == 1 and p1[0] == 0.0
        top, _ = dg.rank(np.array([1, 2, 3], dtype=np.int32), 3)
        assert top.tolist() == [1, 3, -1]
    finally:
        dg.set_evidence([], [])
